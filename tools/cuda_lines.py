"""Per-CUDA-line instruction and stall totals from `ncu --page source --csv --print-source cuda,sass`.
python tools/cuda_lines.py file.csv [N] [stall]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur = None
out = {}
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0]:
        continue

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    key = (cur, int(r[0]))
    o = out.setdefault(key, [0.0, 0.0, r[1][:90]])
    o[0] += f(r[7])
    o[1] += f(r[4])
ti = sum(v[0] for v in out.values())
ts = sum(v[1] for v in out.values())
print(f"total warp instr {ti:.4e} stall samples {ts:.0f}")
k = 1 if len(sys.argv) > 3 and sys.argv[3] == "stall" else 0
for (fn, ln), v in sorted(out.items(), key=lambda kv: -kv[1][k])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{v[0] / ti * 100:5.1f}% ins {v[1] / max(ts, 1) * 100:5.1f}% stall {fn}:{ln:<4} {v[2]}")
