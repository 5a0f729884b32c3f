"""Per-source-line totals from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur_file = None
out = []
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        ins = float(r[7].replace(",", "")); smp = float(r[4].replace(",", ""))
    except ValueError:
        continue
    out.append((ins, smp, cur_file, r[0], r[1][:90]))
tot_i = sum(o[0] for o in out); tot_s = sum(o[1] for o in out)
print(f"total instr {tot_i:.3e}  samples {tot_s:.0f}")
key = 1 if len(sys.argv) > 3 and sys.argv[3] == "stall" else 0
for o in sorted(out, key=lambda o: -o[key])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{o[0]/tot_i*100:5.1f}% ins {o[1]/max(tot_s,1)*100:5.1f}% stall  {o[2]}:{o[3]:>4}  {o[4]}")
