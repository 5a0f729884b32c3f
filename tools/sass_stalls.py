"""Top SASS lines by warp-stall samples from `ncu -i REP -k KERNEL --page source --csv --print-source sass`.
python tools/sass_stalls.py file.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
tot = sum(f(r[si]) for r in data)
toti = sum(f(r[ii]) for r in data)
print("samples", tot, "warp instr", toti)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 45
idx = sorted(range(len(data)), key=lambda i: -f(data[i][si]))[:n]
for i in sorted(idx):
    r = data[i]
    print(i, f"{f(r[si]) / tot * 100:5.1f}% {f(r[ii]) / toti * 100:5.2f}%i", r[1][:90])
