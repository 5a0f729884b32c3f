"""Summarise an `ncu --page source --csv --print-source sass` dump: hottest instructions by
warp-stall samples and by executed instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


tot_s = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data)
tot_i = sum(num(d["Instructions Executed"]) for d in data)
print(f"instructions executed {tot_i:.3e}, stall samples {tot_s:.0f}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for d in sorted(data, key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))[:n]:
    st = sorted(((num(d[c]), c) for c in stall_cols), reverse=True)[:2]
    print(f"{num(d['Warp Stall Sampling (All Samples)'])/max(tot_s,1)*100:5.1f}% {num(d['Instructions Executed']):10.0f} "
          f"thr{num(d['Avg. Threads Executed']):5.1f} {d['Address']:>6} {d['Source'][:60]:60} {st}")
