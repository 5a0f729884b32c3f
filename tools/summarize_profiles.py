"""Turn the ncu captures of tools/profile_round.sh (gpurun_out/) into committed summaries under
profiles/ (per round): launch-list shares and the key --set full metrics of the top kernels."""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__t_bytes.sum"]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        res.append((d.get("Kernel Name", "?"), {m: (d.get(m), u.get(m)) for m in METRICS if m in d}))
    return res


def launches():
    path = os.path.join(OUT, "launches.csv")
    agg = collections.defaultdict(lambda: [0, 0.0])
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0].split("::")[-1]
                v = float(d["Metric Value"].replace(",", ""))
                scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(d["Metric Unit"], 1.0)
                agg[name][0] += 1
                agg[name][1] += v * scale
    return agg


os.makedirs(PROF, exist_ok=True)
lines = [f"# {rnd}: ncu launch list of `python bench.py --steps 2 --warmup 3 --no-kernels --no-cpu-baseline`",
         "# (--metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised: compare SHARES)",
         "# includes index build + dataset load + 5 k-NN steps of 1000 queries", ""]
agg = launches()
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"{k:44s} launches={v[0]:5d} total_ms={v[1]:9.3f} share={v[1] / tot * 100:5.1f}%")
open(os.path.join(PROF, f"{rnd}_launches.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:16]))

traffic = {}
summ = [f"# {rnd}: key metrics from `ncu --set full --clock-control none` (tools/profile_round.sh)", ""]
for rep, what in [("prof_knn.ncu-rep", "kprof knn --queries 1000 (the bench batch: one ft_knn call; the fused prefilter "
                                     "is k_qt on the 1/32 sample, k_row_threshold, k_qt threshold scan, k_select_fast "
                                     "on the lists, and the (idle) fallback k_qt / k_select_fast)"),
                  ("prof_ftd.ncu-rep", "kprof ft --queries 64 (exhaustive Flowtree over 100k docs: k_ftd + list-mode k_flowtree)"),
                  ("prof_img.ncu-rep", "kprof ft --config image --queries 16 (exhaustive Flowtree over 60k image docs: k_flowtree)"),
                  ("prof_exact.ncu-rep", "kprof exact --queries 1000 (QT 424 -> FT 9 -> exact W1, transportation simplex)")]:
    p = os.path.join(OUT, rep)
    if not os.path.exists(p):
        continue
    summ.append(f"## {rep}: {what}")
    for name, ms in raw_metrics(p):
        short = name.split("(")[0].split("::")[-1]
        summ.append(f"### {short}")
        for m, (v, u) in ms.items():
            summ.append(f"  {m} = {v} {u}")
        # the Flowtree stage is k_ftd plus the list-mode k_flowtree: their traffic is summed
        # the quadtree stage = every prefilter kernel of the call; the Flowtree stage = k_ftd + k_flowtree
        key = {("k_qt", "prof_knn.ncu-rep"): "quadtree", ("k_row_threshold", "prof_knn.ncu-rep"): "quadtree",
               ("k_dist_i8", "prof_knn.ncu-rep"): "dist_table",
               ("k_ftd", "prof_knn.ncu-rep"): "flowtree", ("k_flowtree", "prof_knn.ncu-rep"): "flowtree"}.get(
            (short.split("<")[0], rep))
        if key:
            rd = float(ms["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(ms["dram__bytes_write.sum"][0].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            kk = f"{key}_dram_bytes_per_launch"
            traffic[kk] = traffic.get(kk, 0.0) + rd * scale.get(ms["dram__bytes_read.sum"][1], 1) + \
                wr * scale.get(ms["dram__bytes_write.sum"][1], 1)
        summ.append("")
open(os.path.join(PROF, f"{rnd}_ncu_summary.txt"), "w").write("\n".join(summ) + "\n")
if traffic:
    traffic["source"] = (f"profiles/{rnd}_ncu_summary.txt: dram read+write of one ncu --set full capture of "
                         "kprof knn on the 1000-query bench batch (one ft_knn call, as one bench step): quadtree = "
                         "the k_qt launches + k_row_threshold of the fused prefilter; dist_table = k_dist_i8; "
                         "flowtree = k_ftd + list-mode k_flowtree")
    json.dump(traffic, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)
    print(traffic)
