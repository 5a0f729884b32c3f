#!/bin/bash
# Run on the GPU box (gpurun): launch list of the bench command + ncu --set full of the top kernels.
# Each ncu command runs only after the same command line exited 0 without ncu.  (The selection
# kernels are left out of the full captures: under ncu's instrumentation k_select_fast fails to
# launch — it runs at the 64-register cap with the maximum shared-memory carveout — and the
# target application then aborts before the distance-table and Flowtree kernels.)
set -u
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-kernels --no-cpu-baseline --no-configs"
$B > gpurun_out/bench_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B \
  > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
K="python tools/kprof.py knn --queries 1000 --reps 1"
$K > gpurun_out/kp_knn.log 2>&1 && \
  ncu --set full --clock-control none --import-source on \
  -k regex:"k_qt$|k_row_threshold|k_dist_i8|k_ftd|k_flowtree|k_vocab|k_tiles|k_dist_prep" -c 12 \
  -o gpurun_out/prof_knn $K > gpurun_out/ncu_knn.log 2>&1
echo "knn rc=$?"
X="python tools/kprof.py ft --queries 64 --reps 1"
$X > gpurun_out/kp_ftd.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_ftd|k_flowtree" -c 2 -o gpurun_out/prof_ftd $X \
  > gpurun_out/ncu_ftd.log 2>&1
echo "ftd rc=$?"
I="python tools/kprof.py ft --config image --queries 16 --reps 1"
$I > gpurun_out/kp_img.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_flowtree" -c 1 -o gpurun_out/prof_img $I \
  > gpurun_out/ncu_img.log 2>&1
echo "img rc=$?"
E="python tools/kprof.py exact --queries 1000 --reps 1"
$E > gpurun_out/kp_exact.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_exact" -c 1 -o gpurun_out/prof_exact $E \
  > gpurun_out/ncu_exact.log 2>&1
echo "exact rc=$?"
