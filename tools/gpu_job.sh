set -u
mkdir -p gpurun_out
I="python tools/kprof.py ft --config image --queries 16 --reps 1"
$I > gpurun_out/kp_img.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_ftg" -c 1 -o gpurun_out/prof_ftg $I \
  > gpurun_out/ncu_ftg.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_ftg.log
