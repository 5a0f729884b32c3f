set -u
mkdir -p gpurun_out
timeout 1000 python tools/fuzz_parity.py --poison --random-opts --seconds 700 --seed0 30000 > gpurun_out/fuzz5.log 2>&1; echo "fuzz rc $?" >> gpurun_out/fuzz5.log
