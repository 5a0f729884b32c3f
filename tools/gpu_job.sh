set -u
mkdir -p gpurun_out
timeout 900 python tools/fuzz_parity.py --poison --seconds 600 --seed0 2000 > gpurun_out/fuzz3.log 2>&1; echo "fuzz rc $?" >> gpurun_out/fuzz3.log
