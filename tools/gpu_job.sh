set -u
mkdir -p gpurun_out
timeout 800 python tools/fuzz_parity.py --poison --gen 3 --seconds 500 --seed0 0 > gpurun_out/fuzz6.log 2>&1; echo "fuzz rc $?" >> gpurun_out/fuzz6.log
