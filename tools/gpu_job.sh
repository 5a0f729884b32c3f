set -u
mkdir -p gpurun_out
timeout 1300 python tools/fuzz_parity.py --poison --seconds 1000 > gpurun_out/fuzz2.log 2>&1; echo "fuzz rc $?" >> gpurun_out/fuzz2.log
