set -u
mkdir -p gpurun_out
timeout 900 python tools/fuzz_parity.py --poison --directed > gpurun_out/directed.log 2>&1; echo "rc $?" >> gpurun_out/directed.log
timeout 200 python tools/fuzz_parity.py --only 20313 > gpurun_out/s20313.log 2>&1; echo "rc $?" >> gpurun_out/s20313.log
