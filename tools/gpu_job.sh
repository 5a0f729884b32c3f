set -u
mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py -x -q -k "distance or subsets or full_size" > gpurun_out/pytest_kz.log 2>&1; echo "rc $?" >> gpurun_out/pytest_kz.log
python tools/variant_bench.py reviews 1000 prev main > gpurun_out/vb_kz.log 2>&1
