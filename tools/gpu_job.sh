set -u
mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py -x -q -k "lane_per_pair or chunked or flow_export or degenerate or subsets or full_size_sampled or tile_major or bounds_checked" > gpurun_out/pytest_small.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_small.log
