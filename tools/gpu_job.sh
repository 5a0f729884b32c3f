set -u
mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py -x -q -k "lane_per_pair or chunked or flow_export or degenerate or full_size_sampled or knn" > gpurun_out/pytest_small.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_small.log
python tools/ft_exh.py reviews 64 > gpurun_out/minb.log 2>&1
python tools/chunk_sweep.py reviews 0 >> gpurun_out/minb.log 2>&1
python tools/chunk_sweep.py stress 0 >> gpurun_out/minb.log 2>&1
