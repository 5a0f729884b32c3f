set -u
mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py -x -q -k "tile_major or chunked or lane_per_pair or flow_export or subsets or near_pairs or degenerate" > gpurun_out/pytest_small.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_small.log
python tools/ft_exh.py reviews 64 > gpurun_out/ftexh.log 2>&1
python tools/ft_exh.py text 64 >> gpurun_out/ftexh.log 2>&1
python tools/ft_exh.py stress 16 >> gpurun_out/ftexh.log 2>&1
python tools/chunk_sweep.py text 0 >> gpurun_out/ftexh.log 2>&1
