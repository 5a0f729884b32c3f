set -u
mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py -x -q -k "chunk_pairs or knn or prefilter or quadtree or full_size_sampled" > gpurun_out/pytest_small.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_small.log
python tools/chunk_sweep.py reviews 0 > gpurun_out/stages.log 2>&1
python tools/chunk_sweep.py stress 0 >> gpurun_out/stages.log 2>&1
