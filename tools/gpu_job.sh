set -u
mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py -x -q -k "prefilter or full_size or knn" > gpurun_out/pytest_pf.log 2>&1; echo "rc $?" >> gpurun_out/pytest_pf.log
python tools/variant_bench.py reviews 1000 main > gpurun_out/vb_pf.log 2>&1
python tools/variant_bench.py stress 256 main >> gpurun_out/vb_pf.log 2>&1
python tools/variant_bench.py reviews:q48 1000 main g48 >> gpurun_out/vb_pf.log 2>&1
