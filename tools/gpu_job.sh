set -u
mkdir -p gpurun_out
python -m pytest tests/test_multiproc.py tests/test_parity_gpu.py -x -q -m gpu -k "library_doc_sharded or bounds_checked or two_shard" > gpurun_out/pytest_mp.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_mp.log
