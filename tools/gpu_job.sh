set -u
mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py -x -q -k "tiny or subsets or vocab_hash or capped or degenerate or image or chunked" > gpurun_out/pytest_b2.log 2>&1; echo "rc $?" >> gpurun_out/pytest_b2.log
python tools/variant_bench.py image 200 main nob > gpurun_out/vb_img2.log 2>&1
