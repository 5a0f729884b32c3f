set -u
mkdir -p gpurun_out
python tools/variant_bench.py reviews 1000 main pred dq > gpurun_out/vb_ftd.log 2>&1
FT_LIB=$PWD/build/variants/dq/libflowtree_b200.so python -m pytest tests/test_parity_gpu.py -x -q -k "flow or subsets or chunked or degenerate or full_size" > gpurun_out/pytest_dq.log 2>&1; echo "rc $?" >> gpurun_out/pytest_dq.log
