set -u
mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/fuzz_parity.py --seed0 6855 --max-cases 8 2>&1 | cut -c1-300 | grep -v "^ok" > gpurun_out/repro_opts.log
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "flowtree or flow_export or lane_per_pair or full_size or degenerate or capped or knn or bounds" > gpurun_out/pytest_sub.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_sub.log
for c in reviews text stress; do timeout 300 python tools/ft_exh.py $c $([ $c = stress ] && echo 16 || echo 64) >> gpurun_out/exh.log 2>&1; done
FT_LIB=$PWD/paper_1910_04126_b200/libflowtree_b200_checked.so timeout 700 python tools/fuzz_parity.py --poison --seed0 5400 --seconds 500 2>&1 | grep -v "^ok" > gpurun_out/fuzz_checked.log
