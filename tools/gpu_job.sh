set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "knn or prefilter or full_size or vocab or quadtree" > gpurun_out/pytest_sub.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_sub.log
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-kernels --no-cpu-baseline --no-configs > gpurun_out/bench_quick_$i.json 2> gpurun_out/bench_quick_err.log; done
