set -u
mkdir -p gpurun_out
: > gpurun_out/var.log
V=$PWD/build/variants
FT_LIB=$V/w8b5/libflowtree_b200.so timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "flowtree or flow_export or lane_per_pair or full_size or degenerate or capped or knn" > gpurun_out/pytest_w.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_w.log
for v in base w16b3 w16b2 w8b5 w8b4 w8b6; do
  echo "== $v" >> gpurun_out/var.log
  L=""; [ "$v" != base ] && L="FT_LIB=$V/$v/libflowtree_b200.so"
  env $L timeout 300 python tools/ft_exh.py reviews 64 >> gpurun_out/var.log 2>&1
  env $L timeout 300 python tools/ft_exh.py text 64 >> gpurun_out/var.log 2>&1
  env $L timeout 300 python tools/ft_exh.py stress 16 >> gpurun_out/var.log 2>&1
done
timeout 600 python tools/variant_bench.py reviews 1000 main w16b3 w16b2 w8b5 w8b4 w8b6 >> gpurun_out/var.log 2>&1
