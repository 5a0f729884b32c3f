set -u
mkdir -p gpurun_out
: > gpurun_out/var.log
for v in base pv m2 pvm2; do
  echo "== $v" >> gpurun_out/var.log
  L=""; [ "$v" != base ] && L="FT_LIB=$PWD/build/variants/$v/libflowtree_b200.so"
  env $L timeout 300 python tools/ft_exh.py reviews 64 >> gpurun_out/var.log 2>&1
  env $L timeout 300 python tools/ft_exh.py text 64 >> gpurun_out/var.log 2>&1
  env $L timeout 300 python tools/ft_exh.py stress 16 >> gpurun_out/var.log 2>&1
done
timeout 600 python tools/variant_bench.py reviews 1000 main pv m2 pvm2 >> gpurun_out/var.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
