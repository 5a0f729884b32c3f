set -u
mkdir -p gpurun_out
: > gpurun_out/ncopy.log
for v in base c96 c128 c128e4; do
  echo "== $v" >> gpurun_out/ncopy.log
  L=""; [ "$v" != base ] && L="FT_LIB=$PWD/build/variants/$v/libflowtree_b200.so"
  env $L timeout 300 python tools/chunk_sweep.py reviews 0 >> gpurun_out/ncopy.log 2>&1
  env $L timeout 300 python tools/chunk_sweep.py stress 0 >> gpurun_out/ncopy.log 2>&1
  env $L timeout 300 python tools/ft_exh.py reviews 64 >> gpurun_out/ncopy.log 2>&1
done
