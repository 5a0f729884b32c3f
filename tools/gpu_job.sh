set -u
mkdir -p gpurun_out
: > gpurun_out/grp.log
for v in base g48 g64b32; do
  echo "== $v" >> gpurun_out/grp.log
  L=""; [ "$v" != base ] && L="FT_LIB=$PWD/build/variants/$v/libflowtree_b200.so"
  env $L python tools/chunk_sweep.py reviews 0 >> gpurun_out/grp.log 2>&1
  env $L python tools/chunk_sweep.py stress 0 >> gpurun_out/grp.log 2>&1
  env $L python tools/ft_exh.py reviews 64 >> gpurun_out/grp.log 2>&1
  env $L python tools/ft_exh.py text 64 >> gpurun_out/grp.log 2>&1
done
