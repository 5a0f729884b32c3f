set -u
mkdir -p gpurun_out
: > gpurun_out/drb.log
for v in base drb12 drb16 drb12m3; do
  echo "== $v" >> gpurun_out/drb.log
  L=""; [ "$v" != base ] && L="FT_LIB=$PWD/build/variants/$v/libflowtree_b200.so"
  env $L python tools/ft_exh.py reviews 64 >> gpurun_out/drb.log 2>&1
  env $L python tools/chunk_sweep.py reviews 0 >> gpurun_out/drb.log 2>&1
done
