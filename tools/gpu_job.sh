set -u
mkdir -p gpurun_out
for v in h03 h045 h08; do
  FT_LIB=$PWD/build/variants/$v/libflowtree_b200.so python tools/chunk_sweep.py reviews 0 > gpurun_out/hv_$v.log 2>&1
  FT_LIB=$PWD/build/variants/$v/libflowtree_b200.so python tools/chunk_sweep.py stress 0 >> gpurun_out/hv_$v.log 2>&1
done
FT_OPT=1 python -c "
import sys; sys.argv=['x','reviews','0']
" 
