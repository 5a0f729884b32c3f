set -u
mkdir -p gpurun_out
FT_LIB=$PWD/paper_1910_04126_b200/libflowtree_b200_checked.so timeout 1000 python tools/fuzz_parity.py --poison --seconds 800 --seed0 20000 > gpurun_out/fuzz4.log 2>&1; echo "fuzz rc $?" >> gpurun_out/fuzz4.log
