set -u
mkdir -p gpurun_out
timeout 300 python tools/fuzz_parity.py --gen 3 --only 1818 > gpurun_out/s1818.log 2>&1; echo "rc $?" >> gpurun_out/s1818.log
FT_LIB=$PWD/paper_1910_04126_b200/libflowtree_b200_checked.so timeout 800 python tools/fuzz_parity.py --poison --random-opts --gen 3 --seconds 420 --seed0 5000 > gpurun_out/fuzz7.log 2>&1; echo "fuzz rc $?" >> gpurun_out/fuzz7.log
