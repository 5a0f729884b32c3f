set -u
mkdir -p gpurun_out
python tools/variant_bench.py reviews 1000 st ko ko6 ko4 > gpurun_out/vb_ko.log 2>&1
