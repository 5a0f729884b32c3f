set -u
mkdir -p gpurun_out
python tools/chunk_sweep.py reviews 0 256 128 64 32 16 > gpurun_out/chunk_reviews.log 2>&1
python tools/chunk_sweep.py stress 0 128 64 32 16 > gpurun_out/chunk_stress.log 2>&1
