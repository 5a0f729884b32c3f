# The round's GPU job (gpurun -- bash tools/gpu_job.sh): full GPU suite, smoke, both bench arms, ncu profiles.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_line.json 2> gpurun_out/bench_err.log; echo "bench rc $?" >> gpurun_out/bench_err.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref_err.log; echo "ref rc $?" >> gpurun_out/bench_ref_err.log
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1
