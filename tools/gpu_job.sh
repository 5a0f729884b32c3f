set -u
mkdir -p gpurun_out
which compute-sanitizer > gpurun_out/san.log 2>&1; ls /usr/local/cuda/bin/compute-sanitizer >> gpurun_out/san.log 2>&1
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py >> gpurun_out/san.log 2>&1; echo "memcheck rc $?" >> gpurun_out/san.log
