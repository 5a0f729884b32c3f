set -u
mkdir -p gpurun_out
python tools/opt_sweep.py reviews FT_OPT_QT_WAVES 4 6 8 12 16 > gpurun_out/waves.log 2>&1
python tools/opt_sweep.py stress FT_OPT_QT_WAVES 4 6 8 12 16 >> gpurun_out/waves.log 2>&1
