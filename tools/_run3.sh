export HCOV_WATCHDOG_S=40
timeout 180 python tools/gpu_debug.py small > gpurun_out/r3_small.log 2>&1; echo "small rc=$?"
timeout 300 python tools/gpu_debug.py big > gpurun_out/r3_big.log 2>&1; echo "big rc=$?"
