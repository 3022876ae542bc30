export HCOV_WATCHDOG_S=100
timeout 200 python tools/gpu_debug.py small > gpurun_out/r6_small.log 2>&1; echo "small rc=$?"
timeout 300 python tools/timeline.py run tl65k 65536 0.5 0.1 1e-6 20 > gpurun_out/r6.log 2>&1; echo "tl rc=$?"
timeout 300 python tools/timeline.py run tl131k 131072 0.5 0.0864 1e-6 16 >> gpurun_out/r6.log 2>&1; echo "tl rc=$?"
