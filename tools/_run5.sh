export HCOV_WATCHDOG_S=200
timeout 300 python tools/timeline.py run tl16k 16384 1.5 0.05 1e-4 0 > gpurun_out/r5.log 2>&1
timeout 300 python tools/timeline.py run tl65k 65536 0.5 0.1 1e-6 20 >> gpurun_out/r5.log 2>&1
