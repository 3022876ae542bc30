export HCOV_WATCHDOG_S=1200
timeout 2400 python tools/timeline.py run tl2m 2097152 1.0 0.05 1e-6 20 > gpurun_out/r16.log 2>&1; echo "tl rc=$?"
