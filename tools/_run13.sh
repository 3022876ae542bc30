export HCOV_WATCHDOG_S=150
timeout 300 python tools/timeline.py run tl131k 131072 0.5 0.0864 1e-6 16 > gpurun_out/r13.log 2>&1; echo "tl rc=$?"
