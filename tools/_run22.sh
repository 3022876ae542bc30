export HCOV_WATCHDOG_S=600
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r22.log
timeout 900 python tools/timeline.py run tl524k 524288 0.5 0.1 1e-6 20 >> gpurun_out/r22.log 2>&1; echo "tl rc=$?"
