export HCOV_WATCHDOG_S=150
timeout 200 python tools/gpu_debug.py small > gpurun_out/r14_small.log 2>&1; echo "small rc=$?"
timeout 300 python tools/timeline.py run tl131k 131072 0.5 0.0864 1e-6 16 > gpurun_out/r14.log 2>&1; echo "tl rc=$?"
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r14_pytest.log; echo "pytest done"
