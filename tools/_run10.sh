export HCOV_WATCHDOG_S=150
timeout 200 python tools/gpu_debug.py small > gpurun_out/r10_small.log 2>&1; echo "small rc=$?"
timeout 300 python tools/timeline.py run tl65k 65536 0.5 0.1 1e-6 20 > gpurun_out/r10.log 2>&1; echo "tl rc=$?"
timeout 300 python tools/timeline.py run tl131k 131072 0.5 0.0864 1e-6 16 >> gpurun_out/r10.log 2>&1; echo "tl rc=$?"
timeout 300 python tools/timeline.py run tl131kc5 131072 1.0 0.05 1e-6 20 >> gpurun_out/r10.log 2>&1; echo "tl rc=$?"
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r10_pytest.log; echo "pytest done"
timeout 600 python tools/timeline.py run tl524k 524288 0.5 0.1 1e-6 20 >> gpurun_out/r10.log 2>&1; echo "tl rc=$?"
