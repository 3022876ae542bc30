export HCOV_WATCHDOG_S=150
timeout 300 python tools/timeline.py run tl131k 131072 0.5 0.0864 1e-6 16 > gpurun_out/r12.log 2>&1; echo "tl rc=$?"
timeout 600 python tools/timeline.py run tl524k 524288 0.5 0.1 1e-6 20 >> gpurun_out/r12.log 2>&1; echo "tl rc=$?"
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r12_pytest.log; echo "pytest done"
