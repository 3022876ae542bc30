export HCOV_WATCHDOG_S=1200
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/r17_pytest.log; echo "pytest done"
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/r17_mem.log
timeout 2400 python tools/timeline.py run tl2m 2097152 1.0 0.05 1e-6 20 > gpurun_out/r17.log 2>&1; echo "tl rc=$?"
