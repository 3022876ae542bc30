export HCOV_WATCHDOG_S=1200
timeout 1500 python tools/timeline.py run tl2m_t4 2097152 0.33 0.65 1e-5 20 0 1e-4 > gpurun_out/r19.log 2>&1; echo "tl rc=$?"
timeout 1500 python tools/timeline.py run tl2m_c4 2097152 0.5 0.1 1e-6 20 0 1e-6 >> gpurun_out/r19.log 2>&1; echo "tl rc=$?"
