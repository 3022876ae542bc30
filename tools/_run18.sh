export HCOV_WATCHDOG_S=1200
timeout 1500 python tools/timeline.py run tl2m_n4 2097152 1.0 0.05 1e-5 20 0 1e-4 > gpurun_out/r18.log 2>&1; echo "tl rc=$?"
timeout 600 python tools/timeline.py run tl524k_c5 524288 1.0 0.05 1e-6 20 0 1e-6 >> gpurun_out/r18.log 2>&1; echo "tl rc=$?"
