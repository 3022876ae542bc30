#!/bin/bash
# tile x tile terms applied directly in the dense-mode accumulation: 524K timing + parity
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=600
O=gpurun_out/r2z_sweep.jsonl
: > $O
echo "== tt-direct" >> $O
timeout 300 python tools/perf_probe.py 524288 0.5 0.1 1e-6 20 1 >> $O 2>>gpurun_out/r2z_err.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_grid.py tests/test_gpu_batch.py tests/test_gpu_truncate.py -q -x > gpurun_out/r2z_tests.log 2>&1
echo "exit $?" >> gpurun_out/r2z_tests.log
