#!/bin/bash
# dense/factor-mode split A/B at 524K (HCOV_BIG_M), parity spot checks with the factor mode at m = 256
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=600
O=gpurun_out/r2y_sweep.jsonl
: > $O
run() { echo "== $*" >> $O; env "$@" timeout 300 python tools/perf_probe.py 524288 0.5 0.1 1e-6 20 1 >> $O 2>>gpurun_out/r2y_err.log; }
run HCOV_X=base
run HCOV_BIG_M=128
run HCOV_BIG_M=64
run HCOV_BIG_M=128 HCOV_RCHUNK=4
HCOV_BIG_M=128 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_grid.py tests/test_gpu_accuracy.py -q -x > gpurun_out/r2y_tests128.log 2>&1
echo "exit $?" >> gpurun_out/r2y_tests128.log
