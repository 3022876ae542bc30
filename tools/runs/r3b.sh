#!/bin/bash
# A/B at 524K of: min-rank term orientation (HCOV_TERM_MIN), DMMA dense accumulation (HCOV_DENSE_DMMA),
# vectorised band scan (always on); then the parity / accuracy suites on the defaults
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=600
O=gpurun_out/r3b_sweep.jsonl
: > $O
run() { echo "== $*" >> $O; env "$@" timeout 300 python tools/perf_probe.py 524288 0.5 0.1 1e-6 20 1 >> $O 2>>gpurun_out/r3b_err.log; }
run HCOV_X=default
run HCOV_TERM_MIN=0
run HCOV_DENSE_DMMA=0
run HCOV_TERM_MIN=0 HCOV_DENSE_DMMA=0
run HCOV_RCHUNK=4
run HCOV_RCHUNK=5
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_grid.py tests/test_gpu_batch.py tests/test_gpu_truncate.py tests/test_gpu_accuracy.py tests/test_gpu_spd.py tests/test_gpu_solve.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r3b_tests.log 2>&1
echo "exit $?" >> gpurun_out/r3b_tests.log
