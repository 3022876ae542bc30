#!/bin/bash
# round-2 re-entry check: full GPU suite, default 2M bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=1200
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/r2w_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2w_tests.log
timeout 1500 python bench.py --out gpurun_out/r2w_bench2m.json > gpurun_out/r2w_bench2m.log 2>&1
echo "bench exit $?" >> gpurun_out/r2w_bench2m.log
