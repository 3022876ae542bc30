#!/bin/bash
# C4 MLE continuation from the checkpoint in profiles/ (2 iterations)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=900
timeout 800 python tools/mle_run.py --iters-now 2 --trace gpurun_out/r3k_trace.jsonl --out gpurun_out/r3k_result.json > gpurun_out/r3k_mle.log 2>&1
echo "mle exit $?" >> gpurun_out/r3k_mle.log
