#!/bin/bash
# 2M engine timeline (critical chain) on the final library; C4 MLE continuation from the checkpoint
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=1800
timeout 900 python tools/timeline.py run tl2m_r3j 2097152 0.5 0.1 1e-6 20 > gpurun_out/r3j_tl2m.log 2>&1; echo "tl rc=$?" >> gpurun_out/r3j_tl2m.log
timeout ${MLE_TIMEOUT:-1500} python tools/mle_run.py --iters-now ${MLE_ITERS:-3} > gpurun_out/r3j_mle.log 2>&1
echo "mle exit $?" >> gpurun_out/r3j_mle.log
