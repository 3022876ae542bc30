#!/bin/bash
# round 2, call G: factor-debug of the large-capacity defect; diagnostics tests after the solve-pool fix
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/dbg_factor.py 1200 > gpurun_out/r2g_dbg.log 2>&1
echo "dbg exit $?" >> gpurun_out/r2g_dbg.log
timeout 900 python -m pytest tests/test_gpu_diagnostics.py -m gpu -q -rA -p no:cacheprovider > gpurun_out/r2g_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2g_pytest.log
