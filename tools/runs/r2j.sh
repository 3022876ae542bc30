#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/dbg_race.py > gpurun_out/r2j_race.log 2>&1
echo "exit $?" >> gpurun_out/r2j_race.log
HCOV_VERBOSE=1 timeout 900 python -m pytest tests/test_gpu_diagnostics.py tests/test_gpu_solve.py -m gpu -q -rA -x -p no:cacheprovider > gpurun_out/r2j_diag.log 2>&1
echo "exit $?" >> gpurun_out/r2j_diag.log
