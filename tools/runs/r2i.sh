#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_truncate.py -m gpu -q -rf -p no:cacheprovider -k "dense_mode or full_rank_tight" > gpurun_out/r2i_trunc.log 2>&1
echo "exit $?" >> gpurun_out/r2i_trunc.log
HCOV_VERBOSE=1 timeout 900 python -m pytest tests/test_gpu_diagnostics.py -m gpu -q -rA -x -p no:cacheprovider > gpurun_out/r2i_diag.log 2>&1
echo "exit $?" >> gpurun_out/r2i_diag.log
