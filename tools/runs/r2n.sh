#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spd.py -m gpu -q -rA -p no:cacheprovider > gpurun_out/r2n_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2n_pytest.log
HCOV_VERBOSE=1 timeout 1800 python tools/diag_spd3.py > gpurun_out/r2n_spd3.log 2>&1
echo "exit $?" >> gpurun_out/r2n_spd3.log
