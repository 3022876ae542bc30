#!/bin/bash
# full GPU suite after the PHWR / slot fixes; C5-kernel SPD status
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -rA -p no:cacheprovider --durations=25 > gpurun_out/r2l_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2l_pytest.log
timeout 1500 python tools/diag_spd.py > gpurun_out/r2l_spd.log 2>&1
echo "exit $?" >> gpurun_out/r2l_spd.log
