#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/dbg_race.py > gpurun_out/r2k_race.log 2>&1
echo "exit $?" >> gpurun_out/r2k_race.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_grid.py -m gpu -q -rA -s -p no:cacheprovider > gpurun_out/r2k_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2k_pytest.log
