#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for args in "2097152 1 1e-5 20 20" "2097152 0 1e-5 20 20" "2097152 1 1e-5 20 24"; do
  HCOV_VERBOSE=1 timeout 900 python tools/diag_spd4.py $args >> gpurun_out/r2o_spd4.log 2>&1
  echo "exit $? ($args)" >> gpurun_out/r2o_spd4.log
done
