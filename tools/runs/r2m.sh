#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/diag_spd2.py > gpurun_out/r2m_spd2.log 2>&1
echo "exit $?" >> gpurun_out/r2m_spd2.log
