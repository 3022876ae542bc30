#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/dbg_factor.py 1200 bisect > gpurun_out/r2h_dbg.log 2>&1
echo "dbg exit $?" >> gpurun_out/r2h_dbg.log
