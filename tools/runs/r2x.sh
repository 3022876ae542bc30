#!/bin/bash
# schedule-knob sweep at 524K (perf_probe, one timed eval each) + 524K timeline of the default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=600
O=gpurun_out/r2x_sweep.jsonl
: > $O
run() { echo "== $*" >> $O; env "$@" timeout 300 python tools/perf_probe.py 524288 0.5 0.1 1e-6 20 1 >> $O 2>>gpurun_out/r2x_err.log; }
run HCOV_X=base
run HCOV_RCHUNK=2
run HCOV_RCHUNK=4
run HCOV_RCHUNK=6
run HCOV_RAPP512=2
run HCOV_GANG1_BELOW=1024
run HCOV_GANG1_BELOW=1024 HCOV_RCHUNK=4
run HCOV_GANG_MAX_SMALL=2
timeout 600 python tools/timeline.py run r2x_tl524k 524288 0.5 0.1 1e-6 20 > gpurun_out/r2x_tl524k.log 2>&1
echo "rc=$?" >> gpurun_out/r2x_tl524k.log
