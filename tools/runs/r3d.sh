#!/bin/bash
# chunk-size / panel-width A/B (524K, then 2M for the candidates), then the full GPU suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=900
O=gpurun_out/r3d_sweep.jsonl
: > $O
K4=$GRAFT_REPO_ROOT/paper_1709_08625_b200/libhcov_k4.so
run() { echo "== $*" >> $O; env "$@" timeout 600 python tools/perf_probe.py $N 0.5 0.1 1e-6 20 1 >> $O 2>>gpurun_out/r3d_err.log; }
N=524288
run HCOV_RCHUNK=4
run HCOV_LIB=$K4 HCOV_RCHUNK=4
run HCOV_LIB=$K4 HCOV_RCHUNK=5
run HCOV_LIB=$K4 HCOV_RCHUNK=6
N=2097152
run HCOV_X=default
run HCOV_RCHUNK=4
run HCOV_LIB=$K4 HCOV_RCHUNK=5
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r3d_tests.log 2>&1
echo "exit $?" >> gpurun_out/r3d_tests.log
