#!/bin/bash
# A/B of the fused-reduction panel QR (libhcov_qr.so) against the default library at 524K, and the
# truncation / parity / accuracy suites on the variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=900
O=gpurun_out/r3f_sweep.jsonl
: > $O
QR=$GRAFT_REPO_ROOT/paper_1709_08625_b200/libhcov_qr.so
run() { echo "== $*" >> $O; env "$@" timeout 600 python tools/perf_probe.py 524288 0.5 0.1 1e-6 20 1 >> $O 2>>gpurun_out/r3f_err.log; }
run HCOV_X=default
run HCOV_LIB=$QR
HCOV_LIB=$QR timeout 1500 python -m pytest tests/test_gpu_truncate.py tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_accuracy.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r3f_tests.log 2>&1
echo "exit $?" >> gpurun_out/r3f_tests.log
