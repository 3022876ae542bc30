#!/bin/bash
# GPU tests (3-D, LDL, MLE parity); one-CTA gang threshold probes at 524K; C5-as-written SPD probe
# at 524K; single-pass ncu DRAM traffic of k_engine at 2M; C4 MLE continuation
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=900
timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_ldl.py tests/test_gpu_mle.py -q -s > gpurun_out/r2s_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2s_tests.log
for g in 0 1024 2048 4096 16384; do
  HCOV_GANG1_BELOW=$g timeout 300 python tools/perf_probe.py 524288 0.5 0.1 1e-6 20 2 >> gpurun_out/r2s_probe.log 2>&1
  echo "g1=$g exit $?" >> gpurun_out/r2s_probe.log
done
HCOV_VERBOSE=1 timeout 600 python tools/diag_spd4.py 524288 1 1e-5 20 48 > gpurun_out/r2s_c5spd524k.log 2>&1
echo "exit $?" >> gpurun_out/r2s_c5spd524k.log
python tools/prof_engine.py 2097152 0.5 0.1 1e-6 20 > gpurun_out/r2s_p2m.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_engine -s 1 -c 1 --csv --log-file gpurun_out/r2s_dram2m.csv python tools/prof_engine.py 2097152 0.5 0.1 1e-6 20 > gpurun_out/r2s_ncu_dram2m.log 2>&1
echo "dram2m rc=$?" >> gpurun_out/r2s_ncu.status
timeout 1000 python tools/mle_run.py --iters-now 2 > gpurun_out/r2s_mle.log 2>&1
echo "mle exit $?" >> gpurun_out/r2s_mle.log
