#!/bin/bash
# new GPU tests (3-D, LDL, MLE parity); NT / chunk probes at 524K; single-pass ncu dram traffic of
# k_engine at 524K and 2M; full ncu capture at 65K; C4 MLE continuation
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=900
timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_ldl.py tests/test_gpu_mle.py -x -q -s > gpurun_out/r2r_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2r_tests.log
for v in base nt384 rc2 rc6; do
  case $v in
    base) E="";; nt384) E="HCOV_LIB=$PWD/paper_1709_08625_b200/libhcov_nt384.so";; rc2) E="HCOV_RCHUNK=2";; rc6) E="HCOV_RCHUNK=6";;
  esac
  env $E timeout 300 python tools/perf_probe.py 524288 0.5 0.1 1e-6 20 2 >> gpurun_out/r2r_probe.log 2>&1
  echo "$v exit $?" >> gpurun_out/r2r_probe.log
done
python tools/prof_engine.py 524288 0.5 0.1 1e-6 20 > gpurun_out/r2r_p524k.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_engine -s 1 -c 1 --csv --log-file gpurun_out/r2r_dram524k.csv python tools/prof_engine.py 524288 0.5 0.1 1e-6 20 > gpurun_out/r2r_ncu_dram524k.log 2>&1
echo "dram524k rc=$?" >> gpurun_out/r2r_ncu.status
python tools/prof_engine.py 65536 0.5 0.1 1e-6 20 > gpurun_out/r2r_p65k.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_engine -s 1 -c 1 -o gpurun_out/r2r_engine65k python tools/prof_engine.py 65536 0.5 0.1 1e-6 20 > gpurun_out/r2r_ncu_full.log 2>&1
echo "full65k rc=$?" >> gpurun_out/r2r_ncu.status
timeout 1200 python tools/mle_run.py --iters-now 2 > gpurun_out/r2r_mle.log 2>&1
echo "mle exit $?" >> gpurun_out/r2r_mle.log
