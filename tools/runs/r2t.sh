#!/bin/bash
# GPU tests (3-D at eps 1e-6, LDL, MLE parity); gang-shape probes at 524K (after the local flop
# counter change); k_engine DRAM traffic at 2M (bench workload, single-pass ncu); C4 MLE continuation
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=900
timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_ldl.py tests/test_gpu_mle.py -q -s > gpurun_out/r2t_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2t_tests.log
for v in base rows128 rapp8 max8 all8; do
  case $v in
    base) E="X=0";; rows128) E="HCOV_GANG_ROWS=128";; rapp8) E="HCOV_RAPP512=8";; max8) E="HCOV_GANG_MAX_SMALL=8";;
    all8) E="HCOV_GANG_ROWS=128 HCOV_RAPP512=8 HCOV_GANG_MAX_SMALL=8";;
  esac
  env $E timeout 300 python tools/perf_probe.py 524288 0.5 0.1 1e-6 20 2 >> gpurun_out/r2t_probe.log 2>&1
  echo "$v exit $?" >> gpurun_out/r2t_probe.log
done
timeout 1000 python tools/mle_run.py --iters-now 2 > gpurun_out/r2t_mle.log 2>&1
echo "mle exit $?" >> gpurun_out/r2t_mle.log
timeout 400 python tools/dram_probe.py > gpurun_out/r2t_dram_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_engine -s 3 -c 1 --csv --log-file gpurun_out/r2t_dram2m.csv python tools/dram_probe.py > gpurun_out/r2t_ncu_dram2m.log 2>&1
echo "dram2m rc=$?" >> gpurun_out/r2t_ncu.status
