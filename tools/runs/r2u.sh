#!/bin/bash
# full GPU suite (engine allocated before the pools); 2M eval without a prior factor (the case that
# ran out of memory) + single-pass ncu DRAM traffic at 2M; C4 MLE continuation
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=900
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2u_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2u_pytest.log
timeout 400 python tools/dram_probe.py > gpurun_out/r2u_dram_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_engine -s 3 -c 1 --csv --log-file gpurun_out/r2u_dram2m.csv python tools/dram_probe.py > gpurun_out/r2u_ncu_dram2m.log 2>&1
echo "dram2m rc=$?" >> gpurun_out/r2u_ncu.status
timeout 300 python tools/prof_engine.py 2097152 0.5 0.1 1e-6 20 > gpurun_out/r2u_p2m.log 2>&1
echo "p2m exit $?" >> gpurun_out/r2u_p2m.log
timeout 1700 python tools/mle_run.py --iters-now 4 > gpurun_out/r2u_mle.log 2>&1
echo "mle exit $?" >> gpurun_out/r2u_mle.log
