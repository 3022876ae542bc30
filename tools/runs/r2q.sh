#!/bin/bash
# device tree tests; C4 MLE (first 2 iterations, checkpointed); ncu launch list (524K bench) +
# full capture of k_engine at 524K (traffic)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=900
timeout 900 python -m pytest tests/test_gpu_tree.py -x -q -s > gpurun_out/r2q_tree.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2q_tree.log
timeout 1500 python tools/mle_run.py --iters-now 2 > gpurun_out/r2q_mle.log 2>&1
echo "mle exit $?" >> gpurun_out/r2q_mle.log
python bench.py --n 524288 --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/r2q_b524k.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2q_launches_524k.csv python bench.py --n 524288 --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/r2q_ncu_launch.log 2>&1
echo "launch rc=$?" > gpurun_out/r2q_ncu.status
python tools/prof_engine.py 524288 0.5 0.1 1e-6 20 > gpurun_out/r2q_p524k.log 2>&1 && \
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:k_engine -s 1 -c 1 -o gpurun_out/r2q_engine524k python tools/prof_engine.py 524288 0.5 0.1 1e-6 20 > gpurun_out/r2q_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/r2q_ncu.status
