#!/bin/bash
# C5 as written (SPD-preserving order) bench line at n = 131,072; engine timeline at 524K; replicate
# MLE study (time-boxed); C4 MLE continuation
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=900
timeout 900 python bench.py --theta config --n 131072 --factor-trunc --kcap 40 --steps 2 --warmup 3 \
  --out gpurun_out/r2v_bench_c5spd131k.json > gpurun_out/r2v_bench_c5spd131k.log 2>&1
echo "exit $?" >> gpurun_out/r2v_bench_c5spd131k.log
timeout 600 python tools/timeline.py run r2v_tl524k 524288 0.5 0.1 1e-6 20 > gpurun_out/r2v_tl524k.log 2>&1
echo "rc=$?" >> gpurun_out/r2v_tl524k.log
timeout 1500 python tools/replicates.py --sizes 2000,4000,8000 --reps 6 --budget-s 1200 > gpurun_out/r2v_rep.log 2>&1
echo "rep exit $?" >> gpurun_out/r2v_rep.log
timeout 1000 python tools/mle_run.py --iters-now 2 > gpurun_out/r2v_mle.log 2>&1
echo "mle exit $?" >> gpurun_out/r2v_mle.log
timeout 600 python -m pytest tests/test_gpu_3d.py tests/test_gpu_ldl.py tests/test_gpu_mle.py -q -s > gpurun_out/r2v_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2v_tests.log
