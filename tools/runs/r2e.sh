#!/bin/bash
# round 2, call E: side-split RAPP gangs; batch bench; diagnostics tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity.py tests/test_gpu_solve.py tests/test_gpu_diagnostics.py -m gpu -q -rA -s -p no:cacheprovider --deselect tests/test_gpu_parity.py::test_near_full_rank_mode > gpurun_out/r2e_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2e_pytest.log
timeout 600 python tools/timeline.py run tl_c4_r2e 524288 0.5 0.1 1e-6 20 > gpurun_out/r2e_tl.log 2>&1
echo "tl exit $?" >> gpurun_out/r2e_tl.log
timeout 900 python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline --acc-cols 0 --out gpurun_out/r2e_bench_c4.json > gpurun_out/r2e_bench_c4.log 2>&1
echo "bench exit $?" >> gpurun_out/r2e_bench_c4.log
timeout 1200 python bench.py --config C4 --cands-per-rank 8 --steps 1 --warmup 3 --no-cpu-baseline --acc-cols 0 --out gpurun_out/r2e_bench_c4b8.json > gpurun_out/r2e_bench_c4b8.log 2>&1
echo "bench exit $?" >> gpurun_out/r2e_bench_c4b8.log
