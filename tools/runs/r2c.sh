#!/bin/bash
# round 2, call C: GPU tests, accuracy diagnostics, 2M bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2c_smi.txt 2>&1
timeout 900 python tools/diag_r2c.py nfr c3 gen2m > gpurun_out/r2c_diag.log 2>&1
echo "diag exit $?" >> gpurun_out/r2c_diag.log
timeout 2700 python -m pytest tests -m gpu -q -rA -p no:cacheprovider --deselect tests/test_gpu_parity.py::test_near_full_rank_mode > gpurun_out/r2c_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2c_pytest.log
timeout 1500 python bench.py --steps 2 --warmup 3 --out gpurun_out/r2c_bench.json > gpurun_out/r2c_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/r2c_bench.log
