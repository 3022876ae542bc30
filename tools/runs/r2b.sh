#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solve.py tests/test_gpu_accuracy.py tests/test_gpu_parity.py -m gpu -q -rA -s -p no:cacheprovider -k "solve or pcg or matvec or transpose or interm or c1 or smoke or dense" > gpurun_out/r2b_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2b_pytest.log
timeout 900 python tools/diag_r2.py nfr c3 gen2m > gpurun_out/r2b_diag.log 2>&1
echo "diag exit $?" >> gpurun_out/r2b_diag.log
nproc >> gpurun_out/r2b_diag.log
timeout 1500 python bench.py --steps 2 --warmup 3 --out gpurun_out/r2b_bench.json > gpurun_out/r2b_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/r2b_bench.log
