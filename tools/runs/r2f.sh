#!/bin/bash
# round 2, call F (after container re-creation): smoke, full GPU suite, default 2M bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/r2f_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/r2f_smoke.log
timeout 2700 python -m pytest tests -m gpu -q -rA -p no:cacheprovider --durations=40 > gpurun_out/r2f_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2f_pytest.log
timeout 1500 python bench.py --steps 1 --warmup 3 --out gpurun_out/r2f_bench.json > gpurun_out/r2f_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/r2f_bench.log
