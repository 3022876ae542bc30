#!/bin/bash
# round 2, call A: GPU tests + first 2M bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > gpurun_out/r2a_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2a_pytest.log
timeout 1500 python bench.py --steps 2 --warmup 3 --out gpurun_out/r2a_bench.json > gpurun_out/r2a_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/r2a_bench.log
