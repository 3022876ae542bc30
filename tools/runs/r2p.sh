#!/bin/bash
# round-2 re-entry check: GPU suite, C5 as written (SPD-preserving order) at 2M, default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/r2p_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2p_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2p_pytest.log
HCOV_VERBOSE=1 timeout 900 python tools/diag_spd4.py 2097152 1 1e-5 20 20 > gpurun_out/r2p_c5spd.log 2>&1
echo "exit $?" >> gpurun_out/r2p_c5spd.log
timeout 1500 python bench.py --steps 2 --warmup 3 --out gpurun_out/r2p_bench.json > gpurun_out/r2p_bench.log 2>&1
echo "exit $?" >> gpurun_out/r2p_bench.log
