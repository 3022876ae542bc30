#!/bin/bash
# final check of the round: full GPU suite + the default bench line (2M)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=1800
export HCOV_C2_REPORT=gpurun_out/r3e_c2
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=15 -p no:cacheprovider > gpurun_out/r3e_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3e_pytest.log
timeout 1800 python bench.py > gpurun_out/r3e_bench.json 2> gpurun_out/r3e_bench.err
echo "bench exit $?" >> gpurun_out/r3e_bench.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3e_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/r3e_smoke.log
