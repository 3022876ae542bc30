#!/bin/bash
# round 2, re-entry call A: full GPU suite + 2M bench line + 524K timeline on HEAD
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=1800
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=15 -p no:cacheprovider > gpurun_out/r3a_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3a_pytest.log
timeout 900 python tools/timeline.py run tl_r3a 524288 0.5 0.1 1e-6 20 > gpurun_out/r3a_tl.log 2>&1; echo "tl rc=$?" >> gpurun_out/r3a_tl.log
timeout 1800 python bench.py > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err
echo "bench exit $?" >> gpurun_out/r3a_bench.err
