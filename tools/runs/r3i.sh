#!/bin/bash
# final library of the round: full GPU suite, smoke, the default bench line (2M), ncu launch list of
# the bench command at 524K
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=1800
export HCOV_C2_REPORT=gpurun_out/r3i_c2
echo "== gather register rows + aca_full index math" > gpurun_out/r3i_sweep.jsonl
timeout 600 python tools/perf_probe.py 524288 0.5 0.1 1e-6 20 1 >> gpurun_out/r3i_sweep.jsonl 2>>gpurun_out/r3i_err.log
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=15 -p no:cacheprovider > gpurun_out/r3i_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3i_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3i_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/r3i_smoke.log
timeout 1800 python bench.py > gpurun_out/r3i_bench.json 2> gpurun_out/r3i_bench.err
echo "bench exit $?" >> gpurun_out/r3i_bench.err
timeout 600 python bench.py --n 524288 --no-cpu-baseline > gpurun_out/r3i_b524k.json 2> gpurun_out/r3i_b524k.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3i_launches_524k.csv python bench.py --n 524288 --no-cpu-baseline > gpurun_out/r3i_ncu_launch.log 2>&1
echo "launch rc=$?" > gpurun_out/r3i_ncu.status
