#!/bin/bash
# round-2 final evidence on the final library (the 2M bench line is r3e's): full GPU suite, ncu launch
# list of the bench command at 524K, full ncu capture of k_engine at 65K, DRAM traffic at 2M
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export HCOV_WATCHDOG_S=1800
export HCOV_C2_REPORT=gpurun_out/r3g_c2
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=15 -p no:cacheprovider > gpurun_out/r3g_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3g_pytest.log
timeout 600 python bench.py --n 524288 --no-cpu-baseline > gpurun_out/r3g_b524k.json 2> gpurun_out/r3g_b524k.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3g_launches_524k.csv python bench.py --n 524288 --no-cpu-baseline > gpurun_out/r3g_ncu_launch.log 2>&1
echo "launch rc=$?" > gpurun_out/r3g_ncu.status
timeout 300 python tools/prof_engine.py 65536 0.5 0.1 1e-6 20 > gpurun_out/r3g_p65k.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_engine -s 1 -c 1 -f -o gpurun_out/r3g_engine65k python tools/prof_engine.py 65536 0.5 0.1 1e-6 20 > gpurun_out/r3g_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/r3g_ncu.status
timeout 500 python tools/dram_probe.py > gpurun_out/r3g_dram_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_engine -s 3 -c 1 --csv --log-file gpurun_out/r3g_dram2m.csv python tools/dram_probe.py > gpurun_out/r3g_ncu_dram2m.log 2>&1
echo "dram2m rc=$?" >> gpurun_out/r3g_ncu.status
