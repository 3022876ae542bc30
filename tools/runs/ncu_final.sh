# ncu evidence for profiles/: launch list of the bench command at n=131072 and a full capture of
# the engine at n=65536 (each after the same command exited 0 without ncu)
export HCOV_WATCHDOG_S=900
TAG=${1:-r1}
python bench.py --n 131072 --no-cpu-baseline > gpurun_out/${TAG}_b131k.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_131k.csv python bench.py --n 131072 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch rc=$?" > gpurun_out/${TAG}_ncu.status
python tools/prof_engine.py 65536 0.5 0.1 1e-6 20 > gpurun_out/${TAG}_p65k.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_engine -s 1 -c 1 -o gpurun_out/${TAG}_engine65k python tools/prof_engine.py 65536 0.5 0.1 1e-6 20 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/${TAG}_ncu.status
