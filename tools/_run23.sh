export HCOV_WATCHDOG_S=1800
python bench.py > gpurun_out/bench_r1.log 2>gpurun_out/bench_r1.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_r1.csv python bench.py --no-cpu-baseline > gpurun_out/ncu_bench_r1.log 2>&1
echo "rc=$?"
