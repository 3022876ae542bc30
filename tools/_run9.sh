export HCOV_WATCHDOG_S=200
python tools/prof_engine.py 32768 1.0 0.05 1e-6 20 > gpurun_out/r9_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_engine -s 1 -c 1 -o gpurun_out/prof_engine32k \
  python tools/prof_engine.py 32768 1.0 0.05 1e-6 20 > gpurun_out/r9_ncu.log 2>&1
echo "rc=$?"
