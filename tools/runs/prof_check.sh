# GPU tests, 524K timeline, then a full ncu capture of the 65K engine (usage: bash tools/runs/prof_check.sh TAG)
export HCOV_WATCHDOG_S=600
TAG=${1:-chk}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/$TAG.log
timeout 900 python tools/timeline.py run tl_$TAG 524288 0.5 0.1 1e-6 20 >> gpurun_out/$TAG.log 2>&1; echo "tl rc=$?" >> gpurun_out/$TAG.log
timeout 300 python tools/prof_engine.py 65536 0.5 0.1 1e-6 20 > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_engine -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/prof_engine.py 65536 0.5 0.1 1e-6 20 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/$TAG.log
