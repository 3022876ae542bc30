# truncation tests + microbench, all GPU tests, 524K timeline (usage: bash tools/runs/qr_check.sh TAG)
export HCOV_WATCHDOG_S=600
TAG=${1:-q}
timeout 600 python -m pytest tests/test_gpu_truncate.py -q -x 2>&1 | tail -3 > gpurun_out/$TAG.log
for mr in "256 92" "184 92" "128 60" "64 40"; do timeout 120 python tools/bench_trunc.py $mr 20 >> gpurun_out/$TAG.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 >> gpurun_out/$TAG.log
timeout 900 python tools/timeline.py run tl_$TAG 524288 0.5 0.1 1e-6 20 >> gpurun_out/$TAG.log 2>&1; echo "tl rc=$?" >> gpurun_out/$TAG.log
