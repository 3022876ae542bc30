# GPU check: parity tests then a 524K engine timeline (usage: bash tools/runs/gpu_check.sh TAG)
export HCOV_WATCHDOG_S=600
TAG=${1:-chk}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/$TAG.log
timeout 900 python tools/timeline.py run tl_$TAG 524288 0.5 0.1 1e-6 20 >> gpurun_out/$TAG.log 2>&1; echo "tl rc=$?" >> gpurun_out/$TAG.log
