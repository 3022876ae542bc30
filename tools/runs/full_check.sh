# all GPU tests, then the 2M timeline (usage: bash tools/runs/full_check.sh TAG)
export HCOV_WATCHDOG_S=1200
TAG=${1:-f}
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > gpurun_out/$TAG.log
timeout 1500 python tools/timeline.py run tl2m_$TAG 2097152 0.5 0.1 1e-6 20 >> gpurun_out/$TAG.log 2>&1; echo "tl rc=$?" >> gpurun_out/$TAG.log
