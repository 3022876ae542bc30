# engine timeline only (usage: bash tools/runs/tl.sh TAG n)
export HCOV_WATCHDOG_S=1200
TAG=${1:-tl}; N=${2:-524288}
timeout 1500 python tools/timeline.py run $TAG $N 0.5 0.1 1e-6 20 > gpurun_out/$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/$TAG.log
