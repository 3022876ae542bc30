# 2M timeline at the bench kernel (nu=0.5, ell=0.1, eps=1e-6, k=20)
export HCOV_WATCHDOG_S=1800
TAG=${1:-tl2m}
timeout 1500 python tools/timeline.py run $TAG 2097152 0.5 0.1 1e-6 20 > gpurun_out/$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/$TAG.log
