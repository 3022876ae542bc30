set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/gpu_debug.py > gpurun_out/r1_debug.log 2>&1; echo "debug rc=$?"
timeout 120 python tools/probe.py 16384 1.5 0.05 1e-8 0 2 > gpurun_out/r1_p16k.log 2>&1; echo "p16k rc=$?"
timeout 300 python tools/probe.py 131072 0.5 0.0864 1e-6 16 2 > gpurun_out/r1_p131k.log 2>&1; echo "p131k rc=$?"
timeout 600 python tools/probe.py 524288 0.5 0.1 1e-6 20 1 > gpurun_out/r1_p524k.log 2>&1; echo "p524k rc=$?"
