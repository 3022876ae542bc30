set -x
./tools/fp64_peak > gpurun_out/r2_fp64.log 2>&1; cat gpurun_out/r2_fp64.log
timeout 300 python bench.py --n 32768 --steps 2 --warmup 3 > gpurun_out/r2_bench32k.log 2>&1; echo "bench rc=$?"
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?"
