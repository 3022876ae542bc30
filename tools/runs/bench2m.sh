# default bench line (C5, 2M) (usage: bash tools/runs/bench2m.sh TAG)
export HCOV_WATCHDOG_S=1800
TAG=${1:-b}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "rc=$?" >> gpurun_out/bench_$TAG.err
