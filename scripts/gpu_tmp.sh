mkdir -p gpurun_out
T=${1:-x32}
python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_$T.log
for w in c2 c5 c1x c2s c4p; do timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 30 --warmup 5 --e2e-steps 1 2>&1 | tail -1 > gpurun_out/bench_${w}_$T.json; done
