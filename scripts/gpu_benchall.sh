#!/bin/bash
# Every bench workload once (20 steps) after the -m gpu suite: a quick round checkpoint.
# usage: scripts/gpu_benchall.sh TAG [skip_tests]
TAG=${1:-ck}
mkdir -p gpurun_out
if [ -z "$2" ]; then
  timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 2>&1 | tail -5 > gpurun_out/pytest_$TAG.log
fi
for w in c2 c1 c1x c2s c4p c3 c4 c5 train; do
  timeout 1200 python bench.py --workload $w --no-cpu-baseline --steps 20 --warmup 3 --e2e-steps 1 2>&1 | tail -1 > gpurun_out/bench_${w}_$TAG.json
done
