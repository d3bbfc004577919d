#!/bin/bash
# The whole -m gpu suite, then the given bench workloads (20 steps each).
# usage: scripts/gpu_full.sh TAG "workloads..."
TAG=${1:-f}
WL=${2:-"c2 c3 c4 train"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv,noheader | tee gpurun_out/box_$TAG.txt
timeout 2700 python -m pytest tests -m gpu -q --timeout 1500 2>&1 | tail -15 | tee gpurun_out/pytest_$TAG.log
for w in $WL; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1 > gpurun_out/bench_${w}_$TAG.json
done
