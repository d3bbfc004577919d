#!/bin/bash
# Focused check: selected parity tests, then selected bench lines.
# usage: scripts/gpu_wide.sh TAG "pytest -k expr" "workloads..."
TAG=${1:-w}
K=${2:-"wide or every_kernel_shape or two_probe"}
WL=${3:-"c3 c4"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv,noheader | tee gpurun_out/box_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 -k "$K" 2>&1 | tail -30 | tee gpurun_out/pytest_$TAG.log
for w in $WL; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -2 | tee gpurun_out/bench_${w}_$TAG.json
done
