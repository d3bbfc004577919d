#!/bin/bash
# Quick GPU round trip: box facts, the -m gpu suite (optionally -k EXPR), one C2 bench line.
# usage: scripts/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}
K=${2:-}
mkdir -p gpurun_out
{ nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,memory.total --format=csv,noheader; nproc; free -g | head -2; } | tee gpurun_out/box_$TAG.txt
if [ -n "$K" ]; then KARG=(-k "$K"); else KARG=(); fi
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 "${KARG[@]}" 2>&1 | tail -30 | tee gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -2 | tee gpurun_out/bench_c2_$TAG.json
