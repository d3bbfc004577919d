#!/bin/bash
# One GPU round trip: parity tests, bench, launch list and a full ncu capture of the query kernel.
# usage: scripts/gpu_check.sh [tag] [pytest -k expr]
TAG=${1:-run}
K=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -n "$K" ]; then KARG=(-k "$K"); else KARG=(); fi
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 "${KARG[@]}" 2>&1 | tail -25 | tee gpurun_out/pytest_$TAG.log
timeout 600 python bench.py 2>&1 | tail -3 | tee gpurun_out/bench_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flern_query -s 6 -c 1 -o gpurun_out/prof_$TAG -f \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
