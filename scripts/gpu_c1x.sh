#!/bin/bash
# C1x iteration: the -m gpu suite (optionally -k EXPR), then c1x / c1 / c2 bench lines.
# usage: scripts/gpu_c1x.sh TAG [pytest -k expr]
TAG=${1:-x}
mkdir -p gpurun_out
if [ -n "$2" ]; then KARG=(-k "$2"); else KARG=(); fi
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 "${KARG[@]}" 2>&1 | tail -15 | tee gpurun_out/pytest_$TAG.log
for w in c1x c1 c2; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 20 --warmup 3 --e2e-steps 1 2>&1 | tail -1 | tee gpurun_out/bench_${w}_$TAG.json
done
timeout 600 python bench.py --workload c1x --no-model --no-cpu-baseline --steps 20 --e2e-steps 1 2>&1 | tail -1 | tee gpurun_out/bench_c1xnm_$TAG.json
