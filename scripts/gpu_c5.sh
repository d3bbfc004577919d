#!/bin/bash
# C5 / a8 round trip: the new -m gpu tests, then the C5 bench line at N=1 (SF100 on one GPU)
TAG=${1:-c5}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -k "${2:-multirank or c5 or streamed or int32}" 2>&1 | tail -30 | tee gpurun_out/pytest_$TAG.log
timeout 1200 python bench.py --workload c5 --steps 20 --warmup 3 --e2e-steps 2 2> gpurun_out/bench_c5_$TAG.err | tail -1 | tee gpurun_out/bench_c5_$TAG.json

tail -5 gpurun_out/bench_c5_$TAG.err
