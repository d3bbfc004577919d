#!/bin/bash
# compute-sanitizer over one small run of every kernel family (scripts/sanitize_run.py) and the small
# join / training GPU tests: memcheck (out-of-bounds / misaligned global and shared accesses) and synccheck.
# usage: scripts/gpu_sanitize.sh TAG
T=${1:-san}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitize_memcheck_$T.log 2>&1; echo "exit $?" >> gpurun_out/sanitize_memcheck_$T.log
timeout 1500 $CS --tool synccheck --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitize_synccheck_$T.log 2>&1; echo "exit $?" >> gpurun_out/sanitize_synccheck_$T.log
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_joins.py tests/test_gpu_train.py -m gpu -q -x -k "not trajectory" > gpurun_out/sanitize_memcheck_tests_$T.log 2>&1; echo "exit $?" >> gpurun_out/sanitize_memcheck_tests_$T.log
