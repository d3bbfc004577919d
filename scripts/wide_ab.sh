#!/bin/bash
# Wide-kernel A/B on the diagnostic build: wait accounting for FLERN_DBG_MODE = 0 (full), 1 (no epilogue work),
# 2 (no operand loads), 3 (neither).  usage: scripts/wide_ab.sh [workload] [sf]
W=${1:-c3}; SF=${2:-1}
mkdir -p gpurun_out
for m in 0 1 2 3; do
  echo "== FLERN_DBG_MODE=$m"
  FLERN_DBG_MODE=$m FLERN_LIB=libflern_diag.so timeout 600 python scripts/trace_wide.py $W $SF 2>&1 | head -16
done
