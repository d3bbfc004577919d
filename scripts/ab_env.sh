#!/bin/bash
# A/B a tuning environment variable over workloads: scripts/ab_env.sh VAR "v1 v2 ..." "c2 c1x ..." [extra bench args]
# The knobs are read only by the diagnostic build (make paper_2311_02781_b200/lib/libflern_diag.so).
export FLERN_LIB=libflern_diag.so
VAR=$1; VALS=$2; WLS=$3; shift 3
for v in $VALS; do
  for w in $WLS; do
    extra=""
    if [ "$w" = "c2nm" ]; then w=c2; extra="--no-model"; fi
    r=$(env $VAR=$v timeout 600 python bench.py --workload $w $extra --no-cpu-baseline --e2e-steps 1 --steps 30 --warmup 5 "$@" 2>&1 | tail -1)
    echo "$VAR=$v $w$extra $(echo "$r" | python -c 'import json,sys
try:
  j=json.loads(sys.stdin.read()); print("%.3fe9 rows/s  %.4f ms  frac %.3f  clk %s %s" % (j["value"]/1e9, j["ms_per_step"], j["roofline"]["frac"], j["clocks"]["sm_mhz"], j["clocks"]["reasons"]))
except Exception as e: print("ERR", e)')"
  done
done
