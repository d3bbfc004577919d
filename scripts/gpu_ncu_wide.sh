#!/bin/bash
# Full ncu capture (with source) of one wide-kernel launch (C3) and the training kernel; summaries made on
# the box (the reports themselves exceed gpurun's copy-back limit).
TAG=${1:-w3}
WL=${2:-"c3 train"}
mkdir -p gpurun_out
for w in $WL; do
  k=regex:flern_query; s=1; [ $w = train ] && k=regex:flern_train_kernel && s=2
  timeout 900 ncu --set full --clock-control none --import-source on -k $k -s $s -c 1 -o /tmp/prof_${w}_$TAG -f \
    python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_${w}_$TAG.log 2>&1
  python scripts/ncu_summary.py /tmp/prof_${w}_$TAG.ncu-rep > gpurun_out/ncusum_${w}_$TAG.md 2>&1
  ncu -i /tmp/prof_${w}_$TAG.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_${w}.csv 2>/dev/null
  python scripts/ncu_stalls.py /tmp/src_${w}.csv "" 60 > gpurun_out/stalls_${w}_$TAG.txt 2>&1
  ncu -i /tmp/prof_${w}_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_${w}_$TAG.csv 2>/dev/null
done
ls -la gpurun_out/
