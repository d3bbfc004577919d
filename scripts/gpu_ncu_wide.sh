#!/bin/bash
# Full ncu capture (with source) of one wide-kernel launch (C3) and the training kernel; summaries on the box.
TAG=${1:-w3}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flern_query_wide -s 1 -c 1 -o gpurun_out/prof_c3_$TAG -f \
  python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c3_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flern_train_kernel -s 2 -c 1 -o gpurun_out/prof_train_$TAG -f \
  python bench.py --workload train --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_train_$TAG.log 2>&1
for w in c3 train; do
  [ -f gpurun_out/prof_${w}_$TAG.ncu-rep ] && python scripts/ncu_summary.py gpurun_out/prof_${w}_$TAG.ncu-rep > gpurun_out/ncusum_${w}_$TAG.md
  ncu -i gpurun_out/prof_${w}_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_${w}_$TAG.csv 2>/dev/null
  ncu -i gpurun_out/prof_${w}_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_${w}_$TAG.csv 2>/dev/null
done
ls -la gpurun_out/
