#!/bin/bash
# One GPU round trip: parity tests, bench lines for every workload, launch list and a full ncu
# capture of the query kernel (C2). usage: scripts/gpu_round.sh TAG [skip_tests]
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv,noheader | tee gpurun_out/smi_$TAG.txt
nproc >> gpurun_out/smi_$TAG.txt
if [ -z "$2" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -30 | tee gpurun_out/pytest_$TAG.log
fi
timeout 600 python bench.py 2>&1 | tail -2 | tee gpurun_out/bench_c2_$TAG.json
for w in c1 c1x c4p c3 c4; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline --steps 20 --warmup 3 --e2e-steps 2 2>&1 | tail -2 | tee gpurun_out/bench_${w}_$TAG.json
done
timeout 600 python bench.py --workload c2 --no-model --no-cpu-baseline --steps 50 --e2e-steps 1 2>&1 | tail -1 | tee gpurun_out/bench_c2nomodel_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2_$TAG.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flern_query -s 6 -c 1 -o gpurun_out/prof_c2_$TAG -f \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c2_$TAG.log 2>&1
tail -2 gpurun_out/ncu_c2_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flern_query_wide -s 4 -c 1 -o gpurun_out/prof_c3_$TAG -f \
  python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c3_$TAG.log 2>&1
tail -2 gpurun_out/ncu_c3_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flern_query -s 4 -c 1 -o gpurun_out/prof_c1x_$TAG -f \
  python bench.py --workload c1x --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c1x_$TAG.log 2>&1
tail -2 gpurun_out/ncu_c1x_$TAG.log
# the reports (~27 MB each) exceed gpurun's 64 MiB copy-back together: extract what profile_summary.py
# reads into text on the box, keep the C2 report only
for w in c2 c3 c1x; do
  [ -f gpurun_out/prof_${w}_$TAG.ncu-rep ] && python scripts/ncu_summary.py gpurun_out/prof_${w}_$TAG.ncu-rep > gpurun_out/ncusum_${w}_$TAG.md
done
ncu -i gpurun_out/prof_c3_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_c3_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_c2_$TAG.ncu-rep --page source --csv --print-source cuda,sass > /tmp/_src.csv 2>/dev/null
python scripts/ncu_roles.py /tmp/_src.csv 3 > gpurun_out/roles_c2_$TAG.txt
rm -f gpurun_out/prof_c3_$TAG.ncu-rep gpurun_out/prof_c1x_$TAG.ncu-rep
