#!/bin/bash
# Round-2 evidence on one fresh B200: the -m gpu suite, a bench line per workload, the C2 launch list,
# per-workload ncu counters (duration, DRAM bytes, tensor-pipe activity, bf16 tensor ops, issue, occupancy)
# and full captures (with source, for the role split) of C2 and C1x.
# usage: scripts/gpu_round2.sh TAG [skip_tests]
TAG=${1:-r02}
mkdir -p gpurun_out
{ nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,memory.total --format=csv,noheader; nproc; } | tee gpurun_out/box_$TAG.txt
if [ -z "$2" ]; then
  timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 2>&1 | tail -15 | tee gpurun_out/pytest_$TAG.log
fi
timeout 900 python bench.py 2>&1 | tail -1 | tee gpurun_out/bench_c2_$TAG.json
for w in c1 c1x c2s c4p c3 c4 c5 train; do
  timeout 1200 python bench.py --workload $w --no-cpu-baseline --steps 20 --warmup 3 --e2e-steps 2 2>&1 | tail -1 > gpurun_out/bench_${w}_$TAG.json
done
timeout 600 python bench.py --workload c2 --no-model --no-cpu-baseline --steps 50 --e2e-steps 1 2>&1 | tail -1 > gpurun_out/bench_c2nomodel_$TAG.json
timeout 600 python bench.py --workload c1x --no-model --no-cpu-baseline --steps 20 --e2e-steps 1 2>&1 | tail -1 > gpurun_out/bench_c1xnomodel_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2_$TAG.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed
M=$M,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed
M=$M,sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
M=$M,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active
M=$M,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum
for w in c2 c1x c2s c4p c3 c4 c5 c1 train c2nm c1xnm; do
  ww=$w; extra=""; k="regex:flern_query"
  [ $w = c2nm ] && ww=c2 && extra="--no-model"
  [ $w = c1xnm ] && ww=c1x && extra="--no-model"
  [ $w = train ] && k="regex:flern_train_kernel"
  timeout 900 ncu --metrics $M --clock-control none -k $k -s 2 -c 1 --csv --log-file gpurun_out/counters_${w}_$TAG.csv \
    python bench.py --workload $ww $extra --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flern_query -s 6 -c 1 -o /tmp/prof_c2_$TAG -f \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c2_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flern_query -s 4 -c 1 -o /tmp/prof_c1x_$TAG -f \
  python bench.py --workload c1x --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c1x_$TAG.log 2>&1
for w in c2 c1x; do
  [ -f /tmp/prof_${w}_$TAG.ncu-rep ] && python scripts/ncu_summary.py /tmp/prof_${w}_$TAG.ncu-rep > gpurun_out/ncusum_${w}_$TAG.md
  ncu -i /tmp/prof_${w}_$TAG.ncu-rep --page source --csv --print-source cuda,sass > /tmp/_src_$w.csv 2>/dev/null
  python scripts/ncu_roles.py /tmp/_src_$w.csv 3 > gpurun_out/roles_${w}_$TAG.txt
done
rm -f gpurun_out/prof_c1x_$TAG.ncu-rep
