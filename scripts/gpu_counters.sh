#!/bin/bash
# Per-workload ncu counters (the gpu_round2.sh set) for the given workloads only.
# usage: scripts/gpu_counters.sh TAG "workloads..."
TAG=${1:-r02c}
WL=${2:-"c3 c4"}
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed
M=$M,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed
M=$M,sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
M=$M,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active
M=$M,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum
for w in $WL; do
  k="regex:flern_query"
  [ $w = train ] && k="regex:flern_train_kernel"
  timeout 900 ncu --metrics $M --clock-control none -k $k -s 2 -c 1 --csv --log-file gpurun_out/counters_${w}_$TAG.csv \
    python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
ls -la gpurun_out/
