mkdir -p gpurun_out
bash scripts/ab_env.sh FLERN_DBG_MODE "0 2" "c1x c4p" 2>&1 | tee gpurun_out/c1x_ab.txt
timeout 300 python bench.py --workload c1x --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 1 2>&1 | tail -1 > gpurun_out/c1x_line.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flern_query -s 4 -c 1 -o gpurun_out/prof_c1x -f \
  python bench.py --workload c1x --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c1x.log 2>&1
tail -2 gpurun_out/ncu_c1x.log
