python -c "
import torch
p=torch.cuda.get_device_properties(0)
print('persistingL2CacheMaxSize', p.persisting_l2_cache_max_size if hasattr(p,'persisting_l2_cache_max_size') else 'n/a', 'L2', p.L2_cache_size)
"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "wide or two_probe or c1_full or c2_mlp" 2>&1 | tail -2
bash scripts/ab_env.sh FLERN_WINDOW_HT "0" "c3 c4"
FLERN_WINDOW_HT=1 bash scripts/ab_env.sh FLERN_DBG_MODE "0" "c3"
bash scripts/ab_env.sh FLERN_DBG_MODE "0" "c2"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:flern_query_wide -s 4 -c 1 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | grep -E "dram__|gpu__time|lts__t" 
