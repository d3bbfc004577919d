timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -3 > gpurun_out/pytest_ab1.log
bash scripts/ab_env.sh FLERN_SPIN_NS "0 32 64 128 256" "c1x c2 c4p c3" > gpurun_out/ab_spin.txt 2>&1
