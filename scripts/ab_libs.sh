# A/B of alternate libflern builds: bench c2 + c4p + no-model for each
cp paper_2311_02781_b200/lib/libflern.so /tmp/libflern_main.so
for v in main tools/libflern_nopf tools/libflern_pf1 tools/libflern_pf4; do
  if [ $v = main ]; then cp /tmp/libflern_main.so paper_2311_02781_b200/lib/libflern.so; else cp $v.so paper_2311_02781_b200/lib/libflern.so; fi
  for w in c2 c4p; do
    echo "$v $w $(python bench.py --workload $w --no-cpu-baseline --e2e-steps 1 --steps 30 --warmup 5 2>&1 | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]/1e9,3), j["ms_per_step"])')"
  done
  echo "$v nomodel $(python bench.py --workload c2 --no-model --no-cpu-baseline --e2e-steps 1 --steps 30 --warmup 5 2>&1 | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]/1e9,3))')"
done
cp /tmp/libflern_main.so paper_2311_02781_b200/lib/libflern.so
