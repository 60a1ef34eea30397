# round 2, session 5: token mixer residency (TG_TOKMIX_MINB 3 vs 2) on C
set -x
O=gpurun_out/r02s5e
mkdir -p $O
for v in 2 3; do
  if [ $v = 3 ]; then export TG_LIB_PATH=$PWD/paper_2402_05396_b200/libtaser_b200_m3.so; fi
  timeout 900 python bench.py --workload C --steps 20 --warmup 5 --no-cpu --no-e2e > $O/bench_C_minb$v.json 2> $O/bench_C_minb$v.err; echo "C minb$v rc=$?"
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), (d.get('parity') or {}).get('mismatches'), (d.get('parity') or {}).get('q_max_rel_err'))" $O/bench_C_minb$v.json
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:token_mix -c 6 --csv --log-file $O/tok_minb$v.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1; echo "ncu rc=$?"
  python scripts/launch_agg.py $O/tok_minb$v.csv 3
done
