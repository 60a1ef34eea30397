# round 2, session 5: token MLP layer 1 on tcgen05 (TG_K7_TOKMIX_TC=1) -- parity tests, C bench vs default, ncu
set -x
O=gpurun_out/r02s5f
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "token_mixer_variants or scoring_f32" > $O/pytest_tok.txt 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest_tok.txt
for v in default TC; do
  if [ $v = TC ]; then export TG_K7_TOKMIX_TC=1; fi
  timeout 600 python bench.py --workload C --steps 20 --warmup 5 --no-cpu --no-e2e > $O/bench_C_$v.json 2> $O/bench_C_$v.err; echo "C $v rc=$?"; tail -3 $O/bench_C_$v.err
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), (d.get('parity') or {}).get('mismatches'), (d.get('parity') or {}).get('q_max_rel_err'))" $O/bench_C_$v.json
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:token_mix -c 6 --csv --log-file $O/tok_$v.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1; echo "ncu rc=$?"
  python scripts/launch_agg.py $O/tok_$v.csv 3
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:token_mix_tc -s 2 -c 1 -o $O/ncu_toktc python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > $O/ncu.log 2>&1; echo "ncu full rc=$?"
ncu -i $O/ncu_toktc.ncu-rep --page raw --csv > $O/toktc_raw.csv 2>/dev/null
ncu -i $O/ncu_toktc.ncu-rep --page source --csv --print-source sass > $O/toktc_sass.csv 2>/dev/null
