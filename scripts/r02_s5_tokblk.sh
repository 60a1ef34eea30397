# round 2, session 5: channel-block token mixer (default) -- scoring / adaptive GPU tests,
# C bench (new default vs the CTA kernel), C launch list, A step-group sweep
set -x
O=gpurun_out/r02s5c
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -k "scoring or adaptive or token or sampler or aggregator" > $O/pytest_sub.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_sub.txt
for v in default CTA; do
  if [ $v = CTA ]; then export TG_K7_TOKMIX_CTA=1; fi
  timeout 900 python bench.py --workload C --steps 20 --warmup 5 --no-cpu > $O/bench_C_$v.json 2> $O/bench_C_$v.err; echo "C $v rc=$?"
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), (d.get('parity') or {}).get('mismatches'), (d.get('parity') or {}).get('q_max_rel_err'))" $O/bench_C_$v.json
done
unset TG_K7_TOKMIX_CTA
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_C.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1; echo "ncu launches rc=$?"
python scripts/launch_agg.py $O/launches_C.csv 12 > $O/launches_C.txt; cat $O/launches_C.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:token_mix -s 2 -c 1 -o $O/ncu_tok python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > $O/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $O/ncu_tok.ncu-rep --page raw --csv > $O/tok_raw.csv 2>/dev/null
ncu -i $O/ncu_tok.ncu-rep --page source --csv --print-source sass > $O/tok_sass.csv 2>/dev/null
for kg in "3 2" "4 4" "4 8" "6 4"; do
  set -- $kg
  timeout 600 python bench.py --workload A --steps 20 --warmup 5 --no-cpu --no-e2e --inflight $1 --graph-batches $2 > $O/A_k$1_g$2.json 2> $O/A_k$1_g$2.err; echo "A k$1 g$2 rc=$?"
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), (d.get('parity') or {}).get('mismatches'))" $O/A_k$1_g$2.json
done
