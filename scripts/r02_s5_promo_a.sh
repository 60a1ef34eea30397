# round 2, session 5: promotion rule by table size -- A (L2-sized table) and E, driver flags
set -x
O=gpurun_out/r02s5x
mkdir -p $O
for w in A E; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w rc=$?"
python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), (d.get('e2e') or {}).get('value'), (d.get('parity') or {}).get('mismatches'))" $O/bench_$w.json; done
TG_K5_G4_PROMO=1 timeout 900 python bench.py --workload A --steps 20 --warmup 5 --no-cpu --no-e2e > $O/bench_A_p1.json 2> /dev/null
python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'))" $O/bench_A_p1.json
