# round 2, session 5: E / B bench lines (driver flags) with the e2e leg back on three slots
set -x
O=gpurun_out/r02s5q
mkdir -p $O
for w in E B; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w rc=$?"
python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), (d.get('e2e') or {}).get('value'), (d.get('e2e') or {}).get('note'), (d.get('parity') or {}).get('mismatches'), d.get('clocks'))" $O/bench_$w.json; done
