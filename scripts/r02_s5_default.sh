# round 2, session 5: the driver's default invocation (no flags) on the final tree
set -x
O=gpurun_out/r02s5u
mkdir -p $O
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "rc=$?"
python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(d.get('steps'), d.get('warmup'), d.get('ms_per_step'), d.get('value'), r.get('frac'), (d.get('e2e') or {}).get('value'), (d.get('parity') or {}).get('mismatches'), (d.get('cpu_baseline') or {}).get('value'), d.get('clocks'))" $O/bench_default.json
