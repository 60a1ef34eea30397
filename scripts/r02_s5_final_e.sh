# round 2, session 5: final check after the 64-B promotion default -- gather tests, smoke, E / B / A lines, default bench
set -x
O=gpurun_out/r02s5w
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "gather or g4 or pipeline or generator or bench" > $O/pytest_sub.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_sub.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.txt
for w in E B A; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w rc=$?"
python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('minibatch_gen_ms'), d.get('value'), r.get('achieved'), r.get('frac'), (d.get('e2e') or {}).get('value'), (d.get('parity') or {}).get('mismatches'), (d.get('cpu_baseline') or {}).get('value'), d.get('clocks'))" $O/bench_$w.json; done
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "default rc=$?"
python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('steps'), d.get('ms_per_step'), d.get('value'), r.get('frac'), (d.get('e2e') or {}).get('value'), (d.get('parity') or {}).get('mismatches'))" $O/bench_default.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:row_gather_g4 -s 4 -c 1 -o $O/ncu_k5 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity --no-graph > /dev/null 2>&1; echo "ncu k5 rc=$?"
