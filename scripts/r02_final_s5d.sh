# round 2, session 5 final record (3-tile K5 rings, 2 x 2 step groups): GPU suite, smoke, every workload's bench line (driver defaults),
# the reference arm, C in the reference's f64 precision, E launch list
set -x
O=gpurun_out/r02s5final4
mkdir -p $O
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_E.json 2> $O/bench_E.err; echo "E rc=$?"; tail -c 400 $O/bench_E.json
( time timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 ) > $O/bench_E_reference.json 2> $O/bench_E_reference.err; echo "ref rc=$?"
for w in A B C D; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w rc=$?"; done
timeout 900 python bench.py --workload C --precision float64 --steps 3 --warmup 3 --no-cpu > $O/bench_C_f64.json 2> $O/bench_C_f64.err; echo "C f64 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_E.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1; echo "ncu rc=$?"; python scripts/launch_agg.py $O/launches_E.csv 20 > $O/launches_E.txt
for f in $O/bench_*.json; do python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1].split('/')[-1], d.get('ms_per_step'), d.get('value'), d.get('unit'), r.get('frac'), (d.get('e2e') or {}).get('value'), (d.get('parity') or {}).get('mismatches'), (d.get('parity') or {}).get('q_max_rel_err'), (d.get('cpu_baseline') or {}).get('value'), d.get('clocks'))
" $f; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:row_gather_g4 -s 4 -c 1 -o $O/ncu_k5 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity --no-graph > /dev/null 2>&1; echo "ncu k5 rc=$?"
