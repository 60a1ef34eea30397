# round 2, session 5: evict-first L2 hint on K5's tensor stores (TG_K5_STORE_HINT) on E / B
set -x
O=gpurun_out/r02s5k
mkdir -p $O
TG_K5_STORE_HINT=1 timeout 600 python -m pytest tests/test_gpu_round2.py -m gpu -q -x -k "gather_rows_multi" > $O/pytest_hint.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_hint.txt
for rep in 1 2; do
for h in 0 1; do
  for st in 20 200; do
    TG_K5_STORE_HINT=$h timeout 600 python bench.py --workload E --steps $st --warmup 5 --no-cpu --no-e2e --no-parity > $O/E_h${h}_n${st}_r$rep.json 2> /dev/null
    python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), r.get('avg_launch_us'))" $O/E_h${h}_n${st}_r$rep.json
  done
done
done
for h in 0 1; do
  TG_K5_STORE_HINT=$h timeout 600 python bench.py --workload B --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity > $O/B_h$h.json 2> /dev/null
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), r.get('avg_launch_us'))" $O/B_h$h.json
done
TG_K5_STORE_HINT=1 timeout 600 ncu --set full --clock-control none -k regex:row_gather_g4 -s 4 -c 1 -o $O/ncu_k5_hint python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity --no-graph > /dev/null 2>&1; echo "ncu rc=$?"
