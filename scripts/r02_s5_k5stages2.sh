# round 2, session 5: K5 gather4 ring depth, confirmation (E at 20 and 200 steps, two reps; A, B at 20)
set -x
O=gpurun_out/r02s5h
mkdir -p $O
for rep in 1 2; do
for s in 2 3 4; do
  for st in 20 200; do
    TG_K5_G4_STAGES=$s timeout 600 python bench.py --workload E --steps $st --warmup 5 --no-cpu --no-e2e --no-parity > $O/E_s${s}_n${st}_r$rep.json 2> /dev/null
    python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), r.get('avg_launch_us'))" $O/E_s${s}_n${st}_r$rep.json
  done
done
done
for w in A B; do for s in 2 3 4; do
  TG_K5_G4_STAGES=$s timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity > $O/${w}_s$s.json 2> /dev/null
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), r.get('avg_launch_us'))" $O/${w}_s$s.json
done; done
