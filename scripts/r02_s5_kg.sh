# round 2, session 5: E in-flight x graph-batches sweep on the 3-tile K5 rings (driver's 20 steps, two reps)
set -x
O=gpurun_out/r02s5n
mkdir -p $O
for rep in 1 2; do
for kg in "3 2" "3 1" "4 1" "2 2" "4 2" "2 3"; do
  set -- $kg
  timeout 600 python bench.py --workload E --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity --inflight $1 --graph-batches $2 > $O/E_k$1_g$2_r$rep.json 2> /dev/null
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'))" $O/E_k$1_g$2_r$rep.json
done
done
