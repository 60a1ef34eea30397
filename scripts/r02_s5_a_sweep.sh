# round 2, session 5: A (1-hop) step-group / in-flight sweep at the driver's 20 steps
set -x
O=gpurun_out/r02s5b
mkdir -p $O
for kg in "3 2" "4 4" "4 8" "6 4" "4 16"; do
  set -- $kg
  timeout 600 python bench.py --workload A --steps 20 --warmup 5 --no-cpu --no-e2e --inflight $1 --graph-batches $2 > $O/A_k$1_g$2.json 2> $O/A_k$1_g$2.err; echo "A k$1 g$2 rc=$?"
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), (d.get('parity') or {}).get('mismatches'))" $O/A_k$1_g$2.json
done
