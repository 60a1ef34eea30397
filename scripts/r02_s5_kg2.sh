# round 2, session 5: in-flight 2 vs 3 (2 batches per graph) on A / B / E, 20 and 200 steps
set -x
O=gpurun_out/r02s5p
mkdir -p $O
for w in E B A; do for st in 20 200; do for k in 2 3; do
  timeout 600 python bench.py --workload $w --steps $st --warmup 5 --no-cpu --no-e2e --no-parity --inflight $k --graph-batches 2 > $O/${w}_k${k}_n$st.json 2> /dev/null
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'))" $O/${w}_k${k}_n$st.json
done; done; done
