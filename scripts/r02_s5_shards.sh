# round 2, session 5: emulated root shares (rank 0's block alone) on the final defaults -> projected scaling
set -x
O=gpurun_out/r02s5r
mkdir -p $O
for n in 1 2 4 8; do
  if [ $n = 1 ]; then sh=""; else sh="--emulate-shard 0/$n"; fi
  timeout 600 python bench.py --steps 20 --warmup 5 $sh --no-cpu --no-e2e --no-parity > $O/E_shard$n.json 2> /dev/null
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), (d.get('run') or {}).get('inflight'), d.get('emulated_shard') or d.get('projection'))" $O/E_shard$n.json
done
