# round 2, session 5: K5 gather4 ring depth sweep (TG_K5_G4_STAGES) on E and B
set -x
O=gpurun_out/r02s5g
mkdir -p $O
for w in E B; do
for s in 4 3 6 2; do
  TG_K5_G4_STAGES=$s timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity > $O/${w}_s$s.json 2> $O/${w}_s$s.err; echo "$w s$s rc=$?"
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), r.get('avg_launch_us'))" $O/${w}_s$s.json
done
done
