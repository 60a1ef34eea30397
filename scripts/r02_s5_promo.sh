# round 2, session 5: L2 sector promotion of K5's gather4 row loads (TG_K5_G4_PROMO) on E / B
set -x
O=gpurun_out/r02s5v
mkdir -p $O
for rep in 1 2; do for p in 3 0 1 2; do
  TG_K5_G4_PROMO=$p timeout 600 python bench.py --workload E --steps 200 --warmup 5 --no-cpu --no-e2e --no-parity > $O/E_p${p}_r$rep.json 2> /dev/null
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), r.get('avg_launch_us'))" $O/E_p${p}_r$rep.json
done; done
for p in 3 0 2; do
  TG_K5_G4_PROMO=$p timeout 600 python bench.py --workload B --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity > $O/B_p$p.json 2> /dev/null
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), r.get('avg_launch_us'))" $O/B_p$p.json
done
