# round 2, session 5: K5 ring depth on C (1,072-B rows) and gather4 for D's L2-resident node table
set -x
O=gpurun_out/r02s5j
mkdir -p $O
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --workload ${tag%%_*} --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity > $O/$tag.json 2> /dev/null
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'))" $O/$tag.json; }
run C_default X=1
run C_s3 TG_K5_G4_STAGES=3
run C_s4 TG_K5_G4_STAGES=4
run D_default X=1
run D_g4all TG_K5_G4_MIN_MB=0
run D_s3 TG_K5_G4_STAGES=3
