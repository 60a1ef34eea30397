# round 2, session 5: K5 gather4 tile height x ring depth (E at 20 / 200 steps), ring parity tests
set -x
O=gpurun_out/r02s5i
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_round2.py -m gpu -q -x -k "gather4_tile_rings or gather_rows_multi" > $O/pytest_rings.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_rings.txt
for ring in 32x3 16x3 16x4 16x6 32x3; do
  r=${ring%x*}; s=${ring#*x}
  for st in 20 200; do
    TG_K5_G4_ROWS=$r TG_K5_G4_STAGES=$s timeout 600 python bench.py --workload E --steps $st --warmup 5 --no-cpu --no-e2e --no-parity > $O/E_${ring}_n$st.json 2> /dev/null
    python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), r.get('avg_launch_us'))" $O/E_${ring}_n$st.json
  done
done
for ring in 32x3 16x4; do
  r=${ring%x*}; s=${ring#*x}
  TG_K5_G4_ROWS=$r TG_K5_G4_STAGES=$s timeout 600 python bench.py --workload B --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity > $O/B_${ring}.json 2> /dev/null
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), r.get('avg_launch_us'))" $O/B_${ring}.json
done
