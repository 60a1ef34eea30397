# round 2, call 21: K5 tile shape sweep on E (rows x stages at ~96 KB of stages per CTA)
set -x
mkdir -p gpurun_out/r02c21
for cfg in "" 16x8 8x16 16x6; do
env ${cfg:+TG_K5_TILE=$cfg} timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --parity-steps 1 > gpurun_out/r02c21/E_$cfg.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['roofline']['avg_launch_us'], d['roofline']['frac'], d['parity']['mismatches'])" gpurun_out/r02c21/E_$cfg.json
done
