# round 2, call 41: gather4 only for DRAM-sized tables (>= 512 MB); suite; D / E / C
set -x
mkdir -p gpurun_out/r02c41
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c41/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c41/pytest_gpu.txt
for w in D E C; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c41/$w.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['roofline']['frac'], d['parity']['mismatches'], d['parity'].get('q_max_rel_err'))" gpurun_out/r02c41/$w.json; done
TG_K5_NO_G4=1 timeout 900 python bench.py --workload D --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity > gpurun_out/r02c41/D_nog4.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2))" gpurun_out/r02c41/D_nog4.json
