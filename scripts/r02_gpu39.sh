# round 2, call 39: node rows (row * 0.0 for padded slots) through gather4: parity + D
set -x
mkdir -p gpurun_out/r02c39
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c39/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c39/pytest_gpu.txt
for w in D E; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c39/$w.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['roofline']['frac'], d['parity']['mismatches'], d['parity'].get('q_max_rel_err'))" gpurun_out/r02c39/$w.json; done
