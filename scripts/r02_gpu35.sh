# round 2, call 35: gather4 with 8-byte elements (rows up to 2 KB: C's 268-float rows too)
set -x
mkdir -p gpurun_out/r02c35
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c35/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c35/pytest_gpu.txt
for w in E C D B; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c35/$w.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['roofline']['frac'], d['parity']['mismatches'], d['parity'].get('q_max_rel_err'))" gpurun_out/r02c35/$w.json; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02c35/launches_C.csv python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/r02c35/launches_C.csv 14
