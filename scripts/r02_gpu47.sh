# round 2, call 47: residual slab read coalesced through the staging buffer
set -x
mkdir -p gpurun_out/r02c47
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "scoring or adaptive or tc_gemm" > gpurun_out/r02c47/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c47/pytest_gpu.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_gemm -c 6 --csv --log-file gpurun_out/r02c47/gemm.csv python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/r02c47/gemm.csv 4
for w in C D; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c47/$w.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['roofline']['frac'], d['parity']['mismatches'], d['parity'].get('q_max_rel_err'), d['parity'].get('selected_rows_differing'))" gpurun_out/r02c47/$w.json; done
