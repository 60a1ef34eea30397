# round 2, call 24: finder: list + coarse bounds in one round, one counting pass over <= 512 coarse entries, unrolled sweeps
set -x
mkdir -p gpurun_out/r02c24
timeout 900 python -m pytest tests/test_gpu_round2.py tests/test_gpu_parity.py tests/test_gpu_reference_cases.py -x -q > gpurun_out/r02c24/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c24/pytest.txt
for st in 20 200; do
timeout 600 python bench.py --steps $st --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c24/E_s$st.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['minibatch_gen_ms'], [(p['find_us']) for p in d['roofline']['per_layer']], d['roofline']['avg_launch_us'], d['roofline']['path']['frac_over_step'], d['parity']['mismatches'])" gpurun_out/r02c24/E_s$st.json
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity --trace gpurun_out/r02c24/trace.jsonl > /dev/null 2>&1; python scripts/trace_overlap.py gpurun_out/r02c24/trace.jsonl
