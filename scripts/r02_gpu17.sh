# round 2, call 17: finder through the L2-resident coarse time index (every 64th timestamp per node)
set -x
mkdir -p gpurun_out/r02c17
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c17/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c17/pytest_gpu.txt
for st in 20 200; do
timeout 600 python bench.py --steps $st --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c17/E_s$st.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['minibatch_gen_ms'], d['roofline']['finder'], [(p['find_us']) for p in d['roofline']['per_layer']], d['roofline']['frac'], d['roofline']['path']['frac_over_step'], d['parity']['mismatches'])" gpurun_out/r02c17/E_s$st.json
done
for w in B D; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c17/$w.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['parity']['mismatches'])" gpurun_out/r02c17/$w.json; done
