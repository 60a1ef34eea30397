# round 2, call 25: recent-policy finder fetching the selected entries in the pivot sweep's memory round (6 vs 5 resident blocks)
set -x
mkdir -p gpurun_out/r02c25
L=$PWD/paper_2402_05396_b200
timeout 900 python -m pytest tests/test_gpu_round2.py tests/test_gpu_parity.py tests/test_gpu_reference_cases.py -x -q > gpurun_out/r02c25/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c25/pytest.txt
for v in "" _f5; do for st in 20 200; do
TG_LIB_PATH=$L/libtaser_b200$v.so timeout 600 python bench.py --steps $st --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c25/E${v}_s$st.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['minibatch_gen_ms'], [(p['find_us']) for p in d['roofline']['per_layer']], d['roofline']['avg_launch_us'], d['parity']['mismatches'])" gpurun_out/r02c25/E${v}_s$st.json
done; done
