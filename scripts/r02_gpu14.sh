# round 2, call 14: E with every layer's rows in one K5 launch: GPU suite, E bench (20 / 200 steps), trace, ncu of the merged K5
set -x
mkdir -p gpurun_out/r02c14
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c14/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c14/pytest_gpu.txt
for st in 20 200; do timeout 600 python bench.py --steps $st --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c14/E_s$st.json 2> gpurun_out/r02c14/E_s$st.err; echo rc=$?
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['minibatch_gen_ms'], d['run']['host_enqueue_ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d['roofline']['path']['frac_over_step'], d['parity']['mismatches'])" gpurun_out/r02c14/E_s$st.json; done
for kg in "2 2" "4 1" "2 1" "3 1"; do set -- $kg; timeout 300 python bench.py --steps 20 --warmup 5 --inflight $1 --graph-batches $2 --no-cpu --no-e2e --no-parity > gpurun_out/r02c14/E_k$1g$2.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3))" gpurun_out/r02c14/E_k$1g$2.json; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity --trace gpurun_out/r02c14/trace_graph.jsonl > /dev/null 2>&1; python scripts/trace_overlap.py gpurun_out/r02c14/trace_graph.jsonl
timeout 600 ncu --set full --import-source on --clock-control none -k regex:row_gather_bulk -s 4 -c 1 -o gpurun_out/r02c14/ncu_k5_merged python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity --no-graph > /dev/null 2>&1; echo ncu rc=$?
for w in A B; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c14/$w.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['roofline']['frac'], d['parity']['mismatches'])" gpurun_out/r02c14/$w.json; done
