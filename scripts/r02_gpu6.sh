# round 2, call 6: K7 converter changes (integer tf32 rounding, no masking, epilogue back-off): suite, C/D, prof; E concurrency
set -x
mkdir -p gpurun_out/r02c6
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c6/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c6/pytest_gpu.txt
for w in C D; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c6/bench_$w.json 2> gpurun_out/r02c6/bench_$w.err; echo "bench $w rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['roofline']['frac'], d['parity']['q_max_rel_err'], d['parity']['mismatches'], d['parity']['selected_rows_differing'])" gpurun_out/r02c6/bench_$w.json; done
TG_LIB_PATH=$PWD/paper_2402_05396_b200/libtaser_b200_prof.so timeout 300 python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > gpurun_out/r02c6/tcprof_C.txt 2>&1; grep "TCPROF" gpurun_out/r02c6/tcprof_C.txt | grep "cta=0 " | tail -6
for k in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-graph --inflight $k --no-cpu --no-e2e --no-parity > gpurun_out/r02c6/E_ng_k$k.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['minibatch_gen_ms'], d['run']['host_enqueue_ms_per_step'])" gpurun_out/r02c6/E_ng_k$k.json
timeout 300 python bench.py --steps 20 --warmup 5 --inflight $k --graph-batches 1 --no-cpu --no-e2e --no-parity > gpurun_out/r02c6/E_g_k$k.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['minibatch_gen_ms'], d['run']['host_enqueue_ms_per_step'])" gpurun_out/r02c6/E_g_k$k.json
done
