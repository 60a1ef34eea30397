# round 2, call 8: K7 raw-A L2 prefetch distance sweep (0 / 3 / 6 default / 12), CTA-pair variant, per-role waits
set -x
mkdir -p gpurun_out/r02c8
L=$PWD/paper_2402_05396_b200
for v in "" _pf0 _pf3 _pf12; do for w in C D; do
TG_LIB_PATH=$L/libtaser_b200$v.so timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e --parity-steps 1 > gpurun_out/r02c8/bench_$w$v.json 2> gpurun_out/r02c8/bench_$w$v.err; echo "bench $w$v rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['roofline']['frac'], d['parity']['q_max_rel_err'], d['parity']['mismatches'], d['parity']['selected_rows_differing'])" gpurun_out/r02c8/bench_$w$v.json
done; done
TG_TC_PAIR=1 timeout 600 python bench.py --workload C --steps 20 --warmup 5 --no-cpu --no-e2e --parity-steps 1 > gpurun_out/r02c8/bench_C_pair.json 2>&1
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['parity']['q_max_rel_err'], d['parity']['mismatches'])" gpurun_out/r02c8/bench_C_pair.json
TG_LIB_PATH=$L/libtaser_b200_prof.so timeout 300 python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > gpurun_out/r02c8/tcprof_C.txt 2>&1; grep "TCPROF" gpurun_out/r02c8/tcprof_C.txt | grep "cta=0 " | tail -6
