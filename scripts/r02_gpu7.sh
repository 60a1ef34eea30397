# round 2, call 7: K7 converter variants (ln prefetch in all; 3 converter groups + 4 epilogue warps; 4 epilogue warps)
set -x
mkdir -p gpurun_out/r02c7
L=$PWD/paper_2402_05396_b200
for v in "" _g3e4 _e4; do for w in C D; do
TG_LIB_PATH=$L/libtaser_b200$v.so timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e --parity-steps 1 > gpurun_out/r02c7/bench_$w$v.json 2> gpurun_out/r02c7/bench_$w$v.err; echo "bench $w$v rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['roofline']['frac'], d['parity']['q_max_rel_err'], d['parity']['mismatches'], d['parity']['selected_rows_differing'])" gpurun_out/r02c7/bench_$w$v.json
done; done
