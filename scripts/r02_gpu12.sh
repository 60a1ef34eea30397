# round 2, call 12: K7 GEMM with 1-K-step stages (10 / 9 stages, 2 or 4 converter groups) vs 2-K-step stages x5
set -x
mkdir -p gpurun_out/r02c12
L=$PWD/paper_2402_05396_b200
for v in "" _k1g4n10 _k1g2n10 _k1g4n9; do for w in C D; do
TG_LIB_PATH=$L/libtaser_b200$v.so timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e --parity-steps 1 > gpurun_out/r02c12/bench_$w$v.json 2> gpurun_out/r02c12/bench_$w$v.err; echo "bench $w$v rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['roofline']['avg_us_per_layer'], d['parity']['q_max_rel_err'], d['parity']['mismatches'], d['parity']['selected_rows_differing'])" gpurun_out/r02c12/bench_$w$v.json
done; done
TG_LIB_PATH=$L/libtaser_b200_k1g4n10.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_gemm -c 3 --csv --log-file gpurun_out/r02c12/gemm_k1.csv python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/r02c12/gemm_k1.csv 5
