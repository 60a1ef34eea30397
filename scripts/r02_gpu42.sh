# round 2, call 42: K7 light-epilogue GEMMs with D's heavy-epilogue warp split (1 converter group + 16 epilogue warps) etc.
set -x
mkdir -p gpurun_out/r02c42
L=$PWD/paper_2402_05396_b200
for v in "" _g1e16 _g2e12; do
TG_LIB_PATH=$L/libtaser_b200$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_gemm -c 6 --csv --log-file gpurun_out/r02c42/gemm$v.csv python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/r02c42/gemm$v.csv 4
TG_LIB_PATH=$L/libtaser_b200$v.so timeout 600 python bench.py --workload C --steps 20 --warmup 5 --no-cpu --no-e2e --parity-steps 1 > gpurun_out/r02c42/C$v.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['parity']['q_max_rel_err'], d['parity']['mismatches'])" gpurun_out/r02c42/C$v.json
done
