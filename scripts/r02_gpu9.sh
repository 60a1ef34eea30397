# round 2, call 9: K7 GEMM bottleneck experiments (timing only): converted-A stores removed; hi*hi MMA only
set -x
mkdir -p gpurun_out/r02c9
L=$PWD/paper_2402_05396_b200
for v in "" _xNO_STS _xHIHI_ONLY; do for w in C D; do
TG_LIB_PATH=$L/libtaser_b200$v.so timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity > gpurun_out/r02c9/bench_$w$v.json 2> gpurun_out/r02c9/bench_$w$v.err; echo "bench $w$v rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['roofline']['avg_us_per_layer'])" gpurun_out/r02c9/bench_$w$v.json
done; done
