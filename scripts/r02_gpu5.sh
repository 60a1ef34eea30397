# round 2, call 5: E non-graph with private slot streams (1..K) vs graph replay; ncu source capture of K7 GEMM1
set -x
mkdir -p gpurun_out/r02c5
for k in 2 3 4; do for st in 20 200; do
timeout 300 python bench.py --steps $st --warmup 5 --no-graph --inflight $k --no-cpu --no-e2e --no-parity > gpurun_out/r02c5/E_nograph_k${k}_s$st.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['minibatch_gen_ms'])" gpurun_out/r02c5/E_nograph_k${k}_s$st.json
done; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 6 -c 3 -o gpurun_out/r02c5/ncu_gemm_C python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > gpurun_out/r02c5/ncu_gemm.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r02c5/ncu_gemm.log
ls -la gpurun_out/r02c5/
