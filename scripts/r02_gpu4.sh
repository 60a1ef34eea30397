# round 2, call 4: E in-flight / graph-batch sweep at the driver's 20 steps and at 200 steps
set -x
mkdir -p gpurun_out/r02c4
for kg in "3 2" "2 2" "4 1" "5 1" "2 5" "5 2" "4 5" "10 2" "3 1" "6 1"; do
  set -- $kg
  for st in 20 200; do
    timeout 300 python bench.py --steps $st --warmup 5 --inflight $1 --graph-batches $2 --no-cpu --no-e2e --no-parity > gpurun_out/r02c4/E_k$1_g$2_s$st.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['minibatch_gen_ms'])" gpurun_out/r02c4/E_k$1_g$2_s$st.json
  done
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-graph --no-cpu --no-e2e --no-parity > gpurun_out/r02c4/E_nograph.json 2>/dev/null; tail -c 300 gpurun_out/r02c4/E_nograph.json
# K7 per-role wait counters (TG_TC_PROF build), C shape
TG_LIB_PATH=$PWD/paper_2402_05396_b200/libtaser_b200_prof.so timeout 300 python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > gpurun_out/r02c4/tcprof_C.txt 2>&1; echo "prof rc=$?"
grep TCPROF gpurun_out/r02c4/tcprof_C.txt | head -3
# full ncu captures of the two largest K7 kernels (one launch each)
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'tc_gemm_kernel<1,' -s 2 -c 1 -o gpurun_out/r02c4/ncu_gemm1_C python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'token_mix_red' -s 2 -c 1 -o gpurun_out/r02c4/ncu_tokmix_C python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1; echo "ncu2 rc=$?"
ls -la gpurun_out/r02c4/*.ncu-rep
