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
