# round 2, call 29: batched finder (tg_find_batch) + StepGraph capturing generate_batched: suite, E, emulated shards
set -x
mkdir -p gpurun_out/r02c29
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c29/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02c29/pytest_gpu.txt
for cfg in "1 3 2" "1 2 2" "1 2 5" "1 1 10" "2 3 2" "2 2 5" "4 4 4" "4 2 10" "8 4 4" "8 2 10" "8 1 20"; do set -- $cfg
if [ $1 = 1 ]; then sh=""; else sh="--emulate-shard 0/$1"; fi
timeout 300 python bench.py --steps 20 --warmup 5 $sh --inflight $2 --graph-batches $3 --no-cpu --no-e2e --no-parity > gpurun_out/r02c29/E_n$1_k$2g$3.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['run'].get('host_enqueue_ms_per_step'))" gpurun_out/r02c29/E_n$1_k$2g$3.json
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c29/E_default.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['minibatch_gen_ms'], d['parity']['mismatches'])" gpurun_out/r02c29/E_default.json
