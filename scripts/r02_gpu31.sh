# round 2, call 31: bound-graph group sizes dividing the 20 timed steps; host cost of one replay
set -x
mkdir -p gpurun_out/r02c31
for cfg in "8 4 5" "8 2 10" "8 3 5" "8 1 20" "4 4 5" "4 2 10" "2 4 5" "2 2 10" "1 4 5"; do set -- $cfg
if [ $1 = 1 ]; then sh=""; else sh="--emulate-shard 0/$1"; fi
timeout 300 python bench.py --steps 20 --warmup 5 $sh --inflight $2 --graph-batches $3 --no-cpu --no-e2e --no-parity > gpurun_out/r02c31/E_n$1_k$2g$3.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['run'].get('host_enqueue_ms_per_step'))" gpurun_out/r02c31/E_n$1_k$2g$3.json
done
timeout 300 python bench.py --steps 20 --warmup 5 --emulate-shard 0/8 --inflight 4 --graph-batches 4 --no-cpu --no-e2e --no-parity --trace gpurun_out/r02c31/trace_n8.jsonl > /dev/null 2>&1; python scripts/trace_overlap.py gpurun_out/r02c31/trace_n8.jsonl
