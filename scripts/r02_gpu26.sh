# round 2, call 26: E in-flight / graph-batch sweep with the current kernels (driver's 20 steps); emulated root shards 1/2, 1/4, 1/8
set -x
mkdir -p gpurun_out/r02c26
for kg in "3 2" "2 1" "3 1" "4 1" "2 2" "4 2" "6 1"; do set -- $kg
timeout 300 python bench.py --steps 20 --warmup 5 --inflight $1 --graph-batches $2 --no-cpu --no-e2e --no-parity > gpurun_out/r02c26/E_k$1g$2.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['run']['host_enqueue_ms_per_step'])" gpurun_out/r02c26/E_k$1g$2.json
done
for sh in 0/2 0/4 0/8; do n=${sh#0/}
timeout 300 python bench.py --steps 20 --warmup 5 --emulate-shard $sh --no-cpu --no-e2e --no-parity > gpurun_out/r02c26/E_shard$n.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d.get('emulated'), d['run'].get('host_enqueue_ms_per_step'), d['run'].get('launch'))" gpurun_out/r02c26/E_shard$n.json
done
