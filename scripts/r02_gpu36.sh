# round 2, call 36: step-group sweep for the small 1-hop workload A and for B
set -x
mkdir -p gpurun_out/r02c36
for w in A B; do for kg in "3 2" "4 5" "2 10" "4 4" "3 5" "1 20"; do set -- $kg
timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --inflight $1 --graph-batches $2 --no-cpu --no-e2e --no-parity > gpurun_out/r02c36/${w}_k$1g$2.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['roofline']['frac'], d['run'].get('host_enqueue_ms_per_step'))" gpurun_out/r02c36/${w}_k$1g$2.json
done; done
