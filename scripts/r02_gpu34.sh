# round 2, call 34: + cuGraphUpload at capture: E and emulated shards
set -x
mkdir -p gpurun_out/r02c34
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r02c34/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c34/pytest.txt
for cfg in "1 3 2" "1 2 2" "1 4 1" "2 3 2" "2 4 2" "2 4 1" "4 4 4" "4 4 2" "4 8 1" "8 4 4" "8 8 2" "8 4 5" "8 2 10"; do set -- $cfg
if [ $1 = 1 ]; then sh=""; else sh="--emulate-shard 0/$1"; fi
timeout 300 python bench.py --steps 20 --warmup 5 $sh --inflight $2 --graph-batches $3 --no-cpu --no-e2e --no-parity > gpurun_out/r02c34/E_n$1_k$2g$3.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['run'].get('host_enqueue_ms_per_step'))" gpurun_out/r02c34/E_n$1_k$2g$3.json
done
