# round 2, call 28: kernel timeline of an emulated 1/8 root shard (20-batch graph and 4x4)
set -x
mkdir -p gpurun_out/r02c28
timeout 300 python bench.py --steps 20 --warmup 5 --emulate-shard 0/8 --inflight 1 --graph-batches 20 --no-cpu --no-e2e --no-parity --trace gpurun_out/r02c28/trace_n8_g20.jsonl > /dev/null 2>&1; python scripts/trace_overlap.py gpurun_out/r02c28/trace_n8_g20.jsonl
timeout 300 python bench.py --steps 20 --warmup 5 --emulate-shard 0/8 --no-cpu --no-e2e --no-parity --trace gpurun_out/r02c28/trace_n8.jsonl > /dev/null 2>&1; python scripts/trace_overlap.py gpurun_out/r02c28/trace_n8.jsonl
head -30 gpurun_out/r02c28/trace_n8_g20.jsonl
