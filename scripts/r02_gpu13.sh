# round 2, call 13: E kernel timeline (CUPTI via torch.profiler) for graph replay and generate() slots
set -x
mkdir -p gpurun_out/r02c13
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity --trace gpurun_out/r02c13/trace_graph.jsonl > gpurun_out/r02c13/E_graph.json 2> gpurun_out/r02c13/E_graph.err; echo rc=$?
python scripts/trace_overlap.py gpurun_out/r02c13/trace_graph.jsonl
timeout 300 python bench.py --steps 20 --warmup 5 --no-graph --inflight 2 --no-cpu --no-e2e --no-parity --trace gpurun_out/r02c13/trace_ng2.jsonl > gpurun_out/r02c13/E_ng2.json 2> gpurun_out/r02c13/E_ng2.err; echo rc=$?
python scripts/trace_overlap.py gpurun_out/r02c13/trace_ng2.jsonl
tail -3 gpurun_out/r02c13/E_graph.err
