# round 2, call 38: D launch list with the current tree; E trace
set -x
mkdir -p gpurun_out/r02c38
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r02c38/launches_D.csv python bench.py --workload D --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/r02c38/launches_D.csv 30
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity --trace gpurun_out/r02c38/trace_E.jsonl > /dev/null 2>&1; python scripts/trace_overlap.py gpurun_out/r02c38/trace_E.jsonl
