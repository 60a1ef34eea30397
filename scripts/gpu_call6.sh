mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
for K in 1 2 3; do timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu --inflight $K > gpurun_out/bench_k$K.log 2>&1; tail -1 gpurun_out/bench_k$K.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('K', d['config']['inflight'], d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['per_layer'], d['e2e'])"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"find_kernel|row_gather" -s 24 -c 4 -o gpurun_out/prof_tile2 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --inflight 1 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
