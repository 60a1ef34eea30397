python scripts/gather_ceiling.py
TG_K5_REGISTER_PATH=1 python scripts/gather_ceiling.py | head -3
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for K in 3; do timeout 900 python bench.py --steps 200 --warmup 10 --no-cpu --inflight $K > gpurun_out/bench_k$K.log 2>&1; tail -1 gpurun_out/bench_k$K.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('K', d['config']['inflight'], d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['per_layer'], d['roofline']['path'])"; done
TG_K5_REGISTER_PATH=1 timeout 900 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --inflight 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('REG K3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['path'])"
