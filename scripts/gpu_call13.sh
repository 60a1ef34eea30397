timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
for W in C D; do timeout 1200 python bench.py --workload $W --steps 10 --warmup 3 --inflight 1 > gpurun_out/bench_$W.log 2>&1; tail -1 gpurun_out/bench_$W.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['ms_per_step'], json.dumps(d['roofline'])[:900], d.get('cpu_baseline'))"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm_kernel" -s 2 -c 2 -o gpurun_out/prof_k7 python bench.py --workload C --steps 1 --warmup 1 --inflight 1 --no-cpu --no-e2e > gpurun_out/ncu_k7.log 2>&1
tail -1 gpurun_out/ncu_k7.log
