timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C.csv python bench.py --workload C --steps 1 --warmup 1 --inflight 1 --no-cpu --no-e2e > gpurun_out/ncu_launch_C.log 2>&1
