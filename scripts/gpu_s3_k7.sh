set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_all.log 2>&1
timeout 600 python bench.py --workload B --steps 50 --warmup 5 --no-cpu --placement sharded > gpurun_out/bench_B_sharded1.log 2>&1
timeout 900 python bench.py --workload C --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_C.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_C.log 2>&1
tail -n 3 gpurun_out/pytest_gpu_all.log
