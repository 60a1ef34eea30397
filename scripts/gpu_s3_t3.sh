set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "scoring or adaptive or smoke" > gpurun_out/pytest_t3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_t3.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 python bench.py --workload C --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_C_t3.log 2>&1
tail -n 2 gpurun_out/pytest_t3.log
