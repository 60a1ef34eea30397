set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "tc_gemm or scoring or adaptive or graphmixer or tgat or smoke" > gpurun_out/pytest_gemm.log 2>&1
timeout 900 python bench.py --workload C --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_C.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_C.log 2>&1
tail -n 3 gpurun_out/pytest_gemm.log
