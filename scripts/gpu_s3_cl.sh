set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "tc_gemm" > gpurun_out/pytest_cl.log 2>&1 || { echo GEMMFAIL; tail -30 gpurun_out/pytest_cl.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -k "scoring or adaptive or graphmixer or tgat or smoke" >> gpurun_out/pytest_cl.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C_cl.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
TG_TC_NO_CLUSTER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C_nocl.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 python bench.py --workload C --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_C_cl.log 2>&1
tail -n 3 gpurun_out/pytest_cl.log
