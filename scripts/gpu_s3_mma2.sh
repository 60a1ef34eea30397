set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "tc_gemm" > gpurun_out/pytest_mma.log 2>&1 || { echo GEMMFAIL; tail -30 gpurun_out/pytest_mma.log; exit 1; }
for i in 1 2; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_mma2_$i.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
TG_TC_NO_CLUSTER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_mma2nc_$i.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
timeout 600 python bench.py --workload C --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_C_mma.log 2>&1
