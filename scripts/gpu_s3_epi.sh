set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "tc_gemm" > gpurun_out/pytest_epi.log 2>&1 || { echo GEMMFAIL; tail -30 gpurun_out/pytest_epi.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_epi_all.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C_epi.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 python bench.py --workload C --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_C_epi.log 2>&1
timeout 600 python bench.py --workload D --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_D_epi.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"tc_gemm_kernel" -s 3 -c 2 -o gpurun_out/prof_gemm_epi python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
tail -n 3 gpurun_out/pytest_epi.log gpurun_out/pytest_epi_all.log
