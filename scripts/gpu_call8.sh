mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -15 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --workload C --steps 6 --warmup 3 --inflight 1 > gpurun_out/bench_C.log 2>&1; tail -2 gpurun_out/bench_C.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm_kernel" -s 2 -c 2 -o gpurun_out/prof_k7 python bench.py --workload C --steps 1 --warmup 1 --inflight 1 --no-cpu --no-e2e > gpurun_out/ncu_k7.log 2>&1
tail -2 gpurun_out/ncu_k7.log
