set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "scoring or adaptive or smoke or tc_gemm" > gpurun_out/pytest_k7.log 2>&1
timeout 900 python bench.py --workload C --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_C.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_C.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:token_mix_x2 -s 2 -c 1 -o gpurun_out/prof_tok python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_tok.log 2>&1
tail -n 3 gpurun_out/pytest_k7.log
