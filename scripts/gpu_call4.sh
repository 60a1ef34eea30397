mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -30 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv -k regex:"find_kernel|row_gather|count_kernel" python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"find_kernel|row_gather" -s 24 -c 4 -o gpurun_out/prof_tile python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
