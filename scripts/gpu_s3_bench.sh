set -x
mkdir -p gpurun_out
timeout 900 python scripts/bench_select.py > gpurun_out/bench_select.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_select.csv python scripts/bench_select.py --iters 2 --cpu-iters 1 > gpurun_out/ncu_select.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_E.log 2>&1
timeout 900 python bench.py --workload C --steps 20 --warmup 5 > gpurun_out/bench_C.log 2>&1
timeout 900 python bench.py --workload D --steps 20 --warmup 5 > gpurun_out/bench_D.log 2>&1
tail -c 400 gpurun_out/bench_select.log
