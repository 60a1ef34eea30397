set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_D.csv python bench.py --workload D --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_E.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
