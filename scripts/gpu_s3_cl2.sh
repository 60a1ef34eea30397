set -x
mkdir -p gpurun_out
for i in 1 2; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_cl_$i.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
TG_TC_NO_CLUSTER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_nocl_$i.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
nvidia-smi -q -d CLOCK | head -30 > gpurun_out/clk.txt
