set -x
mkdir -p gpurun_out
for st in 4 5 6; do
TG_TC_STAGES=$st timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_st$st.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
TG_TC_NO_CLUSTER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_st6nc.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
