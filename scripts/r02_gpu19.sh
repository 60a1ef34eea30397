# round 2, call 19: compute-sanitizer (memcheck, racecheck, synccheck) on a small workload covering every kernel
# family; K1 / K6 / K8 launch list with DRAM bytes at the E and C shapes
set -x
mkdir -p gpurun_out/r02c19
for tool in memcheck racecheck synccheck; do
timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_workload.py > gpurun_out/r02c19/san_$tool.txt 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/r02c19/san_$tool.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02c19/setup_E.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity --no-graph > /dev/null 2>&1; echo ncuE rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:wor_kernel --csv --log-file gpurun_out/r02c19/wor_C.csv python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1; echo ncuC rc=$?
