# round 2, call 23: ncu source-level capture of the E finder (hop-1 and hop-2 launches)
set -x
mkdir -p gpurun_out/r02c23
timeout 600 ncu --set full --import-source on --clock-control none -k regex:find_kernel -s 2 -c 2 -o gpurun_out/r02c23/ncu_find_E python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity --no-graph > /dev/null 2>&1; echo ncu rc=$?
