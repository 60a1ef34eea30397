# round 2, call 43: timing experiment: K7 GEMM epilogue without its output stores
set -x
mkdir -p gpurun_out/r02c43
L=$PWD/paper_2402_05396_b200
TG_LIB_PATH=$L/libtaser_b200_xnes.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_gemm -c 6 --csv --log-file gpurun_out/r02c43/gemm_xnes.csv python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/r02c43/gemm_xnes.csv 4
