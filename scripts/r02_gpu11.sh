# round 2, call 11: K7 GEMM ingress experiments (timing only): weight stage loads removed; raw-A loads removed
set -x
mkdir -p gpurun_out/r02c11
L=$PWD/paper_2402_05396_b200
for v in "" _xNO_WLOAD _xNO_ALOAD; do for w in C; do
TG_LIB_PATH=$L/libtaser_b200$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_gemm -c 3 --csv --log-file gpurun_out/r02c11/gemm$v.csv python bench.py --workload $w --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/r02c11/gemm$v.csv 5
done; done
