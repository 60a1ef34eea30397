# MMA-issuer wait breakdown of the raw-A GEMM (debug build with -DTG_TC_PROF):
# cycles spent waiting for the accumulator (epilogue) vs the stage (feed)
mkdir -p gpurun_out
L=paper_2402_05396_b200/libtaser_b200.so
cp $L /tmp/libA.so
cp exp/libtaser_b200_exp.so $L
timeout 300 python bench.py --workload C --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/tcprof_C.log 2>&1
timeout 300 python bench.py --workload D --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/tcprof_D.log 2>&1
cp /tmp/libA.so $L
grep -c TCPROF gpurun_out/tcprof_C.log gpurun_out/tcprof_D.log
# build of exp/libtaser_b200_exp.so: copy paper_2402_05396_b200/csrc and include/ to a scratch tree,
# add -DTG_TC_PROF to NVFLAGS in its Makefile, `make OUT=<repo>/exp/libtaser_b200_exp.so`
