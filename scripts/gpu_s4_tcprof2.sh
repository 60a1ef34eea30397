mkdir -p gpurun_out
L=paper_2402_05396_b200/libtaser_b200.so
cp $L /tmp/libA.so
cp exp/libtaser_b200_exp.so $L
timeout 120 python scripts/tc_issue_probe.py 300000 328 16,128 > gpurun_out/tcprof_probe.log 2>&1
timeout 300 python bench.py --workload C --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/tcprof_C2.log 2>&1
cp /tmp/libA.so $L
