# final-ish ncu captures: E step (find + bulk gather), C step K7 GEMMs + token mixer
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"find_kernel|row_gather_bulk" -s 24 -c 4 -o gpurun_out/prof_E python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --inflight 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_E.csv python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e --inflight 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm_kernel|token_mix|encode_misc|tc_pack_a" -c 6 -o gpurun_out/prof_C python bench.py --workload C --steps 1 --warmup 0 --inflight 1 --no-cpu --no-e2e > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
