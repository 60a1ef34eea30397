set -x
mkdir -p gpurun_out/final6
O=gpurun_out/final6
nvidia-smi > $O/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 900 python bench.py > $O/bench_E.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_E_ref.log 2>&1
timeout 900 python bench.py --workload C --steps 20 --warmup 5 > $O/bench_C.log 2>&1
timeout 900 python bench.py --workload D --steps 20 --warmup 5 > $O/bench_D.log 2>&1
timeout 600 python bench.py --workload B --steps 50 --warmup 5 > $O/bench_B.log 2>&1
timeout 600 python bench.py --workload A --steps 50 --warmup 5 > $O/bench_A.log 2>&1
timeout 600 python scripts/bench_select.py > $O/bench_select.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_E.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_launch_E.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_launch_C.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_D.csv python bench.py --workload D --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_launch_D.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"row_gather_bulk|find_kernel" -s 20 -c 4 -o $O/prof_E python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_full_E.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"token_mix_x2|tc_gemm_kernel|encode_misc" -s 4 -c 4 -o $O/prof_C python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_full_C.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"chunk_classify|pw_leaf8|chunk_walk" -c 3 -o $O/prof_K9 python scripts/bench_select.py --iters 1 --cpu-iters 1 > $O/ncu_full_K9.log 2>&1
ls -la $O
tail -n 2 $O/pytest_gpu.log $O/smoke.log
