set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv -k regex:"find_kernel|gather_kernel" python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:find_kernel -s 12 -c 2 -o gpurun_out/prof_find python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
