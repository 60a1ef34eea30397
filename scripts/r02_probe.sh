nproc; free -g; cat /proc/meminfo | head -3; nvidia-smi -L; cat /proc/sys/vm/overcommit_memory; df -h /tmp | tail -1
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r02_probe_bench.json 2> gpurun_out/r02_probe_bench.err
tail -c 600 gpurun_out/r02_probe_bench.json
