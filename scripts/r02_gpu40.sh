set -x
mkdir -p gpurun_out/r02c40
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r02c40/launches_D.csv python bench.py --workload D --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/r02c40/launches_D.csv 12
TG_K5_NO_G4=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r02c40/launches_D_nog4.csv python bench.py --workload D --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/r02c40/launches_D_nog4.csv 12
