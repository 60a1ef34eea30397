# round 2, call 3: C/D bench (cpu baseline fixed), TF32 peak, launch lists of C and D
set -x
mkdir -p gpurun_out/r02c3
python scripts/tf32_peak.py gpurun_out/r02c3/tf32_peak.json
for w in C D; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r02c3/bench_$w.json 2> gpurun_out/r02c3/bench_$w.err; echo "bench $w rc=$?"; tail -c 2500 gpurun_out/r02c3/bench_$w.json; tail -3 gpurun_out/r02c3/bench_$w.err; done
for w in C D; do timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c3/launches_$w.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1; echo "ncu $w rc=$?"; python scripts/launch_agg.py gpurun_out/r02c3/launches_$w.csv 25; done
