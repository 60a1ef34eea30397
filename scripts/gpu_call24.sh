for W in C D; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv python bench.py --workload $W --steps 1 --warmup 1 --inflight 1 --no-cpu --no-e2e > /dev/null 2>&1
done
for W in C D; do timeout 1200 python bench.py --workload $W --steps 10 --warmup 3 --inflight 1 > gpurun_out/bench_$W.log 2>&1; tail -1 gpurun_out/bench_$W.log | cut -c1-400; done
