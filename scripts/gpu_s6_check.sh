# full GPU suite + C/D on the current tree
set -x
mkdir -p gpurun_out/final6b
O=gpurun_out/final6b
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
tail -n 3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -n 1 $O/smoke.log
for w in C D; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > $O/bench_$w.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
for w in C D; do tail -n 1 $O/bench_$w.log | cut -c1-120; done
