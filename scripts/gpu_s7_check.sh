# end-of-session check: full GPU suite, smoke, bench E (default) and C/D on the final tree
set -x
mkdir -p gpurun_out/final7
O=gpurun_out/final7
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
tail -n 2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -n 1 $O/smoke.log
timeout 900 python bench.py > $O/bench_E.log 2>&1
for w in C D; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > $O/bench_$w.log 2>&1; done
for w in E C D; do tail -n 1 $O/bench_$w.log | cut -c1-110; done
