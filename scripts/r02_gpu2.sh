# round 2, call 2 (re-entry): GPU suite on the restored tree, E/C/D bench,
# launch list of E, reference arm on E
set -x
mkdir -p gpurun_out/r02c2
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c2/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/r02c2/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c2/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02c2/smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02c2/bench_E.json 2> gpurun_out/r02c2/bench_E.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02c2/bench_E.json; tail -3 gpurun_out/r02c2/bench_E.err
for w in C D; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r02c2/bench_$w.json 2> gpurun_out/r02c2/bench_$w.err; echo "bench $w rc=$?"; tail -c 1500 gpurun_out/r02c2/bench_$w.json; done
( time timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r02c2/ref_E.json 2> gpurun_out/r02c2/ref_E.err; echo "ref rc=$?"
tail -c 2000 gpurun_out/r02c2/ref_E.json; tail -5 gpurun_out/r02c2/ref_E.err
