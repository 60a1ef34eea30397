# round 2, call 1: GPU suite, E bench with the full-size parity check, the
# reference arm (real tgadapt from baseline/_ref) on the full E graph
set -x
mkdir -p gpurun_out/r02c1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c1/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02c1/pytest_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02c1/bench_E.json 2> gpurun_out/r02c1/bench_E.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r02c1/bench_E.json
( time timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r02c1/ref_E.json 2> gpurun_out/r02c1/ref_E.err; echo "ref rc=$?"
tail -c 2500 gpurun_out/r02c1/ref_E.json; tail -5 gpurun_out/r02c1/ref_E.err
