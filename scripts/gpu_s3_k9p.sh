set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_selector.py -x -q > gpurun_out/pytest_sel.log 2>&1
timeout 600 python scripts/bench_select.py --cpu-iters 1 > gpurun_out/bench_select.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"chunk_classify|pw_leaf8" -c 2 -o gpurun_out/prof_k9b python scripts/bench_select.py --iters 1 --cpu-iters 1 > /dev/null 2>&1
tail -n 2 gpurun_out/pytest_sel.log; tail -c 300 gpurun_out/bench_select.log
