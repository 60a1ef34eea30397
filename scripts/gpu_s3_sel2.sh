set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_selector.py -x -q > gpurun_out/pytest_sel.log 2>&1
timeout 600 python scripts/bench_select.py --cpu-iters 1 > gpurun_out/bench_select.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_select.csv python scripts/bench_select.py --iters 2 --cpu-iters 1 > gpurun_out/ncu_select.log 2>&1
tail -n 30 gpurun_out/pytest_sel.log
tail -c 500 gpurun_out/bench_select.log
