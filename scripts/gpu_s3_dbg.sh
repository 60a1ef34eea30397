set -x
mkdir -p gpurun_out
TG_SELECT_STATS=1 timeout 600 python scripts/bench_select.py --iters 2 --cpu-iters 1 > gpurun_out/bench_select_dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_aggregator.py -x -q > gpurun_out/pytest_agg.log 2>&1
tail -n 12 gpurun_out/bench_select_dbg.log
tail -n 30 gpurun_out/pytest_agg.log
