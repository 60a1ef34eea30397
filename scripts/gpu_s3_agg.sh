set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_aggregator.py -q > gpurun_out/pytest_agg.log 2>&1
tail -n 40 gpurun_out/pytest_agg.log
