set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_selector.py -x -q > gpurun_out/pytest_sel.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_all.log 2>&1
tail -n 30 gpurun_out/pytest_sel.log
tail -n 3 gpurun_out/pytest_gpu_all.log
