mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "scoring or adaptive" -x > gpurun_out/pytest_k7.log 2>&1
tail -30 gpurun_out/pytest_k7.log
