timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k tc_gemm 2>&1 | tail -3
timeout 300 python scripts/diag_k7.py 2>&1 | tail -14
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
