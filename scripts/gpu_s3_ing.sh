set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "ingest or manifest or fmat" > gpurun_out/pytest_ing.log 2>&1
tail -n 40 gpurun_out/pytest_ing.log
