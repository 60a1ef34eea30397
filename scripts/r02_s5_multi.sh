# round 2, session 5: multi-rank / bench GPU tests on the new step-group defaults
set -x
O=gpurun_out/r02s5t
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q > $O/pytest_multi.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_multi.txt
