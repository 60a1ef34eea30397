# round 2, call 46: full GPU suite with the TMA-store epilogue; ncu --set full of the LN-fused GEMM
set -x
mkdir -p gpurun_out/r02c46
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02c46/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c46/pytest_gpu.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 4 -c 2 -o gpurun_out/r02c46/ncu_gemm_C python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1; echo ncu rc=$?
