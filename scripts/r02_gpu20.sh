# round 2, call 20: GPU suite incl. the round-2 parity tests; memcheck / racecheck after the LN-parameter bound fix
set -x
mkdir -p gpurun_out/r02c20
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c20/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02c20/pytest_gpu.txt
for tool in memcheck racecheck; do
timeout 1500 compute-sanitizer --tool $tool --print-limit 30 python scripts/sanitize_workload.py > gpurun_out/r02c20/san_$tool.txt 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/r02c20/san_$tool.txt
done
