set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "tc_gemm" > gpurun_out/pytest_mma.log 2>&1 || { echo GEMMFAIL; tail -30 gpurun_out/pytest_mma.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -k "scoring or adaptive or graphmixer or tgat or smoke" >> gpurun_out/pytest_mma.log 2>&1
for st in 6 4; do
TG_TC_STAGES=$st timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_mma_st$st.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
timeout 600 python bench.py --workload C --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_C_mma.log 2>&1
tail -n 3 gpurun_out/pytest_mma.log
