set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "scoring or adaptive or smoke" > gpurun_out/pytest_tok.log 2>&1
TG_K7_TOKMIX_SMEMW=1 timeout 900 python -m pytest tests -m gpu -q -k "scoring or adaptive" > gpurun_out/pytest_tok_ws.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C_a.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
TG_K7_TOKMIX_SMEMW=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C_b.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
tail -n 2 gpurun_out/pytest_tok.log gpurun_out/pytest_tok_ws.log
