# raw-A GEMM (TMA + converter warps) vs the pre-split A image: parity, then
# same-box A/B of workloads C and D and the launch lists
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "tc_gemm" > gpurun_out/pytest_rawa_gemm.log 2>&1 || { tail -n 60 gpurun_out/pytest_rawa_gemm.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "scoring or adaptive or smoke or graphmixer or tgat or aggregator" > gpurun_out/pytest_rawa.log 2>&1
tail -n 30 gpurun_out/pytest_rawa.log
for i in 1 2; do
for w in C D; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/rawa_${w}_$i.json 2> gpurun_out/rawa_${w}_$i.err
TG_TC_PACKA=1 timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/packa_${w}_$i.json 2> gpurun_out/packa_${w}_$i.err
done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_rawa_C.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
TG_TC_PACKA=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_packa_C.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
for f in gpurun_out/rawa_*.json gpurun_out/packa_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"; done
