# CTA-pair (cta_group::2) raw-A GEMM: parity first (short timeouts: a barrier
# mistake deadlocks), then same-box A/B against the 1-CTA raw-A kernel
set -x
mkdir -p gpurun_out
TG_TC_PAIR=1 timeout 120 python -m pytest tests -m gpu -x -q -k "tc_gemm_3xtf32" > gpurun_out/pytest_pair_gemm.log 2>&1 || { tail -n 40 gpurun_out/pytest_pair_gemm.log; exit 1; }
tail -n 2 gpurun_out/pytest_pair_gemm.log
TG_TC_PAIR=1 timeout 300 python -m pytest tests -m gpu -x -q -k "scoring or adaptive or graphmixer or tgat or smoke" > gpurun_out/pytest_pair.log 2>&1
tail -n 5 gpurun_out/pytest_pair.log
for i in 1 2; do
for w in C D; do
TG_TC_PAIR=1 timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/pair_${w}_$i.json 2>gpurun_out/pair_${w}_$i.err
timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/single_${w}_$i.json 2>/dev/null
done
done
TG_TC_PAIR=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_pair_C.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
for f in gpurun_out/pair_*.json gpurun_out/single_*.json; do echo "$f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])")"; done
