# MMA issue from a whole warp with elect.sync (uniform operands): parity, probe, C/D
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "tc_gemm or scoring or graphmixer or tgat or adaptive" > gpurun_out/pytest_elect.log 2>&1; tail -n 2 gpurun_out/pytest_elect.log
timeout 120 python scripts/tc_issue_probe.py 300000 328 16,64,128 > gpurun_out/probe_elect.log 2>&1
for w in C D; do
timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/elect_${w}.json 2>/dev/null
done
cat gpurun_out/probe_elect.log
for f in gpurun_out/elect_*.json; do echo "$f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])")"; done
