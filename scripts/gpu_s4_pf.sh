# raw-A GEMM: L2 prefetch of the next unit's A rows vs none (same box)
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "tc_gemm_3xtf32 or scoring or graphmixer" > gpurun_out/pytest_pf.log 2>&1; tail -n 2 gpurun_out/pytest_pf.log
timeout 300 python scripts/tc_issue_probe.py > gpurun_out/tc_probe_pf.log 2>&1
TG_TC_NO_PREFETCH=1 timeout 300 python scripts/tc_issue_probe.py > gpurun_out/tc_probe_nopf.log 2>&1
for i in 1 2; do
for w in C D; do
timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/pf_${w}_$i.json 2>/dev/null
TG_TC_NO_PREFETCH=1 timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/nopf_${w}_$i.json 2>/dev/null
done
done
cat gpurun_out/tc_probe_pf.log gpurun_out/tc_probe_nopf.log
for f in gpurun_out/pf_*.json gpurun_out/nopf_*.json; do echo "$f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])")"; done
