# raw-A GEMM: 2-CTA clusters (weight multicast) vs independent CTAs, same box
set -x
mkdir -p gpurun_out
for i in 1 2; do
for w in C D; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/cl_${w}_$i.json 2>/dev/null
TG_TC_NO_CLUSTER=1 timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/nocl_${w}_$i.json 2>/dev/null
done
done
for f in gpurun_out/cl_*.json gpurun_out/nocl_*.json; do echo "$f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])")"; done
