# two converter groups (alternate chunks) + 8 epilogue warps: parity, C/D x2
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "tc_gemm or scoring or graphmixer or tgat or adaptive" > gpurun_out/pytest_grp.log 2>&1; tail -n 2 gpurun_out/pytest_grp.log
for i in 1 2; do for w in C D; do
timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/grp_${w}_$i.json 2>gpurun_out/grp_${w}_$i.err
done; done
for f in gpurun_out/grp_*.json; do echo "$f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])")"; done
