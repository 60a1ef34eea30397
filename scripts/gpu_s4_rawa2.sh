# raw-A GEMM, 8 converter warps + 64B-swizzled tile: parity, A/B vs the pre-split image, one ncu capture
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "tc_gemm or scoring or graphmixer" > gpurun_out/pytest_rawa2.log 2>&1 || { tail -n 60 gpurun_out/pytest_rawa2.log; exit 1; }
tail -n 2 gpurun_out/pytest_rawa2.log
for w in C D; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/rawa2_${w}.json 2> gpurun_out/rawa2_${w}.err
TG_TC_PACKA=1 timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/packa2_${w}.json 2> gpurun_out/packa2_${w}.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_rawa2_C.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 30 -c 2 -o gpurun_out/prof_rawa python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_rawa.log 2>&1
for f in gpurun_out/rawa2_*.json gpurun_out/packa2_*.json; do echo "$f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])")"; done
