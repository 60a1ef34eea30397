# same-box A/B: in-tree library (A) vs exp/libtaser_b200_exp.so (B): GEMM probe, parity, C/D
set -x
mkdir -p gpurun_out
L=paper_2402_05396_b200/libtaser_b200.so
cp $L /tmp/libA.so
for v in A B; do
if [ $v = A ]; then cp /tmp/libA.so $L; else cp exp/libtaser_b200_exp.so $L; fi
timeout 120 python scripts/tc_issue_probe.py 300000 328 16,128 > gpurun_out/ab2_probe_$v.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "tc_gemm_3xtf32 or scoring or graphmixer" > gpurun_out/ab2_pytest_$v.log 2>&1
for w in C D; do
timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab2_${v}_${w}.json 2>/dev/null
done
done
cp /tmp/libA.so $L
tail -n 1 gpurun_out/ab2_pytest_A.log gpurun_out/ab2_pytest_B.log
cat gpurun_out/ab2_probe_A.log gpurun_out/ab2_probe_B.log
for f in gpurun_out/ab2_*.json; do echo "$f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])")"; done
