# same-box A/B of two builds of the library: in-tree (A) vs exp/libtaser_b200_exp.so (B)
set -x
mkdir -p gpurun_out
L=paper_2402_05396_b200/libtaser_b200.so
cp $L /tmp/libA.so
for i in 1 2; do
for v in A B; do
if [ $v = A ]; then cp /tmp/libA.so $L; else cp exp/libtaser_b200_exp.so $L; fi
for w in C D; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_${v}_${w}_$i.json 2> gpurun_out/ab_${v}_${w}_$i.err
done
done
done
timeout 300 python -m pytest tests -m gpu -x -q -k "tc_gemm or scoring or graphmixer" > gpurun_out/pytest_ab.log 2>&1; tail -n 2 gpurun_out/pytest_ab.log
cp /tmp/libA.so $L
for f in gpurun_out/ab_*.json; do echo "$f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])")"; done
