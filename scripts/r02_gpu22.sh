# round 2, call 22: K5 on the TMA 4-row gather (tile::gather4) vs the per-row bulk copies
set -x
mkdir -p gpurun_out/r02c22
timeout 900 python -m pytest tests/test_gpu_round2.py tests/test_gpu_parity.py -x -q > gpurun_out/r02c22/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c22/pytest.txt
for e in "" "TG_K5_NO_G4=1"; do for st in 20 200; do
env $e timeout 600 python bench.py --steps $st --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c22/E${e:+_nog4}_s$st.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['minibatch_gen_ms'], d['roofline']['avg_launch_us'], d['roofline']['frac'], d['roofline']['path']['frac_over_step'], d['parity']['mismatches'])" gpurun_out/r02c22/E${e:+_nog4}_s$st.json
done; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:row_gather_g4 -s 4 -c 1 -o gpurun_out/r02c22/ncu_k5_g4 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity --no-graph > /dev/null 2>&1; echo ncu rc=$?
