# round 2, call 18: warp-per-root token mixer (vs the CTA kernel), finder without warp-divergence fallbacks
set -x
mkdir -p gpurun_out/r02c18
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c18/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c18/pytest_gpu.txt
for e in "" "TG_K7_TOKMIX_CTA=1"; do
env $e timeout 600 python bench.py --workload C --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c18/C${e:+_cta}.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['roofline']['frac'], d['roofline']['avg_us_per_layer'], d['parity']['q_max_rel_err'], d['parity']['mismatches'], d['parity']['selected_rows_differing'])" gpurun_out/r02c18/C${e:+_cta}.json
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c18/E.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e9,3), d['minibatch_gen_ms'], [(p['find_us']) for p in d['roofline']['per_layer']], d['parity']['mismatches'])" gpurun_out/r02c18/E.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02c18/launches_C.csv python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/r02c18/launches_C.csv 14
