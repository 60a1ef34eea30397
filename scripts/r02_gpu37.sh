# round 2, call 37: gather4 tiles written back by ONE tensor store per tile (padded smem pitch) vs per-group bulk stores
set -x
mkdir -p gpurun_out/r02c37
timeout 900 python -m pytest tests/test_gpu_round2.py tests/test_gpu_parity.py -x -q > gpurun_out/r02c37/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c37/pytest.txt
for e in "" "TG_K5_G4_BULKSTORE=1"; do for w in E C; do
env $e timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02c37/$w${e:+_bulk}.json 2>/dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']; print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), r['frac'], r.get('avg_launch_us'), d['parity']['mismatches'])" gpurun_out/r02c37/$w${e:+_bulk}.json
done; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:row_gather_g4 -c 4 --csv --log-file gpurun_out/r02c37/g4.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity --no-graph > /dev/null 2>&1; python scripts/launch_bw.py gpurun_out/r02c37/g4.csv
