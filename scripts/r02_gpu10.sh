# round 2, call 10: K7 weight multicast over 2-CTA clusters (halves the L2 weight reads) vs independent CTAs
set -x
mkdir -p gpurun_out/r02c10
for e in "" "TG_TC_CLUSTER=1"; do for w in C D; do
env $e timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e --parity-steps 1 > gpurun_out/r02c10/bench_$w${e:+_cl}.json 2> /dev/null
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], round(d['value']/1e6,2), d['roofline']['avg_us_per_layer'], d['parity']['q_max_rel_err'], d['parity']['mismatches'])" gpurun_out/r02c10/bench_$w${e:+_cl}.json
done; done
TG_TC_CLUSTER=1 timeout 900 ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum,dram__bytes_read.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:tc_gemm -c 6 --csv --log-file gpurun_out/r02c10/gemm_cl.csv python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum,dram__bytes_read.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:tc_gemm -c 6 --csv --log-file gpurun_out/r02c10/gemm_nocl.csv python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
python - <<'PY'
import csv
for f in ("gpurun_out/r02c10/gemm_nocl.csv","gpurun_out/r02c10/gemm_cl.csv"):
    rows=[r for r in csv.reader(open(f)) if len(r)>10]
    h=rows[0]
    for r in rows[1:]:
        d=dict(zip(h,r))
        print(f[-12:], d["ID"], d["Kernel Name"][:30], d["Metric Name"], d["Metric Value"], d["Metric Unit"])
PY
