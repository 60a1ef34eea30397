# round 2, session 5: single-batch latency (minibatch_gen_ms) with merged vs per-layer overlapped K5 (E, B)
set -x
O=gpurun_out/r02s5l
mkdir -p $O
for w in E B; do for v in 0 1; do
  TG_BENCH_LAT_SPLIT=$v timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e --no-parity > $O/${w}_split$v.json 2> /dev/null
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d.get('ms_per_step'), d.get('minibatch_gen_ms'))" $O/${w}_split$v.json
done; done
