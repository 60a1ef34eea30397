# round 2, session 5: step groups for emulated 1/2, 1/4, 1/8 shares on the 3-tile K5 rings
set -x
O=gpurun_out/r02s5s
mkdir -p $O
for n in 2 4 8; do for kg in "4 1" "2 2" "4 2" "2 4" "4 4" "3 4" "2 8"; do
  set -- $kg
  timeout 300 python bench.py --steps 20 --warmup 5 --emulate-shard 0/$n --inflight $1 --graph-batches $2 --no-cpu --no-e2e --no-parity > $O/E_s${n}_k$1_g$2.json 2> /dev/null
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d.get('ms_per_step'))" $O/E_s${n}_k$1_g$2.json
done; done
