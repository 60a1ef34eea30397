# round 2, session 5: encoder kernel with two threads per TE column (default) vs one (TG_K7_ENC_NOSPLIT)
set -x
O=gpurun_out/r02s5m
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "scoring or adaptive or sampler_grad or reference_cases" > $O/pytest_enc.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_enc.txt
for w in C D; do for v in split nosplit; do
  if [ $v = nosplit ]; then export TG_K7_ENC_NOSPLIT=1; else unset TG_K7_ENC_NOSPLIT; fi
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e > $O/${w}_$v.json 2> /dev/null
  python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[1], d.get('ms_per_step'), d.get('value'), r.get('frac'), (d.get('parity') or {}).get('mismatches'), (d.get('parity') or {}).get('q_max_rel_err'))" $O/${w}_$v.json
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:encode_misc -c 6 --csv --log-file $O/enc_${w}_$v.csv python bench.py --workload $w --steps 3 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1
  python scripts/launch_agg.py $O/enc_${w}_$v.csv 2
done; done
