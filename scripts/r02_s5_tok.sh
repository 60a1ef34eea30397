# round 2, session 5: C launch list on the current tree + ncu --set full of the K7 token mixer (C shape)
set -x
O=gpurun_out/r02s5a
mkdir -p $O
nvidia-smi -L
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_C.csv python bench.py --workload C --steps 3 --warmup 3 --no-cpu --no-e2e --no-parity > /dev/null 2>&1; echo "ncu launches rc=$?"
python scripts/launch_agg.py $O/launches_C.csv 20 > $O/launches_C.txt; cat $O/launches_C.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:token_mix -s 2 -c 1 -o $O/ncu_tok python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > $O/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $O/ncu_tok.ncu-rep --page raw --csv > $O/tok_raw.csv 2>/dev/null; echo raw rc=$?
ncu -i $O/ncu_tok.ncu-rep --page source --csv --print-source sass > $O/tok_sass.csv 2>/dev/null; echo src rc=$?
