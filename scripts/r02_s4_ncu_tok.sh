# round 2, session 4: ncu --set full of the K7 token mixer (C shape)
set -x
O=gpurun_out/r02s4b
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:token_mix -s 2 -c 1 -o $O/ncu_tok python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > $O/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $O/ncu_tok.ncu-rep --page source --csv --print-source sass > $O/tok_sass.csv 2>/dev/null; echo src rc=$?
