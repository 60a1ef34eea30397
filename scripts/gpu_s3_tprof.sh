set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"token_mix_x2|tc_pack_a|encode_misc" -s 3 -c 4 -o gpurun_out/prof_tok2 python bench.py --workload C --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ls -la gpurun_out/prof_tok2*
