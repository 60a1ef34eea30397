set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "sharded" > gpurun_out/pytest_sharded.log 2>&1
timeout 600 python bench.py --workload B --steps 50 --warmup 5 --no-cpu --placement sharded > gpurun_out/bench_B_sharded1.log 2>&1
timeout 600 python bench.py --workload B --steps 50 --warmup 5 --no-cpu --placement replicated > gpurun_out/bench_B_repl1.log 2>&1
TG_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --workload B --gpus 2 --steps 50 --warmup 5 --placement sharded > gpurun_out/bench_B_sharded2.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_all.log 2>&1
tail -n 3 gpurun_out/pytest_sharded.log gpurun_out/pytest_gpu_all.log
