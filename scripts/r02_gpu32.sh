set -x
mkdir -p gpurun_out/r02c32
timeout 600 python scripts/graph_launch_cost.py 2>&1 | tail -3
