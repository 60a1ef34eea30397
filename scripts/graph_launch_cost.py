"""Host cost of one StepGraph replay: torch CUDAGraph.replay() vs a direct
cudaGraphLaunch of the same executable graph (ctypes, libcudart), and the
GPU time of the replayed work -- is a small root shard host-bound?"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import shapes as oshapes  # noqa: E402
from paper_2402_05396_b200 import MiniBatchGenerator, build_graph  # noqa: E402
from paper_2402_05396_b200.pipeline import StepGraph  # noqa: E402
from paper_2402_05396_b200.shapes import SHAPES  # noqa: E402

spec = SHAPES["E"].scaled(0.01)
og = oshapes.make_graph(spec, seed=0)
g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, edge_features=og.edge_features)
cfg = spec.path_config(batch_size=75)  # a 1/8 root share of a 600-edge batch
gen = MiniBatchGenerator(g, cfg, seed=0)
G = 4
rows = []
for it in range(G):
    n, t = gen.roots_for_iteration(it + 5)
    rows.append(StepGraph.pack_row(len(n), gen.L, n, t, gen.seeds_for(it + 5)))
packed = torch.as_tensor(np.stack(rows)).cuda()
sg = StepGraph(gen, packed.shape[1] // 2 - 1 if False else (packed.shape[1] - gen.L) // 2, key="p", G=G,
               inputs=packed, stream=torch.cuda.Stream())
torch.cuda.synchronize()
N = 200
for _ in range(10):
    sg.launch_bound()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(N):
    sg.launch_bound()
t_torch = (time.perf_counter() - t0) / N * 1e6
torch.cuda.synchronize()
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
res = {"torch_replay_host_us": round(t_torch, 2)}
if cudart is not None:
    exec_ = ctypes.c_void_p(sg.graph.raw_cuda_graph_exec())
    st = ctypes.c_void_p(sg.stream.cuda_stream)
    cudart.cudaGraphLaunch.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        cudart.cudaGraphLaunch(exec_, st)
    res["cudaGraphLaunch_host_us"] = round((time.perf_counter() - t0) / N * 1e6, 2)
    torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(sg.stream)
for _ in range(N):
    sg.launch_bound()
e1.record(sg.stream)
torch.cuda.synchronize()
res["gpu_us_per_replay"] = round(e0.elapsed_time(e1) / N * 1e3, 2)
print(res)
