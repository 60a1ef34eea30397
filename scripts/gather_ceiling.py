"""Attainable bandwidth of the K5 row gather for 186-float rows in 752-B
slots (the GDELT table layout), by index pattern, on a 40 GB table (>> L2):
sequential ids, uniform-random ids, and plain torch copy for reference."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_05396_b200 import _lib  # noqa: E402
from paper_2402_05396_b200.graph import feat_store, padded_rows  # noqa: E402

d = 186
rows = 40 * (1 << 30) // 752
table = padded_rows((rows,), d, "cuda")
n = 198000
out = padded_rows((n,), d, "cuda", zero=False)
store = feat_store(table)
mask = torch.ones(n, dtype=torch.uint8, device="cuda")
g = torch.Generator(device="cuda").manual_seed(0)
pats = {"sequential": torch.arange(n, device="cuda", dtype=torch.int64) + rows // 3,
        "random": torch.randint(0, rows, (n,), device="cuda", generator=g),
        "random-sorted": torch.sort(torch.randint(0, rows, (n,), device="cuda", generator=g)).values}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, ids in pats.items():
    for _ in range(3):
        _lib.lib.tg_gather_rows(_lib.ptr(ids), _lib.ptr(mask), n, store, None, 0, _lib.ptr(out), 188,
                                _lib.stream_ptr())
    torch.cuda.synchronize()
    reps = 20
    e0.record()
    for r in range(reps):
        idr = ids if name == "sequential" else (ids + r * 7919) % rows
        _lib.lib.tg_gather_rows(_lib.ptr(idr), _lib.ptr(mask), n, store, None, 0, _lib.ptr(out), 188,
                                _lib.stream_ptr())
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    gbs = 2 * n * d * 4 / (us * 1e-6) / 1e9
    print(f"{name:14s} {us:7.1f} us  {gbs:7.1f} GB/s algorithmic (read+write)", flush=True)
src = torch.empty(n * 188, device="cuda")
dst = torch.empty_like(src)
for _ in range(3):
    dst.copy_(src)
e0.record()
for _ in range(20):
    dst.copy_(src)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
print(f"torch copy of the same bytes {us:.1f} us {2 * src.numel() * 4 / (us * 1e-6) / 1e9:.1f} GB/s")
