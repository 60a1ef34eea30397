"""Root sharding of one mini-batch across ranks.

The path shards by root: rank r of W takes a contiguous block [a, b) of the
batch's R1 hop-1 roots.  With the T-CSR replicated, its hop-2 queries are its
own targets plus their children, so no data crosses ranks between hops.  To
stay bit-exact with the 1-GPU output, every counter-based draw keeps its
GLOBAL row key:

  finder (finder.py:99)  row stream keyed by the query's global row index;
  WOR (sampler.py:154)   round k of global row g draws PCG64 output k*B_g + g.

In the reference's hop-2 layout [targets || children] (training.py:312),
local target i is global row a + i and local child j is global row
R1 + a*w + j, which is exactly a tg_rowmap(split=b-a, base0=a,
base1=R1+a*w).  The only cross-rank traffic on the path is the epoch
boundary: per-edge cache counters and hit/miss stats are summed
(all_reduce) before the replacement (cache.py:107-118), so every rank
computes the identical resident set.
"""

from __future__ import annotations

from dataclasses import dataclass


def root_partition(R1, rank, world):
    """Contiguous block [a, b) of R1 roots for `rank` (sizes differ by <= 1)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    base, extra = divmod(int(R1), int(world))
    a = rank * base + min(rank, extra)
    return a, a + base + (1 if rank < extra else 0)


@dataclass(frozen=True)
class LayerRows:
    """Global row keys of one layer's local queries: local i < split maps to
    base0 + i, the rest to base1 + (i - split); B_global is the layer's
    global query count (the WOR stream width)."""

    split: int
    base0: int
    base1: int
    B_local: int
    B_global: int

    def global_rows(self, i):
        import numpy as np
        i = np.asarray(i)
        return np.where(i < self.split, self.base0 + i, self.base1 + (i - self.split))

    def c_rowmap(self):
        from . import _lib
        return _lib.rowmap(self.split, self.base0, self.base1)


def layer_rows(R1, w, a, b, layers):
    """LayerRows for layers L..1 (top first) of the shard [a, b).

    w = slots per query that become next-hop children (n adaptive, the
    finder budget otherwise).  Supports L <= 2 (TGAT / GraphMixer,
    aggregators.py:29-30)."""
    if layers not in (1, 2):
        raise ValueError("root sharding supports 1- and 2-layer models")
    top = LayerRows(split=1 << 62, base0=a, base1=0, B_local=b - a, B_global=R1)
    if layers == 1:
        return [top]
    nb = b - a
    hop2 = LayerRows(split=nb, base0=a, base1=R1 + a * w, B_local=nb * (1 + w), B_global=R1 * (1 + w))
    return [top, hop2]


def epoch_allreduce(tensors, group=None):
    """Sum per-rank cache counters / stats in place (the epoch-boundary
    collective; NCCL over NVLink on the GPU box, gloo in CPU tests)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    host = dist.get_backend(group) == "gloo"
    for t in tensors:
        if host and t.is_cuda:  # gloo reduces host memory (CPU tests, shared-GPU runs)
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
