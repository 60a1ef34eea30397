"""Edge-feature placement across the GPUs of one box.

The reference keeps one feature array in host memory and serves every row
from it, whatever the cache says (cache.py:85, training.py:217).  On B200 the
rows live in HBM, and with several GPUs there are two placements:

  replicated   every rank holds the whole table (``graph.edge_features``).
               The upper bound, used when the table fits in one GPU's HBM.
  sharded      rank r holds rows [r*S, (r+1)*S) (S = ceil(rows / world)).
               The cache's resident set is a replicated hot tier in every
               rank's HBM (cache.py:32-55 ``resident``; K6 refills it at the
               epoch boundary).  A miss is read from its owner's shard by K5
               itself: the owner exports a CUDA IPC handle, the other ranks
               map it, and the kernel's row loads cross NVLink.  No staging
               buffer and no collective sit on the data path.

Values never depend on the placement (cache.py:85), so every parity test of
the replicated path holds for the sharded one (tests/test_gpu_parity.py,
``test_sharded_*``).

``ShardedTable`` duck-types a [rows, d] feature table: ``shape``, ``device``
and ``c_store()``.  ``graph.feat_store`` dispatches on it, so a graph whose
``edge_features`` is a ShardedTable runs the unchanged generator.
"""

from __future__ import annotations

import ctypes
import os

from . import _lib
from ._lib import check, ptr
from .graph import padded_rows, row_pitch


def shard_bounds(num_rows, rank, world):
    """[lo, hi) rows of `rank`'s shard: contiguous eid ranges of S = ceil(rows/world)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    S = -(-int(num_rows) // int(world)) if num_rows else 1
    lo = min(rank * S, num_rows)
    return lo, min(lo + S, num_rows), S


class ShardedTable:
    """One rank's view of an f32 [num_rows, d] table sharded by row range.

    shards: list of `world` device tensors (row pitch row_pitch(d)); entry
    `rank` is local, the others are either local tensors (single-process
    virtual shards) or peer memory mapped from other processes.
    """

    def __init__(self, num_rows, d, shard_rows, shards, rank=0, owned=None, mapped=None):
        t = _lib.torch()
        self.num_rows, self.d, self.shard_rows = int(num_rows), int(d), int(shard_rows)
        self.rank, self.world = int(rank), len(shards)
        self.pitch = row_pitch(d)
        self._shards = shards          # keep local tensors alive
        self._owned = owned            # this rank's shard tensor
        self._mapped = mapped or []    # IPC bases to close
        addrs = []
        for s in shards:
            a = s if isinstance(s, int) else int(s.data_ptr())
            if a % 16:
                raise ValueError("shard rows must be 16-byte aligned (taser_b200.h tg_feat_store)")
            addrs.append(a)
        dev = t.device("cuda", t.cuda.current_device())
        self.peer_ptrs = t.tensor(addrs, dtype=t.int64, device=dev)

    # -- table duck-typing ---------------------------------------------------
    @property
    def shape(self):
        return (self.num_rows, self.d)

    @property
    def device(self):
        return self.peer_ptrs.device

    def stride(self, dim):
        return self.pitch if dim == 0 else 1

    def c_store(self, hot=None, hot_ld=0):
        return _lib.tg_feat_store(None, ptr(hot), ptr(self.peer_ptrs), self.shard_rows, self.world, self.d,
                                  self.pitch, int(hot_ld), self.num_rows)

    # -- construction --------------------------------------------------------
    @classmethod
    def split_local(cls, table, world):
        """Single-process virtual shards: `world` separate allocations holding
        the row ranges of a dense [rows, d] CUDA table.  K5 resolves rows
        through the peer table exactly as it does across processes."""
        rows, d = int(table.shape[0]), int(table.shape[1])
        shards = []
        S = None
        for r in range(world):
            lo, hi, S = shard_bounds(rows, r, world)
            sh = padded_rows((max(hi - lo, 1),), d, table.device)
            if hi > lo:
                sh[: hi - lo].copy_(table[lo:hi])
            shards.append(sh)
        return cls(rows, d, S, shards, rank=0, owned=shards[0])

    @classmethod
    def from_process_group(cls, num_rows, d, fill, group=None):
        """Collective: every rank allocates its shard, `fill(shard, lo, hi)`
        writes rows [lo, hi) into it, and the ranks exchange CUDA IPC handles
        (all_gather_object over `group`) and map each other's shards."""
        import torch.distributed as dist
        t = _lib.torch()
        if not (dist.is_available() and dist.is_initialized()):
            # one process: the whole table is this rank's (only) shard
            own = padded_rows((max(int(num_rows), 1),), d, t.device("cuda", t.cuda.current_device()))
            if num_rows:
                fill(own, 0, int(num_rows))
            return cls(num_rows, d, max(int(num_rows), 1), [own], rank=0, owned=own)
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        lo, hi, S = shard_bounds(num_rows, rank, world)
        dev = t.cuda.current_device()
        own = padded_rows((max(hi - lo, 1),), d, t.device("cuda", dev))
        if hi > lo:
            fill(own, lo, hi)
        t.cuda.synchronize()
        hsz = _lib.lib.tg_ipc_handle_size()
        hbuf = ctypes.create_string_buffer(hsz)
        off = ctypes.c_int64(0)
        check(_lib.lib.tg_ipc_export(ptr(own), hbuf, ctypes.byref(off)))
        info = {"rank": rank, "pid": os.getpid(), "handle": bytes(hbuf.raw), "offset": int(off.value)}
        infos = [None] * world
        dist.all_gather_object(infos, info, group=group)
        shards, mapped = [], []
        for r, inf in enumerate(infos):
            if r == rank:
                shards.append(own)
                continue
            base = ctypes.c_void_p()
            check(_lib.lib.tg_ipc_open(ctypes.create_string_buffer(inf["handle"], hsz), ctypes.byref(base)))
            mapped.append(base.value)
            shards.append(int(base.value) + inf["offset"])
        return cls(num_rows, d, S, shards, rank=rank, owned=own, mapped=mapped)

    def close(self):
        """Unmap peer shards (call before the owners free them)."""
        for b in self._mapped:
            _lib.lib.tg_ipc_close(ctypes.c_void_p(b))
        self._mapped = []


def enable_peer_access(world):
    """Direct NVLink access from this device to every other local device.
    Returns the devices that cannot be reached (empty on an NVSwitch box)."""
    t = _lib.torch()
    bad = []
    for p in range(min(world, t.cuda.device_count())):
        ok = ctypes.c_int(0)
        check(_lib.lib.tg_peer_access(p, ctypes.byref(ok)))
        if not ok.value:
            bad.append(p)
    return bad
