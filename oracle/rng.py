"""Counter RNGs of the reference, restated (TEST INFRASTRUCTURE).

splitmix64: finder.py:29-33 (constants), :56-60 (_mix), :63-66 (_next),
:99 (row stream).  Seeds: training.py:111-117 (derive_seed, substream),
purpose codes training.py:121.  PCG64 (numpy) restated from its published
definition (128-bit LCG, multiplier 0x2360ED051FC65DA44385DF649FCCF645,
XSL-RR output; numpy random() = (x >> 11) * 2^-53) for the position
arithmetic the device sampler relies on.
"""

from __future__ import annotations

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
STREAM = 0xA24BAED4963EE407
M64 = (1 << 64) - 1
M128 = (1 << 128) - 1
PCG_MUL = 0x2360ED051FC65DA44385DF649FCCF645

S_MODEL, S_SAMPLER, S_BATCH, S_NEG, S_FINDER, S_POLICY, S_EVAL = range(7)


def mix(z):
    """splitmix64 finalizer on a python int (finder.py:56-60)."""
    z &= M64
    z = ((z ^ (z >> 30)) * MIX1) & M64
    z = ((z ^ (z >> 27)) * MIX2) & M64
    return z ^ (z >> 31)


def mix_np(z):
    """Vectorised finalizer on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
    return z ^ (z >> np.uint64(31))


def row_state(seed, row):
    """Initial state of query row `row` (finder.py:99)."""
    return mix((int(seed) ^ ((int(row) * STREAM) & M64)) & M64)


def draw(state, k):
    """k-th output (1-based) of the row stream (k calls of finder.py:_next)."""
    return mix((state + k * GOLDEN) & M64)


def derive_seed(seed, *keys):
    """training.py:111-113."""
    ss = np.random.SeedSequence([int(seed) & 0x7FFFFFFF] + [int(k) & 0x7FFFFFFF for k in keys])
    return int(ss.generate_state(1, dtype=np.uint64)[0])


def substream(seed, *keys):
    """training.py:116-117."""
    return np.random.default_rng(derive_seed(seed, *keys))


def pcg_step(state, inc):
    return (state * PCG_MUL + inc) & M128


def pcg_output(state):
    hi, lo = state >> 64, state & M64
    x = hi ^ lo
    r = hi >> 58
    return ((x >> r) | (x << ((64 - r) & 63))) & M64


def pcg_double_at(state0, inc, position):
    """numpy random() value number `position` (0-based) of the stream."""
    s = state0
    mul, add = 1, 0
    cm, ca, d = PCG_MUL, inc, position + 1
    while d:
        if d & 1:
            mul, add = (mul * cm) & M128, (add * cm + ca) & M128
        ca = ((cm + 1) * ca) & M128
        cm = (cm * cm) & M128
        d >>= 1
    s = (mul * s + add) & M128
    return (pcg_output(s) >> 11) * (1.0 / 9007199254740992.0)
