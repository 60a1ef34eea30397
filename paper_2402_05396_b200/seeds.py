"""Seed derivation and PCG64 stream arithmetic (host side).

``derive_seed``/``substream`` mirror training.py:111-117 exactly (numpy
SeedSequence -> PCG64), with the purpose codes of training.py:121.  The
device sampler (K8) does not run numpy: it receives the PCG64 (state, inc)
and the LCG jump constants computed here, and reproduces numpy's draws by
position (sampler.py:149-154 draws round k for row b at output k*B + b).
"""

from __future__ import annotations

import numpy as np

from . import _lib

S_MODEL, S_SAMPLER, S_BATCH, S_NEG, S_FINDER, S_POLICY, S_EVAL = range(7)

PCG_MUL = 0x2360ED051FC65DA44385DF649FCCF645
_M128 = (1 << 128) - 1


def derive_seed(seed, *keys):
    ss = np.random.SeedSequence([int(seed) & 0x7FFFFFFF] + [int(k) & 0x7FFFFFFF for k in keys])
    return int(ss.generate_state(1, dtype=np.uint64)[0])


def substream(seed, *keys):
    return np.random.default_rng(derive_seed(seed, *keys))


def lcg_jump(delta, inc):
    """(mul, add) with state_{+delta} = mul*state + add (mod 2^128)."""
    acc_mul, acc_add = 1, 0
    cur_mul, cur_add = PCG_MUL, inc & _M128
    delta = int(delta)
    while delta > 0:
        if delta & 1:
            acc_mul = (acc_mul * cur_mul) & _M128
            acc_add = (acc_add * cur_mul + cur_add) & _M128
        cur_add = ((cur_mul + 1) * cur_add) & _M128
        cur_mul = (cur_mul * cur_mul) & _M128
        delta >>= 1
    return acc_mul, acc_add


def pcg_state(rng):
    """(state, inc) of a numpy PCG64 Generator / BitGenerator."""
    bg = rng.bit_generator if hasattr(rng, "bit_generator") else rng
    st = bg.state
    if st.get("bit_generator") != "PCG64":
        raise ValueError("the device sampler reproduces numpy PCG64 streams only")
    if st.get("has_uint32"):
        # a buffered 32-bit half does not affect random() (full 64-bit draws)
        pass
    return int(st["state"]["state"]), int(st["state"]["inc"])


def device_pcg(rng, B_global):
    """tg_pcg64 for the C-ABI: initial state + jump by B_global draws."""
    state, inc = pcg_state(rng)
    jm, ja = lcg_jump(B_global, inc)
    p = _lib.tg_pcg64()
    p.state_hi, p.state_lo = _lib.u128_split(state)
    p.inc_hi, p.inc_lo = _lib.u128_split(inc)
    p.jmul_hi, p.jmul_lo = _lib.u128_split(jm)
    p.jadd_hi, p.jadd_lo = _lib.u128_split(ja)
    return p
