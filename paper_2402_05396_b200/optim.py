"""Adam on the device for the sampler's parameters (K10, params.py:80-99).

``AdamState`` mirrors the Adam half of the reference's ``ParamStore``: one
(m, v) pair per named tensor, zero-initialised like ``ParamStore.add``
(params.py:47-53), a shared step counter, and ``step`` = ``adam_step``
(bias-corrected update; tensors without a gradient still decay their
moments).  The whole store updates in one launch (``tg_adam_step``) and the
result is bit-identical to the reference's numpy update, float32 and float64.
"""

from __future__ import annotations

import ctypes

from . import _lib
from ._lib import check, stream_ptr


class AdamState:
    def __init__(self, params):
        """params: dict name -> CUDA tensor (float32 or float64, contiguous),
        updated in place by ``step``."""
        t = _lib.torch()
        _lib.require_cuda("AdamState")
        dts = {p.dtype for p in params.values()}
        if len(dts) > 1 or not dts <= {t.float32, t.float64}:
            raise ValueError("one float dtype (float32 or float64) per store")
        for name, p in params.items():
            if not (p.is_cuda and p.is_contiguous()):
                raise ValueError(f"{name}: contiguous CUDA tensor expected")
        self.params = dict(params)
        self.dtype = dts.pop() if dts else t.float64
        self.m = {k: t.zeros_like(p) for k, p in self.params.items()}
        self.v = {k: t.zeros_like(p) for k, p in self.params.items()}
        self.t = 0

    def step(self, grads, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        """ParamStore.adam_step (params.py:80-99).  grads: dict name ->
        tensor (same shape; float64 allowed for a float32 store, as the
        reference's autodiff can hand one over) or None / missing."""
        t = _lib.torch()
        keep = []
        table = (_lib.tg_adam_tensor * max(len(self.params), 1))()
        for i, (name, p) in enumerate(self.params.items()):
            g = grads.get(name) if grads is not None else None
            gd = -1
            if g is not None:
                if not isinstance(g, t.Tensor):
                    import numpy as np
                    g = t.as_tensor(np.ascontiguousarray(g))
                if tuple(g.shape) != tuple(p.shape):
                    raise ValueError(f"{name}: gradient shape {tuple(g.shape)} != {tuple(p.shape)}")
                if g.dtype not in (t.float32, t.float64) or (self.dtype == t.float64 and g.dtype == t.float32):
                    g = g.to(self.dtype)
                g = g.to("cuda").contiguous()
                keep.append(g)
                gd = 0 if g.dtype == t.float32 else 1
            table[i] = _lib.tg_adam_tensor(p.data_ptr(), g.data_ptr() if g is not None else None,
                                           self.m[name].data_ptr(), self.v[name].data_ptr(), p.numel(), gd)
        # every gradient is validated above: only now does the step count
        # advance, so a rejected call leaves the bias correction untouched
        self.t += 1
        bc1 = 1.0 - beta1 ** self.t
        bc2 = 1.0 - beta2 ** self.t
        code = 0 if self.dtype == t.float32 else 1
        check(_lib.lib.tg_adam_step(code, ctypes.cast(table, ctypes.c_void_p), len(self.params), float(lr),
                                    float(beta1), float(beta2), float(eps), bc1, bc2, stream_ptr()))
        del keep
