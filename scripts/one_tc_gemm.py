"""One M=300k, N=K=325 3xTF32 GEMM (pack + persistent GEMM) for ncu."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_05396_b200 import _lib  # noqa: E402

M, K, N = 300000, 325, 325
lda = 328
A = torch.randn(M, lda, device="cuda")
W = torch.randn(K, N, device="cuda") / K ** 0.5
C = torch.empty(M, N, device="cuda")
nb = ctypes.c_size_t(0)
_lib.check(_lib.lib.tg_tc_gemm_workspace(M, N, K, ctypes.byref(nb)))
ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
for _ in range(2):
    _lib.check(_lib.lib.tg_tc_gemm(_lib.ptr(A), lda, M, K, _lib.ptr(W), N, N, None, _lib.ptr(C), N, _lib.ptr(ws),
                                   _lib.stream_ptr()))
torch.cuda.synchronize()
print("done")
