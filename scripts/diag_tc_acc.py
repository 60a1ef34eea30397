"""Where does the 3xTF32 GEMM error come from?  (a) K=8 (one MMA step),
(b) tf32-exact operands (lo = 0: pure accumulation error), (c) full f32."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_05396_b200 import _lib  # noqa: E402


def tf32(x):
    return (x.view(torch.int32) & ~0x1FFF).view(torch.float32)


def run(A, W):
    M, K = A.shape
    N = W.shape[1]
    lda = (K + 3) // 4 * 4
    Ap = torch.zeros(M, lda)
    Ap[:, :K] = A
    nb = ctypes.c_size_t(0)
    _lib.check(_lib.lib.tg_tc_gemm_workspace(M, N, K, ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    Ad, Wd = Ap.cuda(), W.cuda().contiguous()
    C = torch.empty(M, N, device="cuda")
    _lib.check(_lib.lib.tg_tc_gemm(_lib.ptr(Ad), lda, M, K, _lib.ptr(Wd), N, N, None, _lib.ptr(C), N, _lib.ptr(ws),
                                   _lib.stream_ptr()))
    ref = A.double() @ W.double()
    cb = (A.cuda() @ W.cuda()).double().cpu()
    rms = ref.pow(2).mean().sqrt()
    e = (C.double().cpu() - ref)
    e2 = cb - ref
    sgn = torch.sign(ref)
    return (f"tc max {float(e.abs().max() / rms):.2e} rms {float(e.pow(2).mean().sqrt() / rms):.2e} "
            f"signed-bias {float((e * sgn).mean() / rms):+.2e} | cublas max {float(e2.abs().max() / rms):.2e} "
            f"rms {float(e2.pow(2).mean().sqrt() / rms):.2e} bias {float((e2 * sgn).mean() / rms):+.2e}")


torch.backends.cuda.matmul.allow_tf32 = False
g = torch.Generator().manual_seed(1)
M, N = 8192, 128
for K in (8, 64, 328):
    A = torch.randn(M, K, generator=g)
    W = torch.randn(K, N, generator=g) / K ** 0.5
    print(f"K={K} f32      :", run(A, W))
    print(f"K={K} tf32-exact:", run(tf32(A), tf32(W)))
    Ap = torch.rand(M, K, generator=g)
    Wp = torch.rand(K, N, generator=g)
    print(f"K={K} positive :", run(Ap, Wp))
