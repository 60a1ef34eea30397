"""K7 precision diagnostics on the GPU: max relative error of q / log q for the
golden scoring cases (f32 tensor cores, f32 CUDA cores, f64), and the raw
3xTF32 GEMM error (relative to |C| and signed bias) at K=325."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import load_golden  # noqa: E402
from test_oracle_golden import scoring_inputs  # noqa: E402

from paper_2402_05396_b200 import _lib  # noqa: E402
from paper_2402_05396_b200.params import ScoringModel, sampler_params  # noqa: E402
from paper_2402_05396_b200.scoring import score_policy  # noqa: E402

z = load_golden("scoring")
for tag in ["s0", "s1", "s2", "s3", "s4", "s5", "s6", "s7"]:
    c = scoring_inputs(z, tag)
    p = sampler_params(c["store_seed"], c["enc"], c["m"], c["d_v"], c["d_e"], c["decoder"])
    out = []
    for prec, tc in (("float32", True), ("float32", False), ("float64", None)):
        model = ScoringModel(p, c["decoder"], c["enc"], c["m"], c["d_v"], c["d_e"], c["alpha"], c["beta"],
                             precision=prec, tensor_cores=tc)
        dev = lambda x, dt: None if x is None else torch.as_tensor(x).to("cuda", dt)  # noqa: E731
        q, lq = score_policy(model, dev(c["ids"], torch.int64), dev(c["dts"], torch.float64),
                             dev(c["mask"], torch.bool), dev(c["node_rows"], torch.float32),
                             dev(c["edge_rows"], torch.float32), dev(c["tgt_rows"], torch.float32))
        q = q.double().cpu().numpy()
        rq = z[f"{tag}/q"]
        nz = rq > 0
        rel = np.abs(q - rq)[nz] / rq[nz]
        out.append(f"{prec}{'/tc' if tc else ''}: max rel {rel.max():.2e} p99 {np.quantile(rel, 0.99):.2e}")
    print(tag, c["decoder"], " | ".join(out), flush=True)

g = torch.Generator().manual_seed(0)
for K, N in ((325, 325), (425, 425), (266, 100)):
    M = 4096
    lda = (K + 3) // 4 * 4
    A = torch.zeros(M, lda)
    A[:, :K] = torch.randn(M, K, generator=g)
    W = (torch.rand(K, N, generator=g) * 2 - 1) * (6.0 / (K + N)) ** 0.5
    ref = A[:, :K].double() @ W.double()
    nb = ctypes.c_size_t(0)
    _lib.check(_lib.lib.tg_tc_gemm_workspace(M, N, K, ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    Ad, Wd = A.cuda(), W.cuda()
    C = torch.empty(M, N, device="cuda")
    _lib.check(_lib.lib.tg_tc_gemm(_lib.ptr(Ad), lda, M, K, _lib.ptr(Wd), N, N, None, _lib.ptr(C), N, _lib.ptr(ws),
                                   _lib.stream_ptr()))
    f32 = (Ad[:, :K] @ Wd).double().cpu()  # cuBLAS fp32 (TF32 off by default) for comparison
    err = C.double().cpu() - ref
    e32 = f32 - ref
    rms = ref.pow(2).mean().sqrt()
    print(f"gemm K={K} N={N}: tc max|err|/rms {float(err.abs().max() / rms):.2e} mean err/rms "
          f"{float(err.mean() / rms):+.2e} | cublas f32 max {float(e32.abs().max() / rms):.2e} "
          f"mean {float(e32.mean() / rms):+.2e}")
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    M2 = 300000
    _lib.check(_lib.lib.tg_tc_gemm_workspace(M2, N, K, ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    A2 = torch.randn(M2, lda, device="cuda")
    C2 = torch.empty(M2, N, device="cuda")
    for _ in range(3):
        _lib.lib.tg_tc_gemm(_lib.ptr(A2), lda, M2, K, _lib.ptr(Wd), N, N, None, _lib.ptr(C2), N, _lib.ptr(ws),
                            _lib.stream_ptr())
    t0.record()
    for _ in range(10):
        _lib.lib.tg_tc_gemm(_lib.ptr(A2), lda, M2, K, _lib.ptr(Wd), N, N, None, _lib.ptr(C2), N, _lib.ptr(ws),
                            _lib.stream_ptr())
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / 10
    fl = 2.0 * M2 * N * K
    print(f"   M={M2}: {ms * 1e3:.1f} us/launch, {fl / ms / 1e9:.1f} useful TFLOP/s, {3 * fl / ms / 1e9:.1f} issued tf32 TFLOP/s",
          flush=True)
