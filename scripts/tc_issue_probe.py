"""Is the K7 tensor-core GEMM bound by MMA issue or by tensor throughput?
Times tg_tc_gemm (raw-A, bias epilogue) at fixed M, K for N = 16..128 (one
N tile each): issue-bound -> time nearly flat in N; tensor-bound -> time
proportional to N."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2402_05396_b200 import _lib  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 328
NS = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [16, 32, 64, 96, 128]
out = []
for N in NS:
    A = torch.randn(M, K, device="cuda")
    W = torch.randn(K, N, device="cuda") / K ** 0.5
    b = torch.randn(N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    nb = ctypes.c_size_t(0)
    _lib.check(_lib.lib.tg_tc_gemm_workspace(M, N, K, ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    call = lambda: _lib.check(_lib.lib.tg_tc_gemm(_lib.ptr(A), K, M, K, _lib.ptr(W), N, N, _lib.ptr(b), _lib.ptr(C), N,  # noqa: E731
                                                  _lib.ptr(ws), _lib.stream_ptr()))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        call()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    ksteps = (K + 7) // 8
    mtiles = (M + 127) // 128
    per_cta_mma = -(-mtiles // 148) * ksteps * 3
    out.append({"N": N, "us": round(us, 1), "TF/s_useful": round(2 * M * N * K / us / 1e6, 1),
                "cycles_per_mma@1.965GHz": round(us * 1965 / per_cta_mma, 1),
                "tensor_cycles_per_mma": N * 128 * 8 * 2 / 4096, "M": M, "K": K,
                "A_GB/s": round(M * K * 4 / us / 1e3, 1)})
for o in out:
    print(json.dumps(o))
