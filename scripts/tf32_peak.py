"""Dense TF32 tensor-core peak of this B200: cuBLAS f32 GEMM with TF32 math
(torch.matmul, allow_tf32) at 8192^3, 2*N^3 FLOP, best of 10 after warm-up,
CUDA events; also back-to-back for ~3 s (sustained).  Writes the JSON the
bench's K7 roofline reads (profiles/tf32_peak.json)."""
import json
import sys
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = True
N = 8192
a = torch.randn(N, N, device="cuda")
b = torch.randn(N, N, device="cuda")
for _ in range(5):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b)
    e1.record()
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
flop = 2.0 * N ** 3
burst = flop / (best / 1e3) / 1e12
n, t0 = 0, time.time()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 3.0:
    for _ in range(20):
        torch.matmul(a, b)
    n += 20
    torch.cuda.synchronize()
e1.record()
e1.synchronize()
sust = flop * n / (e0.elapsed_time(e1) / 1e3) / 1e12
out = {"tf32_tflops": round(burst, 1), "tf32_tflops_sustained": round(sust, 1),
       "how": "cuBLAS TF32 GEMM (torch.matmul f32, allow_tf32) 8192^3, 2N^3 FLOP, best of 10 (burst); "
              f"back to back for 3 s (sustained); scripts/tf32_peak.py on {torch.cuda.get_device_name()}"}
print(json.dumps(out))
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as fh:
        json.dump(out, fh, indent=1)
