"""cuBLAS int8 (torch._int_mm, s8 x s8 -> s32, no check) on the G2 job stacked into one GEMM: m = runs*256,
k = n = 4096 -- the library-GEMM reference point for the grouped checked launch. usage: cublas_stacked.py [runs]"""
import sys

import torch

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 250
m, n, k = runs * 256, 4096, 4096
a = torch.randint(-128, 128, (m, k), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device="cuda")
for _ in range(3):
    c = torch._int_mm(a, b)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c = torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
print(f"cuBLAS int8 stacked m={m} n={n} k={k}: {ms:.3f} ms -> {2 * m * n * k / ms / 1e9:.1f} TOPS "
      f"({ms * 1e3 / runs:.2f} us per 256-row run)")
