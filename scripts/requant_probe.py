"""Device time of the fused-requantization checked GEMM on the G2 shape, row-stacked (8 runs = 2048 rows per launch,
as abftlp_gemm_checked_requant_host_batched issues it), with and without the int32 C' write, vs the plain checked
GEMM. usage: requant_probe.py"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
R, M, K, N = 8, 256, 4096, 4096
a = torch.randint(0, 256, (R * M, K), dtype=torch.int32, device=dev).to(torch.uint8)
b = torch.randint(-128, 128, (K, N), dtype=torch.int32, device=dev).to(torch.int8)
w = C.c_void_p()
L.call("abftlp_gemm_encode", vp(b), K, N, N, st, C.byref(w))
c = torch.empty((R * M, N), dtype=torch.int32, device=dev)
o = torch.empty((R * M, N), dtype=torch.uint8, device=dev)
cs = torch.empty(R * M, dtype=torch.int32, device=dev)
fl = torch.empty(R * M, dtype=torch.uint8, device=dev)
er = torch.zeros(1, dtype=torch.int32, device=dev)
rs = torch.empty(R * M, dtype=torch.int32, device=dev)
col = torch.empty(N, dtype=torch.int32, device=dev)
L.call("abftlp_gemm_weight_col_sums", w, vp(col), st)
rqp = L.RequantParams(0.02, -0.3, 0.01, 0.1, 37.0, -5.0, K)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


plain = timed(lambda: L.call("abftlp_gemm_checked", vp(a), R * M, K, w, vp(c), N, vp(cs), 1, vp(fl), vp(er), None, st))
rsum = timed(lambda: L.call("abftlp_row_sums_u8", vp(a), R * M, K, K, vp(rs), st))
rq_c = timed(lambda: L.call("abftlp_gemm_checked_requant", vp(a), R * M, K, w, vp(c), N, vp(cs), 1, vp(fl), vp(er), None,
                            vp(rs), vp(col), C.byref(rqp), vp(o), N, st))
rq = timed(lambda: L.call("abftlp_gemm_checked_requant", vp(a), R * M, K, w, None, N, vp(cs), 1, vp(fl), vp(er), None,
                          vp(rs), vp(col), C.byref(rqp), vp(o), N, st))
print(f"{R} runs per launch (m = {R * M}): checked {plain:.1f} us, row sums {rsum:.1f} us, "
      f"checked + requant (C' kept) {rq_c:.1f} us, checked + requant (u8 only) {rq:.1f} us "
      f"= {rq / R:.2f} us per run, {R * 2 * M * K * N / rq / 1e6:.0f} TOPS")
