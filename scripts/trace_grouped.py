"""Steady-state tile timeline of the grouped G2 launch (build with -DABFT_TRACE_STEADY): for each CTA's 9th tile,
the epilogue's duration (accumulator ready -> chunks written) and how long the MMA waited for a free accumulator.
usage: ABFTLP_B200_LIB=... trace_grouped.py [tiling]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

if len(sys.argv) > 1:
    os.environ["ABFTLP_GEMM_TILING"] = sys.argv[1]
M, N, K, nb = 256, 4096, 4096, 200
dev = torch.device("cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
b = torch.randint(-128, 128, (K, N), dtype=torch.int32, device=dev).to(torch.int8)
w = C.c_void_p()
L.call("abftlp_gemm_encode", vp(b), K, N, N, st, C.byref(w))
a = torch.randint(0, 256, (nb, M, K), dtype=torch.int32, device=dev).to(torch.uint8)
c = torch.empty((nb, M, N), dtype=torch.int32, device=dev)
cs = torch.empty((nb, M), dtype=torch.int32, device=dev)
fl = torch.empty((nb, M), dtype=torch.uint8, device=dev)
er = torch.zeros(nb, dtype=torch.int32, device=dev)
tr = torch.zeros(16 * 4096, dtype=torch.int64, device=dev)
L.lib.abftlp_debug_gemm_trace.argtypes = [C.c_void_p]


def run():
    L.call("abftlp_gemm_checked_batched", vp(a), nb, M, K, M * K, w, vp(c), N, M * N, vp(cs), 1, M, vp(fl), M, vp(er),
           None, st)


for _ in range(2):
    run()
tr.zero_()
L.lib.abftlp_debug_gemm_trace(vp(tr))
run()
L.lib.abftlp_debug_gemm_trace(None)
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(-1, 16)
t = t[(t[:, 9] > 0) & (t[:, 10] > 0)]
epi = (t[:, 10] - t[:, 9]) / 1000.0
gap = (t[:, 13] - t[:, 9]) / 1000.0
ok = (t[:, 11] > 0) & (t[:, 12] > 0)
wait = (t[ok, 12] - t[ok, 11]) / 1000.0
print(f"CTAs {len(t)}: tile-8 epilogue (acc ready -> chunks written) med {np.median(epi):.2f} p90 {np.percentile(epi, 90):.2f} us; "
      f"tile 8 -> 9 acc-ready interval med {np.median(gap):.2f} us; MMA wait for free accumulator (leaders) "
      f"med {np.median(wait) if len(wait) else float('nan'):.2f} max {wait.max() if len(wait) else float('nan'):.2f} us")
