"""Per-CTA phase timeline of the batched G1 launch (100 problems m=64 k=512 n=512, each its own weight).
usage: trace_g1.py [tiling]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

if len(sys.argv) > 1:
    os.environ["ABFTLP_GEMM_TILING"] = sys.argv[1]
nb, m, n, k = 100, 64, 512, 512
dev = torch.device("cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
a = torch.randint(0, 256, (nb, m, k), dtype=torch.int32, device=dev).to(torch.uint8)
b = torch.randint(-128, 128, (nb, k, n), dtype=torch.int32, device=dev).to(torch.int8)
w = C.c_void_p()
L.call("abftlp_gemm_encode_batched", vp(b), nb, k, n, n, k * n, st, C.byref(w))
c = torch.zeros((nb, m, n + 1), dtype=torch.int32, device=dev)
fl = torch.zeros((nb, m), dtype=torch.uint8, device=dev)
err = torch.zeros(nb, dtype=torch.int32, device=dev)
trace = torch.zeros(16 * 4096, dtype=torch.int64, device=dev)
L.lib.abftlp_debug_gemm_trace.argtypes = [C.c_void_p]


def run():
    L.call("abftlp_gemm_checked_batched", vp(a), nb, m, k, m * k, w, vp(c), n + 1, m * (n + 1),
           C.c_void_p(c.data_ptr() + 4 * n), n + 1, m * (n + 1), vp(fl), m, vp(err), None, st)


for _ in range(3):
    run()
trace.zero_()
L.lib.abftlp_debug_gemm_trace(vp(trace))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
L.lib.abftlp_debug_gemm_trace(None)
torch.cuda.synchronize()
t = trace.cpu().numpy().reshape(-1, 16)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = np.where(t > 0, (t - t0) / 1000.0, np.nan)
print(f"event {e0.elapsed_time(e1)*1e3:.2f} us, ctas {len(t)}")
for i, nm in {0: "start", 1: "setup", 2: "first_kb(L)", 3: "last_issue(L)", 4: "epi_start", 7: "chunks_done",
              8: "cnt_done", 5: "epi_end", 9: "w0 done*", 10: "w1 done*", 11: "w6 done*", 12: "w7 done*",
              6: "end"}.items():  # * only with -DABFT_TRACE_ROLES
    col = rel[:, i]
    if np.all(np.isnan(col)):
        continue
    print(f"  {nm:14s} min {np.nanmin(col):7.2f}  med {np.nanmedian(col):7.2f}  max {np.nanmax(col):7.2f}")
