"""Per-tile timeline of a batched launch (library variant built with -DABFT_TRACE_TILES): NB requests of one shape
against one encoded weight. usage: trace_batched.py m n k [NB]   (ABFTLP_B200_LIB -> the variant; CHECKED=0 unchecked)"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
NB = int(sys.argv[4]) if len(sys.argv) > 4 else 128
checked = int(os.environ.get("CHECKED", "1"))
dev = torch.device("cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
a = torch.randint(0, 256, (NB, m, k), dtype=torch.int32, device=dev).to(torch.uint8)
b = torch.randint(-128, 128, (k, n), dtype=torch.int32, device=dev).to(torch.int8)
w = C.c_void_p()
L.call("abftlp_gemm_encode", vp(b), k, n, n, st, C.byref(w))
c = torch.empty((NB, m, n), dtype=torch.int32, device=dev)
cs = torch.empty((NB, m), dtype=torch.int32, device=dev)
fl = torch.empty((NB, m), dtype=torch.uint8, device=dev)
er = torch.empty(NB, dtype=torch.int32, device=dev)
tr = torch.zeros(64 * 148, dtype=torch.int64, device=dev)
L.lib.abftlp_debug_gemm_trace.argtypes = [C.c_void_p]


def run():
    if checked:
        L.call("abftlp_gemm_checked_batched", vp(a), NB, m, k, m * k, w, vp(c), n, m * n, vp(cs), 1, m, vp(fl), m, vp(er),
               None, st)
    else:
        L.call("abftlp_gemm_unchecked_batched", vp(a), NB, m, k, m * k, w, vp(c), n, m * n, st)


for _ in range(3):
    run()
torch.cuda.synchronize()
L.lib.abftlp_debug_gemm_trace(vp(tr))
run()
torch.cuda.synchronize()
L.lib.abftlp_debug_gemm_trace(None)
t = tr.cpu().numpy().reshape(148, 64).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1000.0, np.nan)
names = "mma0 mma1 top ready chunks release verdict publish".split()
for cta in (0, 70):
    print(f"CTA {cta}:   " + " ".join(f"{x:>8s}" for x in names))
    for i in range(8):
        if not np.isnan(t[cta, 8 * i]) or not np.isnan(t[cta, 8 * i + 3]):
            print(f"   tile {i:2d}: " + " ".join(f"{t[cta, 8 * i + j]:8.2f}" for j in range(8)))
print("last stamp (all CTAs): max %.2f us" % np.nanmax(t))
