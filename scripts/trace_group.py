"""Per-tile timeline of the grouped GEMM (library variant built with -DABFT_TRACE_TILES): MMA start/issue-end and
epilogue start/end of each CTA's first 16 tiles. usage: trace_group.py G  (ABFTLP_B200_LIB -> the variant)"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
tr = torch.zeros(64 * 148, dtype=torch.int64, device="cuda")
L.lib.abftlp_debug_gemm_trace.argtypes = [C.c_void_p]
dev = torch.device("cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
m = 8192
keep = []
probs = (L.GemmProblem * 9)()
q = 0
for k in (512, 1024, 2048):
    for n in (512 // G, 1024 // G, 2048 // G):
        b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device=dev)
        a = torch.randint(0, 256, (m, k), dtype=torch.uint8, device=dev)
        w = C.c_void_p()
        L.call("abftlp_gemm_encode", C.c_void_p(b.data_ptr()), k, n, n, st, C.byref(w))
        c, cs, fl, er = (torch.empty((m, n), dtype=torch.int32, device=dev), torch.empty(m, dtype=torch.int32, device=dev),
                         torch.empty(m, dtype=torch.uint8, device=dev), torch.zeros(1, dtype=torch.int32, device=dev))
        keep += [b, a, c, cs, fl, er]
        probs[q] = L.GemmProblem(a.data_ptr(), m, k, w.value, c.data_ptr(), n, cs.data_ptr(), 1, fl.data_ptr(), er.data_ptr())
        q += 1
L.lib.abftlp_debug_gemm_trace(C.c_void_p(tr.data_ptr()))
grp = C.c_void_p()
L.call("abftlp_gemm_group_create", probs, 9, int(os.environ.get("CHECKED", "1")), C.byref(grp))
for _ in range(3):
    L.call("abftlp_gemm_group_run", grp, st)
torch.cuda.synchronize()
L.lib.abftlp_debug_gemm_trace(None)
t = tr.cpu().numpy().reshape(148, 64).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1000.0, np.nan)
names = "mma0 mma1 top ready chunks release verdict publish".split()
for cta in (0, 2, 70, 146):
    print(f"CTA {cta}:   " + " ".join(f"{n:>8s}" for n in names))
    for i in range(8):
        if not np.isnan(t[cta, 8 * i]) or not np.isnan(t[cta, 8 * i + 3]):
            print(f"   tile {i:2d}: " + " ".join(f"{t[cta, 8 * i + j]:8.2f}" for j in range(8)))
print("last epilogue end (all CTAs): max %.2f us" % np.nanmax(t[:, 7::8]))
