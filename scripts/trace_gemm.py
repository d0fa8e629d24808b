"""Per-CTA phase timeline of the GEMM kernel (debug instrumentation, abftlp_debug_gemm_trace).
usage: trace_gemm.py M N K [checked] [tiling] [flush]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
checked = int(sys.argv[4]) if len(sys.argv) > 4 else 1
if len(sys.argv) > 5 and sys.argv[5] != "-":
    os.environ["ABFTLP_GEMM_TILING"] = sys.argv[5]
flush = int(sys.argv[6]) if len(sys.argv) > 6 else 1
dev = torch.device("cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
a = torch.randint(0, 256, (m, k), dtype=torch.int32, device=dev).to(torch.uint8)
b = torch.randint(-128, 128, (k, n), dtype=torch.int32, device=dev).to(torch.int8)
w = C.c_void_p()
L.call("abftlp_gemm_encode", vp(b), k, n, n, st, C.byref(w))
c = torch.zeros((m, n), dtype=torch.int32, device=dev)
cs = torch.zeros(m, dtype=torch.int32, device=dev)
fl = torch.zeros(m, dtype=torch.uint8, device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
fb = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
trace = torch.zeros(16 * 4096, dtype=torch.int64, device=dev)
L.lib.abftlp_debug_gemm_trace.argtypes = [C.c_void_p]


def run():
    if checked:
        L.call("abftlp_gemm_checked", vp(a), m, k, w, vp(c), n, vp(cs), 1, vp(fl), vp(err), None, st)
    else:
        L.call("abftlp_gemm_unchecked", vp(a), m, k, w, vp(c), n, st)


for _ in range(3):
    run()
for rep in range(3):
    if flush:
        L.call("abftlp_l2_flush", vp(fb), fb.numel(), rep, st)
    trace.zero_()
    L.lib.abftlp_debug_gemm_trace(vp(trace))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    L.lib.abftlp_debug_gemm_trace(None)
    torch.cuda.synchronize()
    t = trace.cpu().numpy().reshape(-1, 16)
    valid = t[:, 0] > 0
    t = t[valid]
    t0 = t[:, 0].min()
    rel = np.where(t > 0, (t - t0) / 1000.0, np.nan)
    names = {0: "start", 1: "setup", 2: "first_kb(L)", 9: "kb1", 10: "kb2", 11: "kb3", 3: "last_issue(L)",
             4: "epi_start", 14: "split: published / c0 loaded", 12: "split: flag seen / c0 start", 13: "split: partial in / c1 start", 7: "chunks_done",
             8: "cnt_done", 5: "epi_end", 6: "end"}
    print(f"rep {rep}: event {e0.elapsed_time(e1)*1e3:.2f} us, ctas {len(t)}, span {np.nanmax(rel[:, 6]):.2f} us")
    for i, nm in names.items():
        col = rel[:, i]
        if np.all(np.isnan(col)):
            continue
        print(f"  {nm:14s} min {np.nanmin(col):7.2f}  med {np.nanmedian(col):7.2f}  max {np.nanmax(col):7.2f}")
    if len(sys.argv) > 7 and rep == 2:
        order = np.argsort(-np.nan_to_num(rel[:, 6]))
        cols = [0, 1, 2, 3, 4, 7, 8, 5, 6]
        print("  slowest CTAs (block, " + ", ".join(names[c] for c in cols) + ")")
        idx = np.nonzero(valid)[0]
        for r in order[:6]:
            print("   ", idx[r], " ".join(f"{rel[r, c]:7.2f}" for c in cols))
        print("  fastest:", idx[order[-1]], " ".join(f"{rel[order[-1], c]:7.2f}" for c in cols))
