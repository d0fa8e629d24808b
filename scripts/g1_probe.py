"""G1 (BASELINE configs[0]): 100 seeded checked GEMMs m=64 k=512 n=512 -- one batched launch vs 100 launches."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

nb, m, n, k = 100, 64, 512, 512
dev = torch.device("cuda")
s = torch.cuda.Stream()
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
with torch.cuda.stream(s):
    st = C.c_void_p(s.cuda_stream)
    a = torch.randint(0, 256, (nb, m, k), dtype=torch.int32, device=dev).to(torch.uint8)
    b = torch.randint(-128, 128, (nb, k, n), dtype=torch.int32, device=dev).to(torch.int8)
    wb = C.c_void_p()
    L.call("abftlp_gemm_encode_batched", vp(b), nb, k, n, n, k * n, st, C.byref(wb))
    ws = []
    for t in range(nb):
        w = C.c_void_p()
        L.call("abftlp_gemm_encode", vp(b[t]), k, n, n, st, C.byref(w))
        ws.append(w)
    c = torch.empty((nb, m, n + 1), dtype=torch.int32, device=dev)
    fl = torch.empty((nb, m), dtype=torch.uint8, device=dev)
    err = torch.empty(nb, dtype=torch.int32, device=dev)

    def batched():
        L.call("abftlp_gemm_checked_batched", vp(a), nb, m, k, m * k, wb, vp(c), n + 1, m * (n + 1),
               C.c_void_p(c.data_ptr() + 4 * n), n + 1, m * (n + 1), vp(fl), m, vp(err), None, st)

    c2 = torch.empty((nb, m, n), dtype=torch.int32, device=dev)  # aligned C (TMA epilogue), csum separate
    cs2 = torch.empty((nb, m), dtype=torch.int32, device=dev)

    def batched_aligned():
        L.call("abftlp_gemm_checked_batched", vp(a), nb, m, k, m * k, wb, vp(c2), n, m * n, vp(cs2), 1, m, vp(fl), m,
               vp(err), None, st)

    def separate():
        for t in range(nb):
            L.call("abftlp_gemm_checked", vp(a[t]), m, k, ws[t], vp(c[t]), n + 1, C.c_void_p(c[t].data_ptr() + 4 * n),
                   n + 1, vp(fl[t]), vp(err[t:t + 1]), None, st)

    batched()
    batched_aligned()
    separate()
graphs = {}
for name, fn in (("batched", batched), ("batched_aligned_C", batched_aligned), ("separate", separate)):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    graphs[name] = g
with torch.cuda.stream(s):
    for name, g in graphs.items():
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(10):
                g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / 10)
        t = sorted(ts)[len(ts) // 2]
        print(f"G1 {name}: {t:.2f} us per 100 trials -> {t / nb:.3f} us/GEMM, {2 * m * n * k * nb / t / 1e6:.1f} TOPS")
