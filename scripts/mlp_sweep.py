"""D5 MLP shapes (m=8192, k in {512,1024,2048}, n/8 in {64,128,256}): per-GEMM time of the checked GEMM for
each tiling (CUDA graph of 20 launches, distinct A per launch). usage: mlp_sweep.py"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
st = C.c_void_p(s.cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
m, R = 8192, 20
tilings = sys.argv[1:] or ["auto", "64", "128", "256", "64,0,2", "128,0,2"]
for k in (512, 1024, 2048):
    for n in (64, 128, 256):
        b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device=dev)
        w = C.c_void_p()
        L.call("abftlp_gemm_encode", vp(b), k, n, n, st, C.byref(w))
        a = torch.randint(0, 256, (R, m, k), dtype=torch.int32, device=dev).to(torch.uint8)
        c = torch.empty((m, n), dtype=torch.int32, device=dev)
        cs = torch.empty(m, dtype=torch.int32, device=dev)
        fl = torch.empty(m, dtype=torch.uint8, device=dev)
        er = torch.empty(1, dtype=torch.int32, device=dev)
        res = []
        for t in tilings:
            if t == "auto":
                os.environ.pop("ABFTLP_GEMM_TILING", None)
            else:
                os.environ["ABFTLP_GEMM_TILING"] = t

            def run():
                for i in range(R):
                    L.call("abftlp_gemm_checked", vp(a[i]), m, k, w, vp(c), n, vp(cs), 1, vp(fl), vp(er), None, st)
            run()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                run()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / R
            res.append(f"{t}:{us:.1f}")
        roof = max(2 * m * n * k / 3.3e15, (m * k + 4 * m * n) / 6.5e12) * 1e6
        print(f"k={k} n={n}: " + " ".join(res) + f"   roof {roof:.1f} us", flush=True)
        L.lib.abftlp_gemm_weight_free(w)
