"""D5 MLP probe: the 9 layers (m=8192, (k, n/G)) as one grouped launch vs 9 launches, at G = 1 and 8, each forced tile
width. usage: mlp_probe.py"""
import ctypes as C
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
st = C.c_void_p(s.cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
m = 8192


def gus(fn, reps=8):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


for G in (1, 8):
    mlp = []
    for k in (512, 1024, 2048):
        for n in (512 // G, 1024 // G, 2048 // G):
            b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device=dev)
            a = torch.randint(0, 256, (m, k), dtype=torch.uint8, device=dev)
            w = C.c_void_p()
            L.call("abftlp_gemm_encode", vp(b), k, n, n, st, C.byref(w))
            mlp.append((k, n, w, a, torch.empty((m, n), dtype=torch.int32, device=dev), torch.empty(m, dtype=torch.int32, device=dev),
                        torch.empty(m, dtype=torch.uint8, device=dev), torch.zeros(1, dtype=torch.int32, device=dev)))
    alg = sum(m * k + 4 * m * (n + 1) for k, n, *_ in mlp)
    probs = (L.GemmProblem * 9)()
    for q, (k, n, w, a, c, cs, fl, er) in enumerate(mlp):
        probs[q] = L.GemmProblem(a.data_ptr(), m, k, w.value, c.data_ptr(), n, cs.data_ptr(), 1, fl.data_ptr(), er.data_ptr())
    res = {}
    os.environ["ABFTLP_GEMM_GROUP_APF"] = "0"
    grp = C.c_void_p()
    L.call("abftlp_gemm_group_create", probs, 9, 1, C.byref(grp))
    res["auto no-prefetch"] = gus(lambda: L.call("abftlp_gemm_group_run", grp, st))
    L.lib.abftlp_gemm_group_free(grp)
    os.environ.pop("ABFTLP_GEMM_GROUP_APF")
    for bn in ("auto", "64", "128", "256"):
        os.environ.pop("ABFTLP_GEMM_GROUP_EPI", None)
        if "/" in bn:
            os.environ["ABFTLP_GEMM_GROUP_EPI"] = "1" if bn.endswith("stg") else "2"
        if bn.startswith("auto"):
            os.environ.pop("ABFTLP_GEMM_GROUP_BN", None)
        else:
            os.environ["ABFTLP_GEMM_GROUP_BN"] = bn.split("/")[0]
        grp = C.c_void_p()
        L.call("abftlp_gemm_group_create", probs, 9, 1, C.byref(grp))
        res[bn] = gus(lambda: L.call("abftlp_gemm_group_run", grp, st))
        L.lib.abftlp_gemm_group_free(grp)
    os.environ.pop("ABFTLP_GEMM_GROUP_BN", None)
    os.environ.pop("ABFTLP_GEMM_GROUP_EPI", None)
    grp = C.c_void_p()
    L.call("abftlp_gemm_group_create", probs, 9, 0, C.byref(grp))
    res["unchecked auto"] = gus(lambda: L.call("abftlp_gemm_group_run", grp, st))
    L.lib.abftlp_gemm_group_free(grp)

    def sep():
        for k, n, w, a, c, cs, fl, er in mlp:
            L.call("abftlp_gemm_checked", vp(a), m, k, w, vp(c), n, vp(cs), 1, vp(fl), vp(er), None, st)
    res["9 launches"] = gus(sep)
    print(f"G={G}: alg {alg/1e6:.1f} MB, HBM roof {alg / 6548e3:.1f} us; " + ", ".join(f"{k}: {v:.1f} us" for k, v in res.items()), flush=True)
