"""Profiling driver for the D5 per-GPU grouped EmbeddingBag launch (8 tables x 1M x 128 int8, batch 8192, pooling
80, Zipf(1.05)) written into an all-to-all send buffer. usage: prof_d5_group.py [iters]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dev = torch.device("cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
T, R, d, B, pool, G = 8, 1_000_000, 128, 8192, 80, 8
Bg = B // G
rng = np.random.default_rng(5)
cdf = np.cumsum(np.arange(1, R + 1, dtype=np.float64) ** -1.05)
cdf /= cdf[-1]
tabs, keep, offs, ixs = [], [], [], []
for t in range(T):
    rows = torch.randint(-128, 128, (R, d), dtype=torch.int8, device=dev)
    sc = torch.rand(R, device=dev) * 9e-3 + 1e-3
    bi = torch.rand(R, device=dev) * 2 - 1
    h = C.c_void_p()
    L.call("abftlp_eb_table_create", 0, vp(rows), R, d, d, 0, vp(sc), vp(bi), None, st, C.byref(h))
    idx = rng.permutation(R)[np.searchsorted(cdf, rng.random(B * pool))].astype(np.int64)
    offs.append(torch.arange(0, B * pool + 1, pool, dtype=torch.int64, device=dev))
    ixs.append(torch.from_numpy(idx).to(dev))
    tabs.append(h)
    keep.append((rows, sc, bi))
send = torch.empty((G, Bg, T, d), dtype=torch.float32, device=dev)
send_f = torch.empty((G, Bg, T), dtype=torch.uint8, device=dev)
dests = [(torch.tensor([send[g, 0, t].data_ptr() for g in range(G)], dtype=torch.int64, device=dev),
          torch.tensor([send_f[g, 0, t:].data_ptr() for g in range(G)], dtype=torch.int64, device=dev)) for t in range(T)]
P = C.c_void_p
grp = C.c_void_p()
L.call("abftlp_eb_group_create", (P * T)(*tabs), T, (P * T)(*[vp(o) for o in offs]), (P * T)(*[vp(i) for i in ixs]), None,
       (P * T)(*[vp(o) for o, _ in dests]), (P * T)(*[vp(f) for _, f in dests]), C.byref(grp))
cnt = torch.zeros(1, dtype=torch.int32, device=dev)
fb = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ts = []
for i in range(iters):
    L.call("abftlp_l2_flush", vp(fb), fb.numel(), i, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.call("abftlp_eb_group_checked_scatter", grp, B, T * d, T, Bg, vp(cnt), None, st)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print("D5 grouped EB us:", [round(t, 1) for t in ts])
