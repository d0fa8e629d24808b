"""How much of a cold single EmbeddingBag launch is launch / reconfiguration latency? (E3 table and bags)
  a) flush -> [e0] E3 [e1]                      (the bench's single-launch protocol)
  b) flush -> EB(one empty bag) -> [e0] E3 [e1]  (the SM's shared-memory carve-out already set by an EB launch)
  c) flush -> [e0] EB(one empty bag) [e1]       (the fixed cost of a launch of this kernel after the flush)
  d) [e0] EB(one empty bag) [e1] back to back    (fixed cost without the flush before it)"""
import ctypes as C
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
rng = np.random.default_rng(3)
R, d, nb = 4_000_000, 128, 2048
lens = rng.integers(20, 101, nb)
ranks = np.arange(1, R + 1, dtype=np.float64)
cdf = np.cumsum(ranks ** -1.05)
cdf /= cdf[-1]
idx = rng.permutation(R)[np.searchsorted(cdf, rng.random(int(lens.sum())))].astype(np.int64)
rows = torch.randint(0, 256, (R, d), dtype=torch.uint8, device=dev)
sc = torch.rand(R, device=dev) * 9e-3 + 1e-3
bi = torch.rand(R, device=dev) * 2 - 1
off = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)).to(dev)
ix = torch.from_numpy(idx).to(dev)
off0 = torch.zeros(2, dtype=torch.int64, device=dev)
tab = C.c_void_p()
L.call("abftlp_eb_table_create", 1, vp(rows), R, d, d, 0, vp(sc), vp(bi), None, st, C.byref(tab))
o = torch.empty((nb, d), dtype=torch.float32, device=dev)
fl = torch.empty(nb, dtype=torch.uint8, device=dev)
fb = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def eb(n, offs):
    L.call("abftlp_eb_checked", tab, vp(offs), vp(ix), n, None, vp(o), d, vp(fl), None, None, None, None, st)


def run(pre, body, flush=True, reps=8):
    ts = []
    for i in range(reps):
        if flush:
            L.call("abftlp_l2_flush", vp(fb), fb.numel(), i, st)
        pre()
        torch.cuda._sleep(1_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        body()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return round(statistics.median(ts[2:]), 2)


nop = lambda: None  # noqa: E731
print("a) flush -> E3                 :", run(nop, lambda: eb(nb, off)))
print("b) flush -> EB(empty) -> E3     :", run(lambda: eb(1, off0), lambda: eb(nb, off)))
print("c) flush -> EB(empty)           :", run(nop, lambda: eb(1, off0)))
print("d) EB(empty), no flush          :", run(nop, lambda: eb(1, off0), flush=False))
print("e) E3, no flush (L2 warm)       :", run(nop, lambda: eb(nb, off), flush=False))
z = torch.zeros(1, device=dev)
print("f) torch tiny kernel            :", run(nop, lambda: z.add_(1), flush=False))
print("g) EB(empty) x2                 :", run(nop, lambda: (eb(1, off0), eb(1, off0)), flush=False))
print("h) E3 x2                        :", run(nop, lambda: (eb(nb, off), eb(nb, off)), flush=False))
gat = torch.zeros(1, dtype=torch.int32, device=dev)
print("i) gather probe (E3 rows)       :", run(nop, lambda: L.call("abftlp_gather_probe", vp(rows), 128, vp(ix), int(lens.sum()), vp(gat), st)))
print("j) gather probe 1 row           :", run(nop, lambda: L.call("abftlp_gather_probe", vp(rows), 128, vp(ix), 1, vp(gat), st), flush=False))
