"""Profiling driver for the EmbeddingBag kernel. usage: prof_eb.py E3|E4 [checked=1] [iters=4]"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "E3"
checked = int(sys.argv[2]) if len(sys.argv) > 2 else 1
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 4
dev = torch.device("cuda")
torch.cuda.init()
if os.environ.get("L2FETCH"):  # cudaLimitMaxL2FetchGranularity (0x05) experiment
    import glob
    rt = C.CDLL(sorted(glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*")))[0])
    torch.zeros(1, device=dev)
    r = rt.cudaDeviceSetLimit(5, C.c_size_t(int(os.environ["L2FETCH"])))
    v = C.c_size_t()
    rt.cudaDeviceGetLimit(C.byref(v), 5)
    print("L2 fetch granularity set", r, "->", v.value)
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
rng = np.random.default_rng(3)
if cfg == "D5":  # one table of BASELINE configs[4]: 1M x 128 int8, fp32 scale/bias, 8192 bags x 80, Zipf(1.05)
    R, d, nb, elem, sct = 1_000_000, 128, 8192, 0, 0
    lens = np.full(nb, 80)
    ranks = np.arange(1, R + 1, dtype=np.float64)
    cdf = np.cumsum(ranks ** -1.05)
    cdf /= cdf[-1]
    idx = rng.permutation(R)[np.searchsorted(cdf, rng.random(int(lens.sum())))].astype(np.int64)
    if os.environ.get("UNIFORM"):
        idx = rng.integers(0, R, int(lens.sum())).astype(np.int64)
    w = None
    rb = d
elif cfg == "E3":
    R, d, nb, elem, sct = 4_000_000, 128, 2048, 1, 0
    lens = rng.integers(20, 101, nb)
    ranks = np.arange(1, R + 1, dtype=np.float64)
    cdf = np.cumsum(ranks ** -1.05)
    cdf /= cdf[-1]
    idx = rng.permutation(R)[np.searchsorted(cdf, rng.random(int(lens.sum())))].astype(np.int64)
    w = None
    rb = d
else:
    R, d, nb, elem, sct = 8_000_000, 64, 4096, 2, 1
    lens = rng.integers(1, 151, nb)
    if cfg == "E4sorted":  # the same bags, longest first (scheduling-order probe)
        lens = np.sort(lens)[::-1].copy()
    if cfg == "E4fixed":  # same total lookups, every bag the mean length (load-balance probe)
        lens = np.full(nb, int(round(lens.mean())))
    if cfg == "E4short":  # same total lookups in 4x as many 4x shorter bags
        nb = nb * 4
        lens = np.full(nb, int(round(lens.mean() / 4)))
    if os.environ.get("NBAGS"):  # fixed-cost probe: fewer bags
        nb = int(os.environ["NBAGS"])
        lens = lens[:nb]
    idx = rng.integers(0, R, int(lens.sum())).astype(np.int64)
    if cfg == "E4seq":  # gather cost probe: consecutive rows
        idx = np.arange(int(lens.sum()), dtype=np.int64)
    if cfg == "E4hot":  # L2-resident probe: 64K distinct rows
        idx = rng.integers(0, 65536, int(lens.sum())).astype(np.int64)
    w = torch.from_numpy(rng.uniform(0, 1, int(lens.sum())).astype(np.float32)).to(dev)
    rb = d // 2
rows = torch.randint(0, 256, (R, rb), dtype=torch.uint8, device=dev)
sdt = torch.float32 if sct == 0 else torch.float16
sc = (torch.rand(R, device=dev) * 9e-3 + 1e-3).to(sdt)
bi = (torch.rand(R, device=dev) * 2 - 1).to(sdt)
off = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)).to(dev)
ix = torch.from_numpy(idx).to(dev)
tab = C.c_void_p()
L.call("abftlp_eb_table_create", elem, vp(rows), R, d, rb, sct, vp(sc), vp(bi), None, st, C.byref(tab))
o = torch.empty((nb, d), dtype=torch.float32, device=dev)
fl = torch.empty(nb, dtype=torch.uint8, device=dev)
fb = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ts = []
for i in range(iters):
    L.call("abftlp_l2_flush", vp(fb), fb.numel(), i, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if checked:
        L.call("abftlp_eb_checked", tab, vp(off), vp(ix), nb, vp(w) if w is not None else None, vp(o), d, vp(fl),
               None, None, None, None, st)
    else:
        L.call("abftlp_eb_unchecked", tab, vp(off), vp(ix), nb, vp(w) if w is not None else None, vp(o), d, None, st)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(cfg, "checked" if checked else "unchecked", "us:", [round(t, 1) for t in ts])
# back-to-back launches (no flush in between): per-launch time in a stream of batches
if os.environ.get("B2B"):
    nrep = int(os.environ["B2B"])
    torch.cuda.synchronize()
    torch.cuda._sleep(2_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(nrep):
        if checked:
            L.call("abftlp_eb_checked", tab, vp(off), vp(ix), nb, vp(w) if w is not None else None, vp(o), d, vp(fl),
                   None, None, None, None, st)
        else:
            L.call("abftlp_eb_unchecked", tab, vp(off), vp(ix), nb, vp(w) if w is not None else None, vp(o), d, None, st)
    e1.record()
    torch.cuda.synchronize()
    print(cfg, "back-to-back x%d: %.2f us/launch" % (nrep, e0.elapsed_time(e1) * 1e3 / nrep))
    # single launch queued behind a sleep (host latency excluded), L2 flushed first
    L.call("abftlp_l2_flush", vp(fb), fb.numel(), 99, st)
    torch.cuda._sleep(2_000_000)
    e0.record()
    L.call("abftlp_eb_checked", tab, vp(off), vp(ix), nb, vp(w) if w is not None else None, vp(o), d, vp(fl),
           None, None, None, None, st)
    e1.record()
    torch.cuda.synchronize()
    print(cfg, "queued single after flush: %.2f us" % (e0.elapsed_time(e1) * 1e3))
