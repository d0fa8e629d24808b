"""G2 job as grouped launches: chunks of `chunk` problems share the one encoded weight and run in ONE
abftlp_gemm_checked_batched launch each (BN forced through ABFTLP_GEMM_TILING), vs the per-GEMM graph.
usage: grouped_probe.py [jobs] [chunk ...]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

M, N, K = 256, 4096, 4096
JOB = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
CHUNKS = [int(x) for x in sys.argv[2:]] or [50, 100, 250]
OPS = 2 * M * N * K
dev = torch.device("cuda")
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
st = C.c_void_p(s.cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
b = torch.empty((K, N), dtype=torch.int8, device=dev)
L.call("abftlp_generate", vp(b), K * N, 20260823, 1000, 0, 1, 0.0, 0.0, 0, st)
w = C.c_void_p()
L.call("abftlp_gemm_encode", vp(b), K, N, N, st, C.byref(w))
a_pool = torch.empty((JOB, M, K), dtype=torch.uint8, device=dev)
L.call("abftlp_generate", vp(a_pool), JOB * M * K, 20260823, 0, 0, 0, 0.0, 0.0, 0, st)
c_all = torch.empty((JOB, M, N), dtype=torch.int32, device=dev)
csum = torch.empty((JOB, M), dtype=torch.int32, device=dev)
flags = torch.empty((JOB, M), dtype=torch.uint8, device=dev)
errs = torch.zeros(JOB, dtype=torch.int32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def grouped(chunk, checked=True):
    for i0 in range(0, JOB, chunk):
        nb = min(chunk, JOB - i0)
        if checked:
            L.call("abftlp_gemm_checked_batched", vp(a_pool[i0]), nb, M, K, M * K, w, vp(c_all[i0]), N, M * N,
                   vp(csum[i0]), 1, M, vp(flags[i0]), M, vp(errs[i0:]), None, st)
        else:
            L.call("abftlp_gemm_unchecked_batched", vp(a_pool[i0]), nb, M, K, M * K, w, vp(c_all[i0]), N, M * N, st)


def timeit(fn, reps=3):
    out = []
    for r in range(reps):
        L.call("abftlp_l2_flush", vp(flush), flush.numel(), r, st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3)
    return min(out)


ref = None
for tiling in (os.environ.get("TILINGS", "256 128").split()):
    os.environ["ABFTLP_GEMM_TILING"] = tiling
    for chunk in CHUNKS:
        for ck in (True, False):
            grouped(chunk, ck)
            us = timeit(lambda: grouped(chunk, ck))
            print(f"bn={tiling} chunk={chunk} checked={int(ck)}: {us/1e3:.3f} ms/job {us/JOB:.2f} us/GEMM "
                  f"{JOB*OPS/us/1e6:.1f} TOPS", flush=True)
        torch.cuda.synchronize()
        e = errs.cpu()
        snap = c_all[::97].clone()
        if ref is None:
            ref = snap
        print(f"   errs flagged={int((e != 0).sum())} same_C={bool(torch.equal(ref, snap))}", flush=True)
# parity of a grouped problem against the single-GEMM call
os.environ.pop("ABFTLP_GEMM_TILING")
c1 = torch.empty((M, N), dtype=torch.int32, device=dev)
cs1 = torch.empty(M, dtype=torch.int32, device=dev)
f1 = torch.empty(M, dtype=torch.uint8, device=dev)
e1 = torch.zeros(1, dtype=torch.int32, device=dev)
L.call("abftlp_gemm_checked", vp(a_pool[5]), M, K, w, vp(c1), N, vp(cs1), 1, vp(f1), vp(e1), None, st)
torch.cuda.synchronize()
print("single==grouped:", bool(torch.equal(c1, c_all[5])), bool(torch.equal(cs1, csum[5])))
