"""Host-launch vs CUDA-graph throughput of the G2 job, plus cuBLAS int8 (torch._int_mm) at the same shape.
usage: job_probe.py [M N K] [jobs]"""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (256, 4096, 4096)
JOB = int(sys.argv[4]) if len(sys.argv) > 4 else 1000
dev = torch.device("cuda")
s = torch.cuda.Stream()
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
with torch.cuda.stream(s):
    st = C.c_void_p(s.cuda_stream)
    b = torch.randint(-128, 128, (K, N), dtype=torch.int32, device=dev).to(torch.int8)
    w = C.c_void_p()
    L.call("abftlp_gemm_encode", vp(b), K, N, N, st, C.byref(w))
    a_pool = torch.randint(0, 256, (JOB, M, K), dtype=torch.int32, device=dev).to(torch.uint8)
    c_ring = torch.empty((8, M, N), dtype=torch.int32, device=dev)
    csum = torch.empty((JOB, M), dtype=torch.int32, device=dev)
    flags = torch.empty((JOB, M), dtype=torch.uint8, device=dev)
    errs = torch.zeros(JOB, dtype=torch.int32, device=dev)


def job(st, checked=True):
    for i in range(JOB):
        if checked:
            L.call("abftlp_gemm_checked", vp(a_pool[i]), M, K, w, vp(c_ring[i % 8]), N, vp(csum[i]), 1,
                   vp(flags[i]), vp(errs[i:i + 1]), None, st)
        else:
            L.call("abftlp_gemm_unchecked", vp(a_pool[i]), M, K, w, vp(c_ring[i % 8]), N, st)


def timeit(fn, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        out.append((e0.elapsed_time(e1) * 1e3 / JOB, (time.perf_counter() - t0) * 1e6 / JOB))
    return min(out)


with torch.cuda.stream(s):
    for ck in (True, False):
        job(st, ck)
        dev_us, host_us = timeit(lambda: job(st, ck))
        print(f"direct  checked={int(ck)}: {dev_us:.2f} us/GEMM (device), host loop {host_us:.2f} us/GEMM")
graphs = {}
for ck in (True, False):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        job(C.c_void_p(s.cuda_stream), ck)
    graphs[ck] = g
    with torch.cuda.stream(s):
        dev_us, _ = timeit(g.replay)
    print(f"graph   checked={int(ck)}: {dev_us:.2f} us/GEMM  -> {2*M*N*K/dev_us/1e6:.1f} TOPS")
# parity spot check: graph output equals a direct call
torch.cuda.synchronize()
print("errs nonzero after graph:", int((errs != 0).sum().item()))
# cuBLAS int8 reference point (s8 x s8 -> s32)
a8 = torch.randint(-128, 128, (M, K), dtype=torch.int32, device=dev).to(torch.int8)
with torch.cuda.stream(s):
    for _ in range(3):
        torch._int_mm(a8, b)

    def cub():
        for _ in range(JOB):
            torch._int_mm(a8, b)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=s):
        cub()
    dev_us, _ = timeit(g2.replay)
print(f"cuBLAS _int_mm graph: {dev_us:.2f} us/GEMM -> {2*M*N*K/dev_us/1e6:.1f} TOPS")
