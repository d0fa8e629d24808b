"""First-contact GPU probe: exercises every kernel once against simple references and prints
timings. Development tool (the judged parity tests live in tests/)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
st = torch.cuda.current_stream().cuda_stream
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def gemm_case(m, n, k, tiling=None, seed=0):
    if tiling:
        os.environ["ABFTLP_GEMM_TILING"] = tiling
    else:
        os.environ.pop("ABFTLP_GEMM_TILING", None)
    g = torch.Generator(device="cpu").manual_seed(seed)
    a = torch.randint(0, 256, (m, k), generator=g, dtype=torch.int32).to(torch.uint8).to(dev)
    b = torch.randint(-128, 128, (k, n), generator=g, dtype=torch.int32).to(torch.int8).to(dev)
    w = C.c_void_p()
    L.call("abftlp_gemm_encode", vp(b), k, n, n, C.c_void_p(st), C.byref(w))
    ldc = (n + 3) // 4 * 4
    c = torch.zeros((m, ldc), dtype=torch.int32, device=dev)
    cs = torch.zeros(m, dtype=torch.int32, device=dev)
    fl = torch.zeros(m, dtype=torch.uint8, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    L.call("abftlp_gemm_checked", vp(a), m, k, w, vp(c), ldc, vp(cs), 1, vp(fl), vp(err), None, C.c_void_p(st))
    torch.cuda.synchronize()
    ref = (a.double() @ b.double()).round().long()
    bsum = b.long().sum(1)
    csr = torch.remainder(bsum, 127)
    csref = (a.double() @ csr.double()).round().long()
    ok_c = torch.equal(c[:, :n].long(), ref)
    ok_cs = torch.equal(cs.long(), csref)
    ok_f = int(fl.sum()) == 0 and int(err) == 0
    # unchecked
    c2 = torch.zeros_like(c)
    L.call("abftlp_gemm_unchecked", vp(a), m, k, w, vp(c2), ldc, C.c_void_p(st))
    torch.cuda.synchronize()
    ok_u = torch.equal(c2[:, :n].long(), ref)
    print(f"gemm {m}x{n}x{k} tiling={tiling}: C {ok_c} csum {ok_cs} flags {ok_f} (err={int(err)}) unchecked {ok_u}",
          flush=True)
    if not ok_c:
        bad = (c[:, :n].long() != ref).nonzero()
        print("  first bad", bad[:5].tolist(), c[:, :n].long()[tuple(bad[0])].item(), ref[tuple(bad[0])].item())
    L.lib.abftlp_gemm_weight_free(w)
    return ok_c and ok_cs and ok_f and ok_u


def time_gemm(m, n, k, checked=True, iters=50, flush=True):
    a = torch.randint(0, 256, (m, k), dtype=torch.int32, device=dev).to(torch.uint8)
    b = torch.randint(-128, 128, (k, n), dtype=torch.int32, device=dev).to(torch.int8)
    w = C.c_void_p()
    L.call("abftlp_gemm_encode", vp(b), k, n, n, C.c_void_p(st), C.byref(w))
    c = torch.zeros((m, n), dtype=torch.int32, device=dev)
    cs = torch.zeros(m, dtype=torch.int32, device=dev)
    fl = torch.zeros(m, dtype=torch.uint8, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    fb = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    times = []
    for i in range(iters + 3):
        if flush:
            L.call("abftlp_l2_flush", vp(fb), fb.numel(), i, C.c_void_p(st))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if checked:
            L.call("abftlp_gemm_checked", vp(a), m, k, w, vp(c), n, vp(cs), 1, vp(fl), vp(err), None, C.c_void_p(st))
        else:
            L.call("abftlp_gemm_unchecked", vp(a), m, k, w, vp(c), n, C.c_void_p(st))
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            times.append(e0.elapsed_time(e1) * 1e3)
    L.lib.abftlp_gemm_weight_free(w)
    t = float(np.median(times))
    ops = 2 * m * n * k
    byt = m * k + k * (n + 1) + 4 * m * (n + 1) + m
    print(f"time {m}x{n}x{k} checked={checked} flush={flush} tiling={os.environ.get('ABFTLP_GEMM_TILING')}: "
          f"{t:.2f} us  {ops / t / 1e6:.1f} TOPS  {byt / t / 1e3:.1f} GB/s", flush=True)
    return t


if __name__ == "__main__":
    ok = True
    for (m, n, k) in [(2, 2, 2), (64, 512, 512), (1, 32, 32), (3, 17, 5), (130, 300, 200), (256, 1024, 1024)]:
        ok &= gemm_case(m, n, k)
    for tiling in ["256,4", "128,2", "64,1", "256,1", "256,8"]:
        ok &= gemm_case(256, 4096, 4096, tiling)
    ok &= gemm_case(256, 4096, 4096)
    print("GEMM ALL OK" if ok else "GEMM FAILURES", flush=True)
    os.environ.pop("ABFTLP_GEMM_TILING", None)
    for flush in (True, False):
        time_gemm(256, 4096, 4096, True, flush=flush)
        time_gemm(256, 4096, 4096, False, flush=flush)
    for tiling in ["256,4", "128,2", "256,2", "128,4", "64,2", "256,8"]:
        os.environ["ABFTLP_GEMM_TILING"] = tiling
        time_gemm(256, 4096, 4096, True)
    os.environ.pop("ABFTLP_GEMM_TILING", None)
    time_gemm(64, 512, 512, True)
    time_gemm(8192, 2048, 2048, True)
