"""The 28 DLRM GEMM shapes of P:data/shapes.txt: checked and unchecked time per GEMM (CUDA graph of 50
back-to-back launches), ABFT overhead, on the default dispatch (GEMV class for m <= 16).
usage: shapes_sweep.py [out.json]"""
import ctypes as C
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

NK = [(256, 256), (800, 800), (1024, 1024), (3200, 3200), (800, 3200), (3200, 800), (1024, 256)]
SHAPES = [(m, n, k) for m in (1, 8, 32, 64) for n, k in NK]
REPS = 50
NB = int(os.environ.get("NB", "32"))  # requests per batched launch (serving mode)
dev = torch.device("cuda")
s = torch.cuda.Stream()
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
rows = []
for m, n, k in SHAPES:
    with torch.cuda.stream(s):
        st = C.c_void_p(s.cuda_stream)
        a = torch.randint(0, 256, (m, k), dtype=torch.int32, device=dev).to(torch.uint8)
        b = torch.randint(-128, 128, (k, n), dtype=torch.int32, device=dev).to(torch.int8)
        w = C.c_void_p()
        L.call("abftlp_gemm_encode", vp(b), k, n, n, st, C.byref(w))
        c = torch.empty((m, n + 1), dtype=torch.int32, device=dev)
        fl = torch.empty(m, dtype=torch.uint8, device=dev)
        er = torch.empty(1, dtype=torch.int32, device=dev)

        def run(checked):
            for _ in range(REPS):
                if checked:
                    L.call("abftlp_gemm_checked", vp(a), m, k, w, vp(c), n + 1, C.c_void_p(c.data_ptr() + 4 * n), n + 1,
                           vp(fl), vp(er), None, st)
                else:
                    L.call("abftlp_gemm_unchecked", vp(a), m, k, w, vp(c), n + 1, st)
        run(True)
        run(False)
    res = {}
    graphs = {}
    for ck in (True, False):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            run(ck)
        graphs[ck] = g
    ts = {True: [], False: []}
    with torch.cuda.stream(s):
        for ck in (True, False):
            graphs[ck].replay()
        torch.cuda.synchronize()
        for _ in range(9):  # interleaved checked / unchecked measurements, median of each
            for ck in (True, False):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                graphs[ck].replay()
                e1.record(s)
                torch.cuda.synchronize()
                ts[ck].append(e0.elapsed_time(e1) * 1e3 / REPS)
    for ck in (True, False):
        res[ck] = statistics.median(ts[ck])
    # Serving mode: NB independent requests of this shape against the one encoded weight in ONE launch
    # (abftlp_gemm_checked_batched / _unchecked_batched; C' 16-byte aligned, checksum column separate), graphs of 10
    with torch.cuda.stream(s):
        ab = torch.randint(0, 256, (NB, m, k), dtype=torch.int32, device=dev).to(torch.uint8)
        cb = torch.empty((NB, m, n), dtype=torch.int32, device=dev)
        csb = torch.empty((NB, m), dtype=torch.int32, device=dev)
        flb = torch.empty((NB, m), dtype=torch.uint8, device=dev)
        erb = torch.empty(NB, dtype=torch.int32, device=dev)

        def runb(checked):
            for _ in range(10):
                if checked:
                    L.call("abftlp_gemm_checked_batched", vp(ab), NB, m, k, m * k, w, vp(cb), n, m * n, vp(csb), 1, m,
                           vp(flb), m, vp(erb), None, st)
                else:
                    L.call("abftlp_gemm_unchecked_batched", vp(ab), NB, m, k, m * k, w, vp(cb), n, m * n, st)
        runb(True)
        runb(False)
        torch.cuda.synchronize()
        assert int(erb.sum().item()) == 0
    gb = {}
    for ck in (True, False):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            runb(ck)
        gb[ck] = g
    tb = {True: [], False: []}
    with torch.cuda.stream(s):
        for ck in (True, False):
            gb[ck].replay()
        torch.cuda.synchronize()
        for _ in range(9):
            for ck in (True, False):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                gb[ck].replay()
                e1.record(s)
                torch.cuda.synchronize()
                tb[ck].append(e0.elapsed_time(e1) * 1e3 / 10 / NB)
    bres = {ck: statistics.median(tb[ck]) for ck in (True, False)}
    L.lib.abftlp_gemm_weight_free(w)
    ov = 100 * (res[True] - res[False]) / res[False]
    ovb = 100 * (bres[True] - bres[False]) / bres[False]
    rows.append({"m": m, "n": n, "k": k, "checked_us": res[True], "unchecked_us": res[False], "overhead_pct": ov,
                 "checked_tops": 2 * m * n * k / (res[True] * 1e-6) / 1e12,
                 "weight_gbs": k * n / (res[True] * 1e-6) / 1e9,
                 "batched_requests": NB, "batched_checked_us_per_request": bres[True],
                 "batched_unchecked_us_per_request": bres[False], "batched_overhead_pct": ovb})
    print(f"{m:3d}x{n:5d}x{k:5d}: checked {res[True]:7.2f} us  unchecked {res[False]:7.2f} us  overhead {ov:6.1f}%  "
          f"B' stream {k * n / (res[True] * 1e-6) / 1e9:7.1f} GB/s | {NB} requests per launch: checked "
          f"{bres[True]:6.3f} us/request  unchecked {bres[False]:6.3f}  overhead {ovb:6.1f}%", flush=True)
ovs = [r["overhead_pct"] for r in rows]
print(f"ABFT overhead over the 28 shapes: median {statistics.median(ovs):.1f}%, max {max(ovs):.1f}%, "
      f"{sum(o < 20 for o in ovs)}/28 below 20%")
ovb = [r["batched_overhead_pct"] for r in rows]
print(f"ABFT overhead, {NB} requests per launch: median {statistics.median(ovb):.1f}%, max {max(ovb):.1f}%, "
      f"{sum(o < 20 for o in ovb)}/28 below 20%")
if len(sys.argv) > 1:
    json.dump({"shapes": rows, "overhead_median_pct": statistics.median(ovs), "overhead_max_pct": max(ovs),
               "batched_overhead_median_pct": statistics.median(ovb), "batched_overhead_max_pct": max(ovb)},
              open(sys.argv[1], "w"), indent=1)
