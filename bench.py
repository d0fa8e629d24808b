#!/usr/bin/env python3
"""Benchmark driver (one JSON line on rank 0).

Headline workload = BASELINE.json configs[1] ("G2"): checked int8 GEMM m=256, k=4096, n=4096,
A u8 U[0,255], B s8 U[-128,127] (SplitMix64, the reference's draw protocol), B encoded ONCE and
reused for a job of 1000 GEMMs with distinct A matrices; 1% of the runs inject one random bit
flip (half into B' after encoding, half into C' through the epilogue hook) and every injected
run must be flagged. The runs are independent problems against one weight, so they are issued as
GROUPED launches (one problem per run: its own A, C', checksum column, flags and count; the C' faults
ride in the launch's fault list); the runs with a B' fault run as one batched launch, each against its own
B' (encoded from the clean B, one bit flipped after encoding, prepared before timing like the runs' A).
One step = one such job, replayed as a CUDA graph; L2 is flushed between steps (a 256 MiB read).
metric = checked int8 GEMM TOPS (2*m*n*k per GEMM, checksum column excluded).

Secondary lines in the same JSON object: ABFT overhead vs the same kernel with checking compiled
out, the cold single-GEMM latency, and the EmbeddingBag configs E3 (4M x 128 u8, Zipf bags) and
E4 (8M x 64 int4 + fp16, weighted) in algorithmic HBM GB/s.

--impl reference times the reference's own CPU implementation (oracle/_ref, compiled from the
reference sources) on all host cores for the same metric; it falls back to the C restatement
(oracle/liboracle.so) when the reference build is absent.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

M, N, K = 256, 4096, 4096
JOB = 1000
GROUP_MAX = 1000  # runs per grouped launch
SEED = 20260823
OPS = 2 * M * N * K
ALG_BYTES = M * K + K * (N + 1) + 4 * M * (N + 1) + M  # A, B' (incl. checksum column), C', flags


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}
    f = REPO / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        p = {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"], "source": "MEASURED_PEAKS.json"}
    # int8 tensor roof MEASURED on this pool's B200s (scripts/int8_peak.py -> profiles/r*/int8_peak.json): the
    # tcgen05 kind::i8 issue rate on every SM pair with random operands (cuBLASLt int8 is slower on B200), burst
    # (one ~5 ms launch) and sustained (>= 4 s back to back, under the 1 kW power cap). The job is timed as
    # 20 x 3 ms steps with sw_power_cap active, so `peak` is the sustained figure; the burst one rides along.
    caps = sorted(REPO.glob("profiles/r*/int8_peak.json"))
    if caps:
        d = json.loads(caps[-1].read_text())
        p["int8_tops"] = d["int8_peak_sustained_tops"]
        p["int8_tops_burst"] = d["int8_peak_burst_tops"]
        p["int8_source"] = f"{caps[-1].relative_to(REPO)} (tcgen05 kind::i8 microbenchmark, sustained; burst in int8_tops_burst)"
    else:
        p["int8_tops"] = p["int8_tops_burst"] = 2 * p["bf16_tflops"]
        p["int8_source"] = "2 x bf16 dense burst (no measured int8 peak found)"
    return p


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    def __init__(self):
        self.samples, self.proc, self.thread = [], None, None

    def start(self, dev_index: int):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(dev_index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ reference arm (CPU)
def cpu_gemm_sample(threads: int, reps: int = 1):
    """`threads` concurrent checked GEMMs at the G2 shape through the reference's abft_gemm
    (pre-encoded weight, as the job encodes B once). Returns (TOPS, kind, seconds)."""
    sys.path.insert(0, str(REPO / "tests"))
    import oracle_api as O  # noqa: E402  (test infrastructure: the CPU baseline only)
    a, b = O.gemm_inputs(SEED, 0, M, N, K)
    R = O.ref()
    kind = "reference" if R is not None else "port"
    outs = [np.empty((M, N + 1), np.int32) for _ in range(threads)]
    if R is not None:
        w = R.ref_gemm_weight_new(O.P(b), O.sz(K), O.sz(N))

        def one(i):
            err = C.c_uint64()
            R.ref_abft_gemm_w(O.P(a), O.sz(M), O.sz(K), C.c_void_p(w), O.P(outs[i]), C.byref(err))
    else:
        cs = O.row_checksums(b)

        def one(i):
            err = C.c_uint64()
            O.orc().orc_abft_gemm(O.P(a), O.sz(M), O.sz(K), O.P(b), O.sz(N), O.P(cs), O.P(outs[i]), None,
                                  C.byref(err))
    t0 = time.perf_counter()
    for _ in range(reps):
        ths = [threading.Thread(target=one, args=(i,)) for i in range(threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
    dt = time.perf_counter() - t0
    if R is not None:
        R.ref_gemm_weight_free(C.c_void_p(w))
    return threads * reps * OPS / dt / 1e12, kind, dt


def plan_segments(plan: dict, runs: int, group_max: int, max_faults: int = 8) -> list:
    """Split a job of `runs` GEMMs into launches: maximal ranges of runs without a B' fault become grouped
    launches ("group", first, count, [(problem, fault)...]) carrying their C' faults (at most `max_faults`
    per launch, the kernel's fault list); each B'-fault run is its own launch ("B", run, p, j, bit) between a
    flip and an unflip of B'. `plan` maps run -> ("B", p, j, bit) | ("C", row, col, bit)."""
    segments = []
    start = 0
    for run in sorted(r for r, f in plan.items() if f[0] == "B") + [runs]:
        i = start
        while i < run:
            cnt = min(run - i, group_max)
            c_in = [r for r in range(i, i + cnt) if r in plan and plan[r][0] == "C"]
            if len(c_in) > max_faults:  # cut the group before its (max_faults+1)-th C' fault
                cnt = c_in[max_faults] - i
            fl = [(r - i, plan[r]) for r in range(i, i + cnt) if r in plan and plan[r][0] == "C"]
            segments.append(("group", i, cnt, fl))
            i += cnt
        if run < runs:
            segments.append(("B", run) + tuple(plan[run][1:]))
        start = run + 1
    return segments


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _eb_configs(rng):
    """The E3 / E4 host inputs (BASELINE configs[2-3] shapes and distributions; the bags of eb_secondary's kind)."""
    out = {}
    for name in ("E3", "E4"):
        if name == "E3":
            R, d, nb, elem = 4_000_000, 128, 2048, "u8"
            lens = rng.integers(20, 101, nb)
            ranks = np.arange(1, R + 1, dtype=np.float64)
            cdf = np.cumsum(ranks ** -1.05)
            cdf /= cdf[-1]
            idx = rng.permutation(R)[np.searchsorted(cdf, rng.random(int(lens.sum())))].astype(np.int64)
            w, rb, meta_b = None, d, 12
            sc = rng.uniform(1e-3, 1e-2, R).astype(np.float32)
            bi = rng.uniform(-1, 1, R).astype(np.float32)
        else:
            R, d, nb, elem = 8_000_000, 64, 4096, "u4"
            lens = rng.integers(1, 151, nb)
            idx = rng.integers(0, R, int(lens.sum())).astype(np.int64)
            w = rng.uniform(0, 1, int(lens.sum())).astype(np.float32)
            rb, meta_b = d // 2, 8
            sc = rng.uniform(1e-3, 1e-2, R).astype(np.float16)
            bi = rng.uniform(-1, 1, R).astype(np.float16)
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        out[name] = dict(R=R, d=d, nb=nb, elem=elem, idx=idx, w=w, rb=rb, meta_b=meta_b, sc=sc, bi=bi, off=off)
    return out


def _parallel_bags(fn, nb, threads):
    """Run fn(b0, b1) over `threads` contiguous bag ranges concurrently (ctypes releases the GIL); wall seconds."""
    cuts = [nb * i // threads for i in range(threads + 1)]
    ths = [threading.Thread(target=fn, args=(cuts[i], cuts[i + 1])) for i in range(threads) if cuts[i + 1] > cuts[i]]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return time.perf_counter() - t0


def cpu_eb_sample():
    """E3 / E4 batches on the host cores: the oracle's C restatement of abft_embedding_bag
    (u8 / u4 rows: the reference implements s8 rows only) single-thread and on all cores, and the
    REFERENCE itself (oracle/_ref, abft_embedding_bag on a persistent table) on an s8 table of E3's shape, all
    cores. Returns {cfg: {...}}."""
    sys.path.insert(0, str(REPO / "tests"))
    import oracle_api as O  # noqa: E402  (test infrastructure: the CPU baseline only)
    threads = os.cpu_count() or 1
    out = {}
    cfgs = _eb_configs(np.random.default_rng(3))
    for name, c in cfgs.items():
        R, d, nb, elem, rb = c["R"], c["d"], c["nb"], c["elem"], c["rb"]
        rows = np.random.default_rng(4).integers(0, 256, (R, rb), dtype=np.uint8)
        sums = O.row_sums(rows, elem, d)
        off, idx, w = c["off"], c["idx"], c["w"]
        t0 = time.perf_counter()
        O.eb(rows, c["sc"], c["bi"], off, idx, w, elem=elem, dim=d, row_sums_=sums)
        dt1 = time.perf_counter() - t0

        def part(b0, b1):
            o = off[b0:b1 + 1] - off[b0]
            O.eb(rows, c["sc"], c["bi"], o, idx[off[b0]:off[b1]], None if w is None else w[off[b0]:off[b1]],
                 elem=elem, dim=d, row_sums_=sums)
        dtn = _parallel_bags(part, nb, threads)
        L_ = int(off[-1])
        alg = L_ * (rb + c["meta_b"] + 4 + 8 + (4 if w is not None else 0)) + 8 * (nb + 1) + 4 * nb * d + nb
        out[name] = {"ms": dt1 * 1e3, "alg_gbs": alg / dt1 / 1e9, "cores": 1, "kind": "port",
                     "ms_all_cores": dtn * 1e3, "alg_gbs_all_cores": alg / dtn / 1e9, "cores_all": threads,
                     "sample": f"one {name} batch ({nb} bags, {L_} lookups), oracle restatement ({elem} rows)"}
        if name == "E3" and O.ref() is not None:
            Rf = O.ref()
            srows = rows.view(np.int8)
            tab = Rf.ref_eb_table_new(O.P(srows), O.sz(R), O.sz(d), O.P(c["sc"]), O.P(c["bi"]))
            uoff, uidx = off.astype(np.uint64), idx.astype(np.uint64)
            r_out = np.empty((nb, d), np.float32)
            err = np.empty(nb, np.uint8)

            def ref_part(b0, b1):
                Rf.ref_eb_table_check_range(C.c_void_p(tab), O.P(uoff), O.P(uidx), None, O.sz(b0), O.sz(b1),
                                            O.P(r_out), O.P(err))
            dt_r1 = _parallel_bags(ref_part, nb, 1)
            dt_rn = _parallel_bags(ref_part, nb, threads)
            Rf.ref_eb_table_free(C.c_void_p(tab))
            out[name]["reference_s8_same_shape"] = {
                "ms": dt_r1 * 1e3, "ms_all_cores": dt_rn * 1e3, "cores_all": threads, "kind": "reference",
                "alg_gbs_all_cores": alg / dt_rn / 1e9,
                "sample": "the reference's abft_embedding_bag (oracle/_ref) on an s8 table of E3's shape, same bags"}
        del rows, sums
    return out


def cpu_reference_benches():
    """The reference's OWN single-thread benches through its C ABI (oracle/_ref: abftlp_bench_gemm / abftlp_bench_eb,
    P:src/bench.cpp:50-152: median of reps after 2 warm-ups; GEMM encode inside the checked timing; EB cache flush)."""
    sys.path.insert(0, str(REPO / "tests"))
    import oracle_api as O  # noqa: E402  (test infrastructure: the CPU baseline only)
    Rf = O.ref()
    if Rf is None:
        return None

    class BR(C.Structure):
        _fields_ = [("baseline_ns", C.c_double), ("abft_ns", C.c_double), ("overhead_fraction", C.c_double)]
    out = {}
    r = BR()
    if Rf.abftlp_bench_gemm(C.c_uint64(64), C.c_uint64(512), C.c_uint64(512), C.c_uint32(5), C.c_uint64(SEED),
                            C.byref(r)) == 0:
        out["gemm_64x512x512"] = {"plain_ms": r.baseline_ns / 1e6, "abft_ms": r.abft_ns / 1e6,
                                  "overhead_pct": 100 * r.overhead_fraction}
    if Rf.abftlp_bench_eb(C.c_uint64(4_000_000), C.c_uint64(128), C.c_uint64(60), C.c_uint64(2048), C.c_uint32(5),
                          C.c_uint64(SEED), C.byref(r)) == 0:
        out["eb_4Mx128_pool60_batch2048"] = {"plain_ms": r.baseline_ns / 1e6, "abft_ms": r.abft_ns / 1e6,
                                             "overhead_pct": 100 * r.overhead_fraction}
    out["cores"] = 1
    out["kind"] = "reference"
    return out


def cpu_g1_sample():
    """G1 on the host cores: the reference's abft_gemm (oracle/_ref) for the 100 seeded 64x512x512 trials, one
    pre-encoded weight per trial (the device path encodes before timing too), trials spread over every core."""
    sys.path.insert(0, str(REPO / "tests"))
    import oracle_api as O  # noqa: E402  (test infrastructure: the CPU baseline only)
    Rf = O.ref()
    if Rf is None:
        return None
    m, n, k, nt = 64, 512, 512, 100
    threads = os.cpu_count() or 1
    ins = [O.gemm_inputs(SEED, t, m, n, k) for t in range(nt)]
    ws = [Rf.ref_gemm_weight_new(O.P(b), O.sz(k), O.sz(n)) for _, b in ins]
    outs = [np.empty((m, n + 1), np.int32) for _ in range(nt)]

    def part(t0, t1):
        for t in range(t0, t1):
            err = C.c_uint64()
            Rf.ref_abft_gemm_w(O.P(ins[t][0]), O.sz(m), O.sz(k), C.c_void_p(ws[t]), O.P(outs[t]), C.byref(err))
    dt = _parallel_bags(part, nt, threads)
    dt1 = _parallel_bags(part, 10, 1) * nt / 10
    for w in ws:
        Rf.ref_gemm_weight_free(C.c_void_p(w))
    ops = 2 * m * n * k * nt
    return {"us_per_100_all_cores": dt * 1e6, "tops_all_cores": ops / dt / 1e12, "cores": threads,
            "us_per_100_single_thread": dt1 * 1e6, "kind": "reference",
            "sample": "the 100 G1 trials through the reference's abft_gemm (pre-encoded weights)"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_gemm_sample(threads)
    times = []
    for _ in range(args.steps):
        tops, kind, dt = cpu_gemm_sample(threads)
        times.append(dt)
    total = sum(times)
    value = args.steps * threads * OPS / total / 1e12
    line = {"metric": "checked int8 GEMM TOPS", "value": value, "unit": "TOPS", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8xs8->s32",
            "data": "synthetic (SplitMix64, the reference's draw protocol)",
            "config": {"workload": "G2: checked GEMM m=256 k=4096 n=4096 (BASELINE configs[1]); one step = "
                                   f"{threads} concurrent abft_gemm calls (one per host thread) on a pre-encoded B"},
            "cpu_baseline": {"value": value, "unit": "TOPS", "cores": threads, "kind": kind, "cpu_model": cpu_model(),
                             "sample": f"{threads} G2 GEMMs per step on {threads} threads"},
            "e2e": {"value": value, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def run_gpu_arm(args, rank, world, dist):
    import torch
    from paper_2103_00130_b200 import _lib as L
    from paper_2103_00130_b200.rng import SplitMix64

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    # one dedicated stream: the library's per-stream workspace is allocated during warm-up, so the job
    # can then be captured into a CUDA graph (no allocation happens under capture)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    st = C.c_void_p(stream.cuda_stream)
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    pk = peaks()

    # ---- inputs resident in HBM before timing: B encoded once; JOB distinct A matrices
    # Rank r owns the N-column shard r of a (N * world)-wide weight (weak scaling; no data-path
    # collective -- only the per-run verdicts are OR-reduced across ranks at the end of a step).
    b = torch.empty((K, N), dtype=torch.int8, device=dev)
    L.call("abftlp_generate", vp(b), K * N, SEED, 1000 + rank, 0, 1, 0.0, 0.0, 0, st)
    w = C.c_void_p()
    L.call("abftlp_gemm_encode", vp(b), K, N, N, st, C.byref(w))
    # the one-time encoder (reported separately): re-encode in place, CUDA events, L2 flushed
    enc_flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    enc_ts = []
    for i in range(4):
        L.call("abftlp_l2_flush", vp(enc_flush), enc_flush.numel(), 30 + i, st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        L.call("abftlp_gemm_reencode", w, vp(b), N, st)
        e1.record(stream)
        torch.cuda.synchronize()
        enc_ts.append(e0.elapsed_time(e1) * 1e3)
    encode_us = statistics.median(enc_ts[1:])
    # ten re-encodes in one CUDA graph (launch and event latency amortised; B stays L2-resident between them)
    encode_graph_us = None
    try:
        gs = torch.cuda.Stream()
        with torch.cuda.stream(gs):
            gst = C.c_void_p(gs.cuda_stream)
            L.call("abftlp_gemm_reencode", w, vp(b), N, gst)
            torch.cuda.synchronize()
            eg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(eg, stream=gs):
                for _ in range(10):
                    L.call("abftlp_gemm_reencode", w, vp(b), N, gst)
            eg.replay()
            torch.cuda.synchronize()
            gts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(gs)
                eg.replay()
                e1.record(gs)
                torch.cuda.synchronize()
                gts.append(e0.elapsed_time(e1) * 1e3 / 10)
            encode_graph_us = statistics.median(gts)
            del eg
    except Exception:  # noqa: BLE001
        torch.cuda.synchronize()
    del enc_flush
    a_pool = torch.empty((JOB, M, K), dtype=torch.uint8, device=dev)
    L.call("abftlp_generate", vp(a_pool), JOB * M * K, SEED, 0, 0, 0, 0.0, 0.0, 0, st)
    c_all = torch.empty((JOB, M, N), dtype=torch.int32, device=dev)  # every run keeps its C' (4.3 GB)
    csum = torch.empty((JOB, M), dtype=torch.int32, device=dev)
    flags = torch.empty((JOB, M), dtype=torch.uint8, device=dev)
    errs = torch.zeros(JOB, dtype=torch.int32, device=dev)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    # 1% of the runs carry a fault: even ones flip a bit of B' (j < n, bit 0..7) before the GEMM and
    # undo it after; odd ones flip a bit of C' (any column incl. the checksum, bit 0..31) in the epilogue.
    rng = SplitMix64(SEED, 7 + rank)
    fault_runs = sorted({rng.next_below(JOB) for _ in range(JOB // 100 * 3)})[: JOB // 100]
    plan = {}
    for idx, run in enumerate(fault_runs):
        if idx % 2 == 0:
            plan[run] = ("B", rng.next_below(K), rng.next_below(N), rng.next_below(8))
        else:
            plan[run] = ("C", rng.next_below(M), rng.next_below(N + 1), rng.next_below(32))

    # The runs are independent, so the job schedules its B'-fault runs last (each needs its own corrupted weight and
    # they form one batched launch anyway): the other runs are then one contiguous range -- one grouped launch instead
    # of one per gap between B'-fault runs. (The plan keeps its seeded draws; only the runs' positions move.)
    order = [r for r in range(JOB) if not (r in plan and plan[r][0] == "B")] + \
            sorted(r for r, f in plan.items() if f[0] == "B")
    if not os.environ.get("ABFT_BENCH_KEEP_ORDER"):  # (A/B switch: the job with its B'-fault runs in place)
        plan = {pos: plan[run] for pos, run in enumerate(order) if run in plan}

    # The job's runs are independent GEMMs against the one encoded weight, so they are issued as GROUPED
    # launches (abftlp_gemm_checked_batched_faults: problem b = run b, its own A, C', csum, flags and count;
    # the C' faults of the group ride in the launch's fault list). A run with a B' fault must see its own
    # corrupted weight: B is encoded once per such run (checksums of the clean B) and B'(p, j) flipped after
    # encoding -- inject_weight_B's point (P:src/fault_lab.cpp:186-189) -- before timing, like the runs' A;
    # in the job these runs are ONE batched launch, each problem with its own faulted weight.
    segments = plan_segments(plan, JOB, GROUP_MAX)
    b_runs = sorted(r for r, f in plan.items() if f[0] == "B")
    nfb = len(b_runs)
    wf = C.c_void_p()
    if nfb:
        bcopies = b.unsqueeze(0).repeat(nfb, 1, 1).contiguous()
        L.call("abftlp_gemm_encode_batched", vp(bcopies), nfb, K, N, N, K * N, st, C.byref(wf))
        for q, r in enumerate(b_runs):
            _, pp, jj, bit = plan[r]
            L.call("abftlp_gemm_weight_flip_bit_batched", wf, q, pp, jj, bit, st)
        torch.cuda.synchronize()
        del bcopies
        a_f = a_pool[b_runs].contiguous()
        c_f = torch.empty((nfb, M, N), dtype=torch.int32, device=dev)
        cs_f = torch.empty((nfb, M), dtype=torch.int32, device=dev)
        fl_f = torch.empty((nfb, M), dtype=torch.uint8, device=dev)
        err_f = torch.zeros(nfb, dtype=torch.int32, device=dev)

    def launch_group(i0, cnt, fl, checked):
        if checked:
            arr = (L.BatchFault * max(1, len(fl)))()
            for q, (b_, f) in enumerate(fl):
                arr[q] = L.BatchFault(1, b_, f[1], f[2], f[3])
            L.call("abftlp_gemm_checked_batched_faults", vp(a_pool[i0]), cnt, M, K, M * K, w, vp(c_all[i0]), N,
                   M * N, vp(csum[i0]), 1, M, vp(flags[i0]), M, vp(errs[i0:]), arr, len(fl), st)
        else:
            L.call("abftlp_gemm_unchecked_batched", vp(a_pool[i0]), cnt, M, K, M * K, w, vp(c_all[i0]), N, M * N, st)

    def job(checked=True, events=None):
        """Issues the whole job on `st`; returns the number of kernels it launches. With `events`, the grouped
        launches are bracketed by CUDA events (the roofline's per-launch durations; not used when timing)."""
        n = 0
        for sg in segments:
            if sg[0] == "group":
                _, i0, cnt, fl = sg
                if events is not None:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                launch_group(i0, cnt, fl, checked)
                if events is not None:
                    e1.record(stream)
                    events.append((cnt, e0, e1))
                n += 1
                continue
        if nfb:  # the B'-fault runs, each against its own corrupted weight, in one batched launch
            if checked:
                L.call("abftlp_gemm_checked_batched", vp(a_f), nfb, M, K, M * K, wf, vp(c_f), N, M * N, vp(cs_f), 1, M,
                       vp(fl_f), M, vp(err_f), None, st)
            else:
                L.call("abftlp_gemm_unchecked_batched", vp(a_f), nfb, M, K, M * K, wf, vp(c_f), N, M * N, st)
            n += 1
        return n

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps, flush=True):
        total, per = 0.0, []
        for s in range(steps):
            if flush:
                L.call("abftlp_l2_flush", vp(flush_buf), flush_buf.numel(), s, st)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            barrier()
            ms = e0.elapsed_time(e1)
            if dist is not None:
                t = torch.tensor([ms], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            per.append(ms)
            total += ms
        return total, per

    # ---- warm-up on the job stream (workspace, tensor maps, kernel attributes), then capture the job:
    # a step replays 1000 GEMM launches (+ the fault-injection kernels) without per-launch host cost.
    for _ in range(max(1, args.warmup)):
        job(True)
        job(False)
    barrier()
    graphs = {}
    kernels_per_job = {}
    for ck in (True, False):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            kernels_per_job[ck] = job(ck)
        graphs[ck] = g
    torch.cuda.set_stream(stream)
    for _ in range(args.warmup):
        graphs[True].replay()
        graphs[False].replay()
    barrier()

    # checked steps (the metric) interleaved with unchecked ones (the ABFT-overhead baseline), so both see the same
    # clocks under the power cap; each step is flushed and bracketed by barrier + synchronize, timed on the device
    clocks = Clocks()
    clocks.start(dev.index)
    t_total, u_total, t_steps = 0.0, 0.0, []
    for s_ in range(args.steps):
        tc, per_c = timed(graphs[True].replay, 1)
        tu, _ = timed(graphs[False].replay, 1)
        t_total += tc
        u_total += tu
        t_steps += per_c
    clk = clocks.stop()
    launches_timed = args.steps * (kernels_per_job[True] + 1)  # checked steps: the job + the L2 flush before each

    # parity of the job's verdicts: every injected run flagged, no clean run flagged
    e = errs.cpu().numpy()
    ok_clean = all(e[i] == 0 for i in range(JOB) if i not in plan)
    c_runs = [r for r, f in plan.items() if f[0] == "C"]
    ok_c = all(e[r] == 1 for r in c_runs)
    ok_b = nfb == 0 or bool((err_f >= 1).all().item())
    verdict = torch.tensor(e, device=dev)
    if dist is not None:
        dist.all_reduce(verdict, op=dist.ReduceOp.MAX)  # OR of the per-shard verdicts

    # ---- the roofline's kernel: the grouped checked launch, timed IN-GRAPH. A second graph holds only the job's
    # grouped checked launches (the same launches, same order, PDL between them, minus the B'-fault batch); its
    # replay time over the number of launches is the kernel's average launch duration inside the step, so
    # kernel time per step <= ms_per_step by construction. L2 flushed before each replay, as the step.
    def grouped_only():
        n = 0
        for sg in segments:
            if sg[0] == "group":
                launch_group(sg[1], sg[2], sg[3], True)
                n += 1
        return n
    g_grp = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_grp, stream=stream):
        n_grp = grouped_only()
    torch.cuda.set_stream(stream)
    g_grp.replay()
    grp_total, _ = timed(g_grp.replay, args.steps)
    del g_grp
    grp_gemms = sum(sg[2] for sg in segments if sg[0] == "group")
    grp_ms = grp_total / args.steps
    kernel_us = grp_ms * 1e3 / n_grp  # average grouped-launch duration inside the graph
    gemms_per_launch = grp_gemms / n_grp

    # ---- one m=256 GEMM per launch (no grouping): isolated launch latency, and the job as a CUDA graph of
    # 1000 single launches (programmatic dependent launch between them) -- what grouping is compared with
    c1 = torch.empty((M, N), dtype=torch.int32, device=dev)
    cs1 = torch.empty(M, dtype=torch.int32, device=dev)
    f1 = torch.empty(M, dtype=torch.uint8, device=dev)
    e1_ = torch.zeros(1, dtype=torch.int32, device=dev)

    def single(i, c=None):
        L.call("abftlp_gemm_checked", vp(a_pool[i]), M, K, w, vp(c1 if c is None else c), N, vp(cs1), 1, vp(f1),
               vp(e1_), None, st)
    per_launch = []
    torch.cuda.synchronize()
    torch.cuda._sleep(4_000_000)
    for i in range(60):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        single(i)
        e1.record(stream)
        per_launch.append((e0, e1))
    torch.cuda.synchronize()
    single_launch_us = statistics.median(a.elapsed_time(b) * 1e3 for a, b in per_launch[10:])
    # library yardstick in the same run: cuBLASLt int8 (torch._int_mm, s8 x s8 -> s32, NO check) at the same shape
    a8 = torch.randint(-128, 128, (M, K), dtype=torch.int8, device=dev)
    b8 = torch.randint(-128, 128, (K, N), dtype=torch.int8, device=dev)
    for _ in range(5):
        torch._int_mm(a8, b8)
    torch.cuda.synchronize()
    torch.cuda._sleep(4_000_000)
    cub = []
    for _ in range(60):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        torch._int_mm(a8, b8)
        e1.record(stream)
        cub.append((e0, e1))
    torch.cuda.synchronize()
    cublas_us = statistics.median(a.elapsed_time(b) * 1e3 for a, b in cub[10:])
    # the same yardstick as a CUDA graph of 200 calls (each its own A and C', like the ungrouped job below): per-call
    # time without the events' and the launches' host latency
    cublas_graph_us = None
    try:
        a8s = torch.randint(-128, 128, (200, M, K), dtype=torch.int8, device=dev)
        c8s = torch.empty((200, M, N), dtype=torch.int32, device=dev)
        torch._int_mm(a8s[0], b8, out=c8s[0])
        torch.cuda.synchronize()
        gcb = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gcb, stream=stream):
            for i in range(200):
                torch._int_mm(a8s[i], b8, out=c8s[i])
        torch.cuda.set_stream(stream)
        gcb.replay()
        cbt = []
        for s_ in range(3):  # (local timing only: no collective inside an optional section)
            L.call("abftlp_l2_flush", vp(flush_buf), flush_buf.numel(), 200 + s_, st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            gcb.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            cbt.append(e0.elapsed_time(e1))
        cublas_graph_us = statistics.median(cbt) * 1e3 / 200
        del gcb, a8s, c8s
    except Exception:  # noqa: BLE001  (no out= variant / capture unsupported in this torch build)
        torch.cuda.synchronize()
    del a8, b8
    # grouped results are bit-identical to single launches (spot check on a clean run)
    clean_run = next(i for i in range(JOB) if i not in plan)
    single(clean_run)
    torch.cuda.synchronize()
    grouped_eq_single = bool(torch.equal(c1, c_all[clean_run]) and torch.equal(cs1, csum[clean_run]))
    g1k = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1k, stream=stream):
        for i in range(JOB):
            single(i, c_all[i])
    torch.cuda.set_stream(stream)
    g1k.replay()
    ungrouped_total, _ = timed(g1k.replay, max(1, min(3, args.steps)))
    ungrouped_tops = world * max(1, min(3, args.steps)) * JOB * OPS / (ungrouped_total * 1e-3) / 1e12
    del g1k

    # ---- cold single GEMM (L2 flushed before each launch), kernel-only
    cold = []
    for s in range(10):
        L.call("abftlp_l2_flush", vp(flush_buf), flush_buf.numel(), 100 + s, st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        single(s)
        e1.record(stream)
        torch.cuda.synchronize()
        cold.append(e0.elapsed_time(e1) * 1e3)

    # ---- e2e: grouped runs through the host-buffer C-ABI call (pinned host A in; C', csum, flags, counts out),
    # host->device, the grouped launches and device->host pipelined inside the call
    e2e_runs = 100
    a_host = torch.empty((e2e_runs, M, K), dtype=torch.uint8).pin_memory()
    a_host.copy_(a_pool[:e2e_runs].cpu())
    c_host = torch.empty((e2e_runs, M, N), dtype=torch.int32).pin_memory()
    cs_host = torch.empty((e2e_runs, M), dtype=torch.int32).pin_memory()
    fl_host = torch.empty((e2e_runs, M), dtype=torch.uint8).pin_memory()
    ec_host = torch.zeros(e2e_runs, dtype=torch.int32).pin_memory()

    def e2e_job():
        L.call("abftlp_gemm_checked_host_batched", C.c_void_p(a_host.data_ptr()), e2e_runs, M, K, M * K, w,
               C.c_void_p(c_host.data_ptr()), N, M * N, C.c_void_p(cs_host.data_ptr()), M,
               C.c_void_p(fl_host.data_ptr()), M, C.c_void_p(ec_host.data_ptr()), st)
    e2e_job()
    barrier()
    t0 = time.perf_counter()
    e2e_job()
    barrier()
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_tops = world * e2e_runs * OPS / e2e_s / 1e12
    chk = [i for i in range(e2e_runs) if i not in plan][:: 16]
    e2e_eq_device = all(torch.equal(c_host[i], c_all[i].cpu()) and torch.equal(cs_host[i], csum[i].cpu()) for i in chk) \
        and all(int(ec_host[i]) == 0 for i in chk)

    # ---- e2e with the requantization fused (the layer as the DLRM pipeline uses it: u8 in, u8 out; the int32 product
    # never leaves the GPU): abftlp_gemm_checked_requant_host_batched over the same runs
    rqp = L.RequantParams(0.02, -0.3, 0.01, 0.1, 37.0, -5.0, K)
    o_host = torch.empty((e2e_runs, M, N), dtype=torch.uint8).pin_memory()

    def e2e_rq_job():
        L.call("abftlp_gemm_checked_requant_host_batched", C.c_void_p(a_host.data_ptr()), e2e_runs, M, K, M * K, w,
               C.byref(rqp), C.c_void_p(o_host.data_ptr()), N, M * N, C.c_void_p(cs_host.data_ptr()), M,
               C.c_void_p(fl_host.data_ptr()), M, C.c_void_p(ec_host.data_ptr()), st)
    e2e_rq_job()
    barrier()
    t0 = time.perf_counter()
    e2e_rq_job()
    barrier()
    e2e_rq_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_rq_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_rq_s = float(t.item())
    e2e_rq_tops = world * e2e_runs * OPS / e2e_rq_s / 1e12
    # checked against the standalone requantize of the device C' of the same runs
    rs_d = torch.empty(M, dtype=torch.int32, device=dev)
    colsum_d = torch.empty(N, dtype=torch.int32, device=dev)
    o_d = torch.empty((M, N), dtype=torch.uint8, device=dev)
    L.call("abftlp_gemm_weight_col_sums", w, vp(colsum_d), st)
    e2e_rq_eq = True
    for i in chk[:3]:
        L.call("abftlp_row_sums_u8", vp(a_pool[i]), M, K, K, vp(rs_d), st)
        L.call("abftlp_requantize", vp(c_all[i]), c_all[i].stride(0), M, N, vp(rs_d), vp(colsum_d), C.byref(rqp), vp(o_d), N, st)
        torch.cuda.synchronize()
        e2e_rq_eq = e2e_rq_eq and torch.equal(o_host[i], o_d.cpu()) and torch.equal(cs_host[i], csum[i].cpu())

    # D5 runs on every rank (table-wise EB + exchange + N-split MLP); the single-GPU legs on rank 0 only
    d5 = None if args.no_d5 else d5_leg(L, dev, st, vp, pk, rank, world, dist)
    secondary = eb_secondary(L, dev, st, vp, pk) if (rank == 0 and not args.no_eb) else None
    if rank == 0 and secondary is not None:
        secondary["G1"] = g1_secondary(L, dev, st, vp, pk)
    if rank == 0 and d5 is not None:
        secondary = secondary or {}
        secondary["D5"] = d5

    L.lib.abftlp_gemm_weight_free(w)
    if nfb:
        L.lib.abftlp_gemm_weight_free(wf)
    if rank != 0:
        return
    value = world * args.steps * JOB * OPS / (t_total * 1e-3) / 1e12
    # DRAM traffic of the checked kernel from the committed ncu --set full capture (profiles/)
    # DRAM traffic of the grouped checked kernel from the committed ncu --set full capture (profiles/),
    # recorded per GEMM and scaled to this run's GEMMs per launch
    traffic, traffic_src = None, None
    caps = sorted(REPO.glob("profiles/r*/ncu_gemm_g2grouped_*.json"))
    if caps:
        cap = json.loads(caps[-1].read_text())
        traffic, traffic_src = cap["traffic_bytes_per_gemm"] * gemms_per_launch, str(caps[-1].relative_to(REPO))
    achieved = grp_gemms * OPS / (grp_ms * 1e-3) / 1e12
    # unique bytes of one grouped launch: every run's A, C' (incl. checksum column) and flags, plus B' once (the
    # job's weight is read from HBM once and then served from L2)
    uniq_bytes = gemms_per_launch * (M * K + 4 * M * (N + 1) + M) + K * (N + 1)
    line = {
        "metric": "checked int8 GEMM TOPS", "value": value, "unit": "TOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8xs8->s32",
        "data": "synthetic (SplitMix64, the reference's draw protocol); no dataset",
        "config": {"workload": "G2 = BASELINE configs[1]: checked GEMM m=256 k=4096 n=4096, B encoded once, "
                               f"job of {JOB} GEMMs with distinct A, 1% fault runs (B' and C' bit flips)",
                   "step": f"one {JOB}-GEMM job", "l2": "flushed between steps (256 MiB read, untimed); the job's 1 GB of A exceeds L2",
                   "launch": "CUDA graph of the job: one grouped launch over the runs that share the encoded B' (one problem per run, C' faults in the launch's fault list; at most 8 per launch); the B'-fault runs are scheduled last as one batched launch, each against its own B' (clean checksums, one bit flipped after encoding, prepared before timing like the runs' A)",
                   "parallelism": f"N-column shard per GPU (n={N} per rank), verdicts OR-reduced",
                   "gemm_kernel": "tcgen05 cta_group::2 int8, TMEM accumulators, fused mod-127 row check"},
        "e2e": {"value": e2e_tops, "unit": "TOPS", "h2d_bytes_per_step": M * K * e2e_runs,
                "d2h_bytes_per_step": (4 * M * N + 4 * M + M + 4) * e2e_runs,
                "note": f"one abftlp_gemm_checked_host_batched call over {e2e_runs} runs (pinned host A in; C', csum, flags, counts out; copies pipelined with the grouped launches)"},
        "e2e_requant": {"value": e2e_rq_tops, "unit": "TOPS", "h2d_bytes_per_step": M * K * e2e_runs,
                        "d2h_bytes_per_step": (M * N + 4 * M + M + 4) * e2e_runs, "eq_device_requantize": e2e_rq_eq,
                        "note": f"one abftlp_gemm_checked_requant_host_batched call over {e2e_runs} runs: u8 A in, requantized u8 out "
                                "(+ csum, flags, counts); the int32 C' is never written -- an extra, not the headline e2e (which returns C')"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": pk["int8_tops"], "unit": "TOP/s",
                     "frac": achieved / pk["int8_tops"], "traffic": traffic, "traffic_unit": "bytes/launch",
                     "traffic_source": traffic_src,
                     "peak_burst": pk["int8_tops_burst"], "frac_of_burst": achieved / pk["int8_tops_burst"],
                     "kernel": "gemm_pair_kernel<256, checked> (grouped launch)", "kernel_us": kernel_us,
                     "kernel_us_how": f"CUDA-graph replay of the job's {n_grp} grouped checked launches (same launches as the step, "
                                      "L2 flushed before each replay) / launches",
                     "kernel_share_of_step": grp_ms / (t_total / args.steps),
                     "gemms_per_launch": gemms_per_launch, "ops_per_launch": gemms_per_launch * OPS,
                     "unique_bytes_per_launch": uniq_bytes,
                     "unique_gbs": uniq_bytes / (kernel_us * 1e-6) / 1e9,
                     "peak_source": pk["int8_source"],
                     "note": "B' (16.8 MB) is read from HBM once per launch and then served from L2; A and C' stream through HBM, so the bound is the tensor pipe"},
        "per_gemm_launch": {"single_launch_us": single_launch_us,
                            "single_launch_how": "median CUDA-event duration of an isolated m=256 checked launch",
                            "cublas_int8_unchecked_us": cublas_us,
                            "cublas_how": "torch._int_mm (cuBLASLt, s8 x s8 -> s32, no checksum) 256x4096x4096, same method",
                            "graph_us_per_gemm": ungrouped_total / max(1, min(3, args.steps)) * 1e3 / JOB,
                            "cublas_graph_us_per_gemm": cublas_graph_us,
                            "graph_how": "the job's 1000 checked GEMMs as a CUDA graph of single launches (PDL) vs a "
                                         "CUDA graph of 200 torch._int_mm calls (unchecked), each call its own A and "
                                         "C', L2 flushed before each replay: per-call device time",
                            "ungrouped_job_tops": ungrouped_tops,
                            "ungrouped_how": "the same 1000 GEMMs as a CUDA graph of 1000 single launches (PDL)"},
        "encoder": {"us": encode_us, "alg_bytes": 2 * K * N, "alg_gbs": 2 * K * N / (encode_us * 1e-6) / 1e9,
                    "hbm_frac": 2 * K * N / (encode_us * 1e-6) / 1e9 / pk["hbm_gbs"],
                    "us_in_graph_of_10": encode_graph_us,
                    "hbm_frac_in_graph": (2 * K * N / (encode_graph_us * 1e-6) / 1e9 / pk["hbm_gbs"]
                                          if encode_graph_us else None),
                    "note": "abftlp_gemm_reencode of the G2 weight (B read, B' written; checksums): one launch after an "
                            "L2 flush (CUDA events around one launch include ~6 us of launch and event latency), and "
                            "ten re-encodes in one CUDA graph / 10 (B L2-warm)"},
        "cold_gemm": {"us_median": statistics.median(cold), "alg_gbs": ALG_BYTES / (statistics.median(cold) * 1e-6) / 1e9,
                      "hbm_frac": ALG_BYTES / (statistics.median(cold) * 1e-6) / 1e9 / pk["hbm_gbs"],
                      "note": "single checked GEMM with L2 flushed (B' from HBM)"},
        "abft_overhead_pct": 100.0 * (t_total - u_total) / u_total,
        "parity": {"clean_runs_unflagged": bool(ok_clean), "c_faults_flagged": bool(ok_c),
                   "b_faults_flagged": bool(ok_b), "fault_runs": len(plan),
                   "grouped_eq_single_launch": grouped_eq_single, "e2e_eq_device": bool(e2e_eq_device)},
        "gpu_launches": launches_timed,
        "clocks": clk,
    }
    if secondary:
        line["secondary"] = secondary
    if not args.no_cpu and world == 1:
        threads = os.cpu_count() or 1
        tops, kind, dt = cpu_gemm_sample(threads)
        line["cpu_baseline"] = {"value": tops, "unit": "TOPS", "cores": threads, "kind": kind,
                                "sample": f"{threads} concurrent G2 abft_gemm calls ({dt:.1f} s wall)"}
        line["cpu_baseline"]["cpu_model"] = cpu_model()
        if secondary is not None:
            try:
                line["cpu_baseline"]["eb"] = cpu_eb_sample()
            except MemoryError:
                pass
            line["cpu_baseline"]["g1"] = cpu_g1_sample()
            line["cpu_baseline"]["reference_own_benches"] = cpu_reference_benches()
    print(json.dumps(line), flush=True)


def g1_secondary(L, dev, st, vp, pk):
    """BASELINE configs[0] (G1): 100 seeded checked GEMMs m=64 k=512 n=512 (each trial its own A and B,
    the reference's draw protocol, stream t*4), half with one C' bit flip (stream t*4+1 draws) -- ONE
    batched launch (abftlp_gemm_checked_batched) vs 100 single launches, both replayed as CUDA graphs."""
    import torch
    from paper_2103_00130_b200.rng import SplitMix64
    nb, m, n, k = 100, 64, 512, 512
    a = torch.empty((nb, m, k), dtype=torch.uint8, device=dev)
    b = torch.empty((nb, k, n), dtype=torch.int8, device=dev)
    for t in range(nb):
        L.call("abftlp_generate", vp(a[t]), m * k, SEED, t * 4, 0, 0, 0.0, 0.0, 0, st)
        L.call("abftlp_generate", vp(b[t]), k * n, SEED, t * 4, m * k, 1, 0.0, 0.0, 0, st)
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
    faults = []
    for t in range(1, nb, 2):
        r = SplitMix64(SEED, t * 4 + 1)
        faults.append((t, r.next_below(m), r.next_below(n + 1), r.next_below(32)))

    def batched(fault=None):
        f = C.byref(L.BatchFault(1, *fault)) if fault else None
        L.call("abftlp_gemm_checked_batched", vp(a), nb, m, k, m * k, wb, vp(c), n + 1, m * (n + 1),
               C.c_void_p(c.data_ptr() + 4 * n), n + 1, m * (n + 1), vp(fl), m, vp(err), f, st)

    # the same launch with C' in a 16-byte-aligned layout (C m x n, checksum column as a separate vector): the
    # reference's m x (n+1) rows are not 16-byte aligned, so that layout cannot use the TMA-store epilogue
    c2 = torch.empty((nb, m, n), dtype=torch.int32, device=dev)
    cs2 = torch.empty((nb, m), dtype=torch.int32, device=dev)

    def batched_aligned():
        L.call("abftlp_gemm_checked_batched", vp(a), nb, m, k, m * k, wb, vp(c2), n, m * n, vp(cs2), 1, m, vp(fl), m,
               vp(err), None, st)

    def separate():
        for t in range(nb):
            L.call("abftlp_gemm_checked", vp(a[t]), m, k, ws[t], vp(c[t]), n + 1, C.c_void_p(c[t].data_ptr() + 4 * n),
                   n + 1, vp(fl[t]), vp(err[t:t + 1]), None, st)

    stream = torch.cuda.current_stream()
    res = {}
    for name, fn in (("batched", batched), ("batched_aligned", batched_aligned), ("separate", separate)):
        fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fn()
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(10):
                g.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / 10)
        res[name] = statistics.median(ts)
        del g
    # both layouts hold the same C' (and checksum column)
    batched_aligned()
    batched()
    torch.cuda.synchronize()
    layouts_equal = bool(torch.equal(c[:, :, :n], c2) and torch.equal(c[:, :, n], cs2))
    # verdict parity of the G1 protocol: every odd trial's single flip detected, no false positive
    clean_ok = int(err.sum().item()) == 0
    det = 0
    for fault in faults:
        batched(fault)
        det += int(err[fault[0]].item() == 1 and int(err.sum().item()) == 1)
    for w in ws:
        L.lib.abftlp_gemm_weight_free(w)
    L.lib.abftlp_gemm_weight_free(wb)
    ops = 2 * m * n * k * nb
    alg = nb * (m * k + k * (n + 1) + 4 * m * (n + 1) + m)
    aligned_gbs = alg / (res["batched_aligned"] * 1e-6) / 1e9
    return {"roofline": {"bound": "hbm", "achieved": aligned_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": aligned_gbs / pk["hbm_gbs"], "alg_bytes": alg,
                         "kernel": "gemm_pair_kernel batched (100 G1 trials, C' 16-byte aligned)",
                         "note": "A, B', C' incl. checksum column and flags of the 100 trials, one launch; "
                                 "latency-bound at 42.7 MB (HBM roof 6.5 us)"},
            "trials": nb, "batched_us_per_100": res["batched"], "separate_us_per_100": res["separate"],
            "batched_aligned_us_per_100": res["batched_aligned"],
            "batched_aligned_tops": ops / (res["batched_aligned"] * 1e-6) / 1e12,
            "batched_aligned_hbm_frac": alg / (res["batched_aligned"] * 1e-6) / 1e9 / pk["hbm_gbs"],
            "layouts_equal": layouts_equal,
            "batched_tops": ops / (res["batched"] * 1e-6) / 1e12, "alg_gbs": alg / (res["batched"] * 1e-6) / 1e9,
            "hbm_frac": alg / (res["batched"] * 1e-6) / 1e9 / pk["hbm_gbs"], "clean_unflagged": clean_ok,
            "faults_detected": f"{det}/{len(faults)}",
            "note": "one abftlp_gemm_checked_batched launch for the 100 trials (reference m x (n+1) layout; and C' 16-byte aligned with the checksum column separate) vs 100 abftlp_gemm_checked launches"}


def d5_leg(L, dev, st, vp, pk, rank, world, dist, steps=8):
    """BASELINE configs[4] (D5), the whole DLRM-style step on `world` GPUs (one process per GPU):
      * 64 int8-rowwise tables x 1M x 128 (fp32 scale/bias), table-wise sharded (table t on rank t % G), batch
        8192, pooling 80, Zipf(1.05) indices -- every rank's tables pooled by ONE grouped checked launch that
        writes straight into the persistent exchange buffer (vectors + verdict quads);
      * the exchange: ONE all_to_all_single (NCCL over NVLink) to batch-sharded [B/G, 64, 128], then the
        (slot, rank) -> table reorder (one copy kernel each for vectors and verdicts);
      * the checked MLP GEMMs m = 8192, (k, n) in {512,1024,2048}^2 split by N columns across ranks (each rank
        encodes its own column shard), and the OR of the per-row GEMM verdicts (one all-reduce MAX).
    Seeded synthetic data (identical tables and bags at any world size). The step is replayed as a CUDA graph
    when it captures (eager otherwise); times are CUDA events, max over ranks."""
    import torch
    from paper_2103_00130_b200 import embedding as E
    from paper_2103_00130_b200 import sharded as S
    T, R, d, B, pool, m = 64, 1_000_000, 128, 8192, 80, 8192
    G = world
    mine = S.local_tables(T, G, rank)
    ranks = torch.arange(1, R + 1, dtype=torch.float64, device=dev)
    cdf = torch.cumsum(ranks ** -1.05, 0)
    cdf /= cdf[-1].clone()
    tables, bags = {}, {}
    for t in mine:
        gen = torch.Generator(device=dev)
        gen.manual_seed(5000 + t)
        rows = torch.randint(-128, 128, (R, d), dtype=torch.int8, device=dev, generator=gen)
        sc = torch.rand(R, device=dev, generator=gen) * 9e-3 + 1e-3
        bi = torch.rand(R, device=dev, generator=gen) * 2 - 1
        tables[t] = E.QuantEmbeddingTable(rows, sc, bi, elem="s8", dim=d)
        u = torch.rand(B * pool, dtype=torch.float64, device=dev, generator=gen)
        perm = torch.randperm(R, device=dev, generator=gen)
        idx = perm[torch.searchsorted(cdf, u).clamp_(max=R - 1)]
        bags[t] = (torch.arange(0, B * pool + 1, pool, dtype=torch.int64, device=dev), idx.contiguous(), None)
        del rows, sc, bi, u, perm
    del ranks, cdf
    group_ok = True
    eb = S.ShardedEmbeddingBags(tables, T, B, d, device=dev)
    shapes = [(k, n) for k in (512, 1024, 2048) for n in (512, 1024, 2048)]
    mlp = []
    mflags = torch.zeros((len(shapes), m), dtype=torch.uint8, device=dev)
    for q, (k, n) in enumerate(shapes):
        gen = torch.Generator(device=dev)
        gen.manual_seed(9000 + q)
        bfull = torch.randint(-128, 128, (k, n), dtype=torch.int8, device=dev, generator=gen)
        a = torch.randint(0, 256, (m, k), dtype=torch.uint8, device=dev, generator=gen)
        n0, n1 = S.column_shard(n, G, rank)
        bsh = bfull[:, n0:n1].contiguous()
        w = C.c_void_p()
        L.call("abftlp_gemm_encode", vp(bsh), k, n1 - n0, n1 - n0, st, C.byref(w))
        c = torch.empty((m, n1 - n0), dtype=torch.int32, device=dev)
        cs = torch.empty(m, dtype=torch.int32, device=dev)
        er = torch.zeros(1, dtype=torch.int32, device=dev)
        mlp.append((k, n1 - n0, w, a, c, cs, er))
        del bfull, bsh
    # the 9 MLP layers as ONE heterogeneous grouped launch (abftlp_gemm_group_*): same outputs as 9 launches
    probs = (L.GemmProblem * len(mlp))()
    for q, (k, n_loc, w, a, c, cs, er) in enumerate(mlp):
        probs[q] = L.GemmProblem(a.data_ptr(), m, k, w.value, c.data_ptr(), n_loc, cs.data_ptr(), 1,
                                 mflags[q].data_ptr(), er.data_ptr())
    mlp_group = C.c_void_p()
    L.call("abftlp_gemm_group_create", probs, len(mlp), 1, C.byref(mlp_group))

    def phase_eb():
        if eb.local is not None:  # one GPU: the grouped lookups write the final [B, 64, 128] layout directly
            eb.launch(bags)
        else:
            eb.backend.pool_into([tables[t] for t in eb.order], [bags[t] for t in eb.order], eb.xsend, d)

    def phase_x():
        if eb.local is not None:
            return eb.local
        dist.all_to_all_single(eb.xrecv, eb.xsend)
        return S.unpack_exchange(eb.xrecv, T, d, eb.out, eb.flags)

    def phase_mlp():
        L.call("abftlp_gemm_group_run", mlp_group, st)

    def phase_mlp_separate():  # the same 9 checked GEMMs as 9 launches (what the grouped launch replaces)
        for q, (k, n_loc, w, a, c, cs, er) in enumerate(mlp):
            L.call("abftlp_gemm_checked", vp(a), m, k, w, vp(c), n_loc, vp(cs), 1, vp(mflags[q]), vp(er), None, st)

    def phase_or():
        if G > 1:
            dist.all_reduce(mflags, op=dist.ReduceOp.MAX)  # OR of the N-shard verdicts

    def step():
        phase_eb()
        phase_x()
        phase_mlp()
        phase_or()

    def sync_all():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def maxr(x):
        if dist is None:
            return x
        t_ = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        return float(t_.item())

    stream = torch.cuda.current_stream()
    for _ in range(3):
        step()
    sync_all()
    eb.backend.raise_on_status()

    def graph_us(fn, reps):
        """Median device time of fn replayed as a CUDA graph (eager when capture fails), max over ranks."""
        sync_all()
        g, how = None, "CUDA graph replay"
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                fn()
            g.replay()
            sync_all()
        except Exception as e:  # noqa: BLE001  (capture unsupported here: time it eagerly)
            g, how = None, f"eager (graph capture failed: {type(e).__name__})"
            torch.cuda.synchronize()
        run = g.replay if g is not None else fn
        ts = []
        for _ in range(reps):
            sync_all()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(maxr(e0.elapsed_time(e1) * 1e3))
        del g
        return statistics.median(ts), how

    # per-phase device times (each phase captured alone), then the whole step
    phase_us = {}
    for name, fn in (("eb_lookups", phase_eb), ("exchange", phase_x), ("mlp", phase_mlp),
                     ("mlp_as_9_launches", phase_mlp_separate), ("verdict_or", phase_or)):
        if name == "verdict_or" and G == 1:
            phase_us[name] = 0.0  # no collective at one rank
            continue
        phase_us[name] = graph_us(fn, 5)[0]
    # the grouped MLP writes exactly what the 9 launches write (C', checksum column, verdicts)
    c_sep = [c.clone() for *_x, c, _cs, _er in mlp]
    phase_mlp()
    torch.cuda.synchronize()
    mlp_group_eq = all(torch.equal(c_sep[q], mlp[q][4]) for q in range(len(mlp)))
    step_us, how = graph_us(step, steps)
    sync_all()
    flagged_mlp = int(mflags.to(torch.int64).sum().item())
    out, fl = phase_x()
    flagged_eb = int(fl.to(torch.int64).sum().item())
    lookups_rank = len(mine) * B * pool
    # per lookup: the 128-B row, its 16-B metadata record (scale, bias, row sum), the 8-B index; per bag: offsets and
    # the pooled vector (+ its verdict quad in the exchange layout)
    alg_eb = lookups_rank * (d + 16 + 8) + len(mine) * (8 * (B + 1) + 4 * B * (d + S.FLAG_QUAD))
    x_bytes = int(eb.xsend.numel() * 4 * (G - 1) // G) if eb.local is None else 0
    ops = sum(2 * m * n_loc * k for k, n_loc, *_ in mlp)
    mlp_alg = sum(m * k + k * (n_loc + 1) + 4 * m * (n_loc + 1) + m for k, n_loc, *_ in mlp)
    L.lib.abftlp_gemm_group_free(mlp_group)
    for k, n_loc, w, *_ in mlp:
        L.lib.abftlp_gemm_weight_free(w)
    shard = mlp_shard_leg(L, dev, st, vp, pk, graph_us) if G == 1 else None
    res = {
        "workload": f"D5 = BASELINE configs[4] on {G} GPU(s): 64 tables x 1M x 128 int8 (table-wise, {len(mine)} per GPU), "
                    f"batch {B}, pooling {pool}, Zipf(1.05); exchange to [B/G, 64, 128]; 9 checked MLP GEMMs m={m} "
                    "(k, n/G), verdicts OR-reduced",
        "n_gpus": G, "step_us": step_us, "step_how": how, "phase_us": phase_us,
        "samples_per_s": B / (step_us * 1e-6),
        "eb_lookups_per_gpu": lookups_rank, "eb_alg_gbs_per_gpu": alg_eb / (phase_us["eb_lookups"] * 1e-6) / 1e9,
        "eb_hbm_frac": alg_eb / (phase_us["eb_lookups"] * 1e-6) / 1e9 / pk["hbm_gbs"],
        "exchange_bytes_out_per_gpu": x_bytes,
        "exchange_gbs_per_gpu": x_bytes / (phase_us["exchange"] * 1e-6) / 1e9 if G > 1 else None,
        "mlp_tops_per_gpu": ops / (phase_us["mlp"] * 1e-6) / 1e12,
        "mlp_how": "the 9 checked layers in ONE heterogeneous grouped launch (abftlp_gemm_group_run); "
                   "mlp_as_9_launches = the same GEMMs as 9 abftlp_gemm_checked launches",
        "mlp_group_eq_separate": bool(mlp_group_eq),
        "mlp_alg_bytes_per_gpu": mlp_alg,
        "mlp_hbm_frac": mlp_alg / (phase_us["mlp"] * 1e-6) / 1e9 / pk["hbm_gbs"],
        "flagged_bags_rank0_slice": flagged_eb, "flagged_mlp_rows": flagged_mlp,
        "group_fused": bool(group_ok),
    }
    if shard is not None:
        res["mlp_shard_g8"] = shard
    del tables, bags, eb
    torch.cuda.empty_cache()
    return res


def mlp_shard_leg(L, dev, st, vp, pk, graph_us, G=8):
    """One GPU's share of the D5 MLP at G=8 (the N-split layers m=8192, (k, n/8)), measured on this GPU: ONE grouped
    launch vs 9 launches, against its HBM roof (A read once per layer, C' and verdicts written)."""
    import torch
    m = 8192
    mlp, ws = [], []
    for q, (k, n) in enumerate([(k, n // G) for k in (512, 1024, 2048) for n in (512, 1024, 2048)]):
        gen = torch.Generator(device=dev)
        gen.manual_seed(7000 + q)
        b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device=dev, generator=gen)
        a = torch.randint(0, 256, (m, k), dtype=torch.uint8, device=dev, generator=gen)
        w = C.c_void_p()
        L.call("abftlp_gemm_encode", vp(b), k, n, n, st, C.byref(w))
        mlp.append((k, n, w, a, torch.empty((m, n), dtype=torch.int32, device=dev),
                    torch.empty(m, dtype=torch.int32, device=dev), torch.empty(m, dtype=torch.uint8, device=dev),
                    torch.zeros(1, dtype=torch.int32, device=dev)))
    probs = (L.GemmProblem * len(mlp))()
    for q, (k, n, w, a, c, cs, fl, er) in enumerate(mlp):
        probs[q] = L.GemmProblem(a.data_ptr(), m, k, w.value, c.data_ptr(), n, cs.data_ptr(), 1, fl.data_ptr(),
                                 er.data_ptr())
    grp = C.c_void_p()
    L.call("abftlp_gemm_group_create", probs, len(mlp), 1, C.byref(grp))

    def sep():
        for k, n, w, a, c, cs, fl, er in mlp:
            L.call("abftlp_gemm_checked", vp(a), m, k, w, vp(c), n, vp(cs), 1, vp(fl), vp(er), None, st)
    t_grp = graph_us(lambda: L.call("abftlp_gemm_group_run", grp, st), 8)[0]
    t_sep = graph_us(sep, 8)[0]

    def grp10():
        for _ in range(10):
            L.call("abftlp_gemm_group_run", grp, st)
    t_b2b = graph_us(grp10, 5)[0] / 10
    alg = sum(m * k + k * (n + 1) + 4 * m * (n + 1) + m for k, n, *_ in mlp)
    ops = sum(2 * m * n * k for k, n, *_ in mlp)
    L.lib.abftlp_gemm_group_free(grp)
    for _, _, w, *_ in mlp:
        L.lib.abftlp_gemm_weight_free(w)
    return {"grouped_us": t_grp, "as_9_launches_us": t_sep, "alg_bytes": alg, "hbm_roof_us": alg / pk["hbm_gbs"] / 1e3,
            "hbm_frac": alg / (t_grp * 1e-6) / 1e9 / pk["hbm_gbs"], "tops": ops / (t_grp * 1e-6) / 1e12,
            "grouped_us_back_to_back": t_b2b, "hbm_frac_back_to_back": alg / (t_b2b * 1e-6) / 1e9 / pk["hbm_gbs"],
            "b2b_how": "10 grouped launches in one CUDA graph / 10 (the graph's launch and event latency, ~6-8 us of a "
                       "one-launch graph, amortised; the 132 MB working set exceeds L2)",
            "how": "9 checked GEMMs m=8192, (k, n/8), k, n in {512,1024,2048}: one abftlp_gemm_group_run vs 9 "
                   "abftlp_gemm_checked launches, each as a CUDA graph; seeded synthetic A and B"}


def eb_secondary(L, dev, st, vp, pk):
    """E3 / E4 checked EmbeddingBag: algorithmic HBM GB/s (every lookup counted), L2 flushed per step."""
    import torch
    out = {}
    rng = np.random.default_rng(3)
    for name in ("E3", "E4", "E3_uniform"):
        if name.startswith("E3"):
            R, d, nb, elem, st_t, meta_b = 4_000_000, 128, 2048, 1, 0, 12
            lens = rng.integers(20, 101, nb)
            if name == "E3":
                ranks = np.arange(1, R + 1, dtype=np.float64)
                cdf = np.cumsum(ranks ** -1.05)
                cdf /= cdf[-1]
                perm = rng.permutation(R)
                idx = perm[np.searchsorted(cdf, rng.random(int(lens.sum())))].astype(np.int64)
            else:  # uniform-index control (no Zipf-hot rows served from L2)
                idx = rng.integers(0, R, int(lens.sum())).astype(np.int64)
            wts = None
            row_b = d
        else:
            R, d, nb, elem, st_t, meta_b = 8_000_000, 64, 4096, 2, 1, 8
            lens = rng.integers(1, 151, nb)
            idx = rng.integers(0, R, int(lens.sum())).astype(np.int64)
            wts = torch.from_numpy(rng.uniform(0, 1, int(lens.sum())).astype(np.float32)).to(dev)
            row_b = d // 2
        rows = torch.randint(0, 256, (R, row_b), dtype=torch.uint8, device=dev)
        sdt = torch.float32 if st_t == 0 else torch.float16
        sc = (torch.rand(R, device=dev) * 9e-3 + 1e-3).to(sdt)
        bi = (torch.rand(R, device=dev) * 2 - 1).to(sdt)
        off = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)).to(dev)
        ix = torch.from_numpy(idx).to(dev)
        tab = C.c_void_p()
        L.call("abftlp_eb_table_create", elem, vp(rows), R, d, row_b, st_t, vp(sc), vp(bi), None, st, C.byref(tab))
        n_faults = 0
        if name == "E4":  # BASELINE configs[3]: one random bit flip in 0.1% of the rows, after the row sums
            vic = torch.from_numpy(rng.choice(R, R // 1000, replace=False).astype(np.int64)).to(dev)
            fc = torch.from_numpy(rng.integers(0, d, R // 1000).astype(np.int64)).to(dev)
            fbits = torch.from_numpy(rng.integers(0, 4, R // 1000).astype(np.int32)).to(dev)
            L.call("abftlp_eb_table_flip_bits", tab, vp(vic), vp(fc), vp(fbits), R // 1000, None, st)
            n_faults = R // 1000
        o = torch.empty((nb, d), dtype=torch.float32, device=dev)
        fl = torch.empty(nb, dtype=torch.uint8, device=dev)
        fb = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        L_ = int(lens.sum())
        alg = L_ * (row_b + meta_b + 4 + 8 + (4 if wts is not None else 0)) + 8 * (nb + 1) + 4 * nb * d + nb
        res = {}
        for checked in (True, False):
            ts = []
            for s in range(8):
                L.call("abftlp_l2_flush", vp(fb), fb.numel(), s, st)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                if checked:
                    L.call("abftlp_eb_checked", tab, vp(off), vp(ix), nb, vp(wts) if wts is not None else None,
                           vp(o), d, vp(fl), None, None, None, None, st)
                else:
                    L.call("abftlp_eb_unchecked", tab, vp(off), vp(ix), nb, vp(wts) if wts is not None else None,
                           vp(o), d, None, st)
                e1.record()
                torch.cuda.synchronize()
                if s >= 2:
                    ts.append(e0.elapsed_time(e1) * 1e3)
            res[checked] = statistics.median(ts)
        # steady state: 20 batches back to back (programmatic dependent launch overlaps launch and tail)
        def b2b():
            for _ in range(20):
                L.call("abftlp_eb_checked", tab, vp(off), vp(ix), nb, vp(wts) if wts is not None else None, vp(o), d,
                       vp(fl), None, None, None, None, st)
        b2b()
        L.call("abftlp_l2_flush", vp(fb), fb.numel(), 77, st)
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b2b()
        e1.record()
        torch.cuda.synchronize()
        b2b_us = e0.elapsed_time(e1) * 1e3 / 20
        # random-gather floor of the same lookups (abftlp_gather_probe): every looked-up record read once with
        # maximal memory-level parallelism and no arithmetic, L2 flushed -- the practical roof for these batches
        rec = 128 if row_b > 64 else 64  # E3: the 128-B rows; E4: the table's packed 64-B row+meta records
        gtab = rows if rec == row_b else torch.empty((R, rec), dtype=torch.uint8, device=dev)
        sink = torch.zeros(1, dtype=torch.int32, device=dev)
        fts = []
        for s_ in range(5):
            L.call("abftlp_l2_flush", vp(fb), fb.numel(), 50 + s_, st)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            L.call("abftlp_gather_probe", vp(gtab), rec, vp(ix), L_, vp(sink), st)
            e1.record()
            torch.cuda.synchronize()
            fts.append(e0.elapsed_time(e1) * 1e3)
        floor_us = statistics.median(fts[1:])
        del gtab
        flagged = int(fl.to(torch.int64).sum().item())
        L.lib.abftlp_eb_table_free(tab)
        gbs = alg / (res[True] * 1e-6) / 1e9
        out[name] = {"roofline": {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                                  "frac": gbs / pk["hbm_gbs"], "alg_bytes": alg,
                                  "kernel": "eb_bag_async_kernel (checked), one launch after an L2 flush",
                                  "practical_floor_us": floor_us, "frac_of_practical_floor": floor_us / res[True]},
                     "checked_us": res[True], "unchecked_us": res[False], "alg_bytes": alg, "alg_gbs": gbs,
                     "hbm_frac": gbs / pk["hbm_gbs"], "overhead_pct": 100 * (res[True] - res[False]) / res[False],
                     "lookups": L_, "bags": nb, "injected_row_faults": n_faults, "flagged_bags": flagged,
                     "gather_floor_us": floor_us, "frac_of_gather_floor": floor_us / res[True],
                     "checked_us_back_to_back": b2b_us,
                     "b2b_how": "20 batches back to back on one stream (same bags), after one L2 flush",
                     "gather_floor_how": f"abftlp_gather_probe: the {L_} looked-up {rec}-B records, L2 flushed"}
        del rows, sc, bi, off, ix, o, fl, fb
        torch.cuda.empty_cache()
    return out


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-eb", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-d5", action="store_true")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N` outside a launcher: re-run as N ranks, one process per GPU, exactly as the
        # driver's torchrun launch does (rendezvous on 127.0.0.1)
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
        os.execvpe(sys.executable, cmd, env)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"[bench] note: --gpus {args.gpus} but WORLD_SIZE={world}; running {world} rank(s)", file=sys.stderr)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    dist = None
    if world > 1 or os.environ.get("ABFT_BENCH_FORCE_DIST"):  # (the switch runs the N-rank code paths on one rank)
        import torch
        import torch.distributed as tdist
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (rank count) on stderr
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        local = int(os.environ.get("LOCAL_RANK", 0))
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist
        print(f"[bench] rank {rank}: torch.distributed nccl world_size={tdist.get_world_size()} "
              f"device={torch.cuda.get_device_name(local)}:{local}", file=sys.stderr, flush=True)
    run_gpu_arm(args, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
