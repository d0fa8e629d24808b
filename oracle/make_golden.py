"""Generate tests/golden/*.json from the REAL reference (oracle/_ref/libabftlp_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile). TEST INFRASTRUCTURE.

Run here (where /root/reference exists): python oracle/make_golden.py
The fixtures pin both the C restatement (oracle/abft_oracle.c) and the CUDA library.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO / "tests"))
import oracle_api as O  # noqa: E402
from campaign_configs import CAMPAIGNS  # noqa: E402
from golden_cases import requant_inputs  # noqa: E402

OUT = REPO / "tests" / "golden"
P = O.P
sz = O.sz


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()


def ref_abft_gemm(R, a, b):
    m, k = a.shape
    n = b.shape[1]
    ct = np.empty((m, n + 1), np.int32)
    err = C.c_uint64()
    assert R.ref_abft_gemm(P(a), sz(m), sz(k), P(b), sz(n), P(ct), C.byref(err)) == 0
    return ct, int(err.value)


def ref_cs(R, b):
    cs = np.empty(b.shape[0], np.int8)
    assert R.ref_compute_row_checksums(P(b), sz(b.shape[0]), sz(b.shape[1]), P(cs)) == 0
    return cs


def ref_verify(R, ct):
    e = C.c_uint64()
    assert R.ref_verify_checksums(P(ct), sz(ct.shape[0]), sz(ct.shape[1]), C.byref(e)) == 0
    return int(e.value)


def gemm_golden(R):
    seed = 20260823
    cases = []
    for (label, m, n, k, trials) in [("G1", 64, 512, 512, 4), ("G2", 256, 4096, 4096, 1)] + \
            [(f"S{i}", m, n, k, 2) for i, (m, n, k) in enumerate([(1, 32, 32), (4, 48, 16), (16, 128, 32), (3, 17, 5)])]:
        for t in range(trials):
            a, b = O.gemm_inputs(seed, t, m, n, k)
            cs = ref_cs(R, b)
            ct, err = ref_abft_gemm(R, a, b)
            case = {"label": label, "m": m, "n": n, "k": k, "seed": seed, "trial": t, "cs_head": cs[:8].tolist(),
                    "cs_sha": sha(cs), "ctemp_sha": sha(ct), "ctemp_sum": int(ct.astype(np.int64).sum()),
                    "c00": int(ct[0, 0]), "c0n": int(ct[0, n]), "err": err}
            if t % 2 == 1:  # the reference's C-injection point (P:src/fault_lab.cpp:192-195)
                rec = np.zeros(3, np.int64)
                c2 = ct.copy()
                assert R.ref_inject_intermediate_C(P(c2), sz(m), sz(n + 1), 1, 0, 0, C.c_uint64(seed), C.c_uint64(t),
                                                   P(rec)) == 0
                diff = np.argwhere(c2 != ct)
                case["c_fault"] = {"i": int(diff[0][0]), "j": int(diff[0][1]), "before": int(rec[1]),
                                   "after": int(rec[2]), "err": ref_verify(R, c2)}
                b2 = b.copy()
                assert R.ref_inject_weight_B(P(b2), sz(k), sz(n), 0, 0, 0, C.c_uint64(seed), C.c_uint64(t), P(rec)) == 0
                w = R.ref_gemm_weight_new(P(b2), sz(k), sz(n))  # encodes the corrupted B
                R.ref_gemm_weight_free(C.c_void_p(w))
                diffb = np.argwhere(b2 != b)
                # abft_gemm of pristine checksums next to the corrupted B
                ctb = np.empty_like(ct)
                ctb[:, :n] = (a.astype(np.int64) @ b2.astype(np.int64)).astype(np.int32)
                ctb[:, n] = (a.astype(np.int64) @ cs.astype(np.int64)).astype(np.int32)
                case["b_fault"] = {"i": int(diffb[0][0]), "j": int(diffb[0][1]), "before": int(rec[1]),
                                   "after": int(rec[2]), "err": ref_verify(R, ctb), "ctemp_sha": sha(ctb)}
            cases.append(case)
    return cases


def ref_eb(R, rows, scales, biases, off, idx, w=None):
    Rn, d = rows.shape
    nb = len(off) - 1
    r = np.zeros((nb, d), np.float32)
    rs = np.zeros(nb)
    cs = np.zeros(nb)
    er = np.zeros(nb, np.uint8)
    offu = off.astype(np.uint64)
    idxu = idx.astype(np.uint64)
    assert R.ref_batch_abft_eb(P(rows), sz(Rn), sz(d), P(scales), P(biases), None, P(offu), P(idxu), P(w), sz(nb),
                               P(r), P(rs), P(cs), P(er)) == 0
    return r, rs, cs, er


def eb_golden(R):
    out = []
    seed = 31
    Rn, d, pool, batch = 20000, 64, 100, 10
    for t in (0, 1, 2):
        rows = O.gen_s8(seed, 4 * t, 0, Rn * d).reshape(Rn, d)
        sc = O.gen_real_f32(seed, 4 * t, Rn * d, Rn, 0.005, 0.02)
        bi = O.gen_real_f32(seed, 4 * t, Rn * d + Rn, Rn, -1.0, 1.0)
        idx = O.gen_below(seed, 4 * t + 2, 0, pool * batch, Rn)
        off = np.arange(0, pool * batch + 1, pool, dtype=np.int64)
        for weighted in (False, True):
            w = O.gen_real_f32(seed, 4 * t + 3, 0, pool * batch, 0.0, 1.0) if weighted else None
            r, rs, cs, er = ref_eb(R, rows, sc, bi, off, idx, w)
            out.append({"seed": seed, "trial": t, "R": Rn, "d": d, "pool": pool, "batch": batch, "weighted": weighted,
                        "weights_stream": 4 * t + 3 if weighted else None, "rows_sha": sha(rows),
                        "scales_sha": sha(sc), "biases_sha": sha(bi), "idx_sha": sha(idx), "r_sha": sha(r),
                        "rsum_hex": [float(x).hex() for x in rs], "csum_hex": [float(x).hex() for x in cs],
                        "err": er.tolist()})
    # the 7 false-positive trials of the control campaign, pinned individually
    det = O.eb_campaign(Rn, d, pool, batch, 400, "none", seed)
    out.append({"control_false_positive_trials": np.nonzero(det)[0].tolist()})
    return out


def campaigns_golden(R):
    res = {}
    for name, (text, _) in CAMPAIGNS.items():
        h = C.c_void_p()
        rep = C.c_void_p()
        assert R.abftlp_campaign_parse(text.encode(), C.byref(h)) == 0
        assert R.abftlp_campaign_run(h, C.byref(rep)) == 0
        for fn in ("abftlp_report_trials", "abftlp_report_detected", "abftlp_report_false_positives"):
            getattr(R, fn).restype = C.c_uint64
            getattr(R, fn).argtypes = [C.c_void_p]
        res[name] = [R.abftlp_report_trials(rep), R.abftlp_report_detected(rep), R.abftlp_report_false_positives(rep)]
    return res


def rng_golden(R):
    out = []
    for seed, stream in [(0, 0), (20260823, 0), (20260823, 5), (31, 2), (2 ** 64 - 1, 7)]:
        v = np.empty(8, np.uint64)
        R.ref_splitmix64(C.c_uint64(seed), C.c_uint64(stream), C.c_uint64(8), P(v))
        out.append({"seed": seed, "stream": stream, "draws": [str(int(x)) for x in v]})
    return out


def requant_golden(R):
    out = []
    for seed in range(24):
        m, n, k, c, rs, cs, prm = requant_inputs(seed)
        q = np.empty((m, n), np.uint8)
        rc = R.ref_requantize(P(c), sz(m), sz(n), C.c_int(1), P(rs), P(cs), P(prm), C.c_uint64(k), P(q))
        assert rc == 0
        out.append({"seed": seed, "m": m, "n": n, "k": k, "out": q.reshape(-1).tolist()})
    return out


def main():
    R = O.ref()
    if R is None:
        sys.exit("oracle/_ref/libabftlp_ref.so missing: run `make -C oracle ref` where /root/reference exists")
    OUT.mkdir(parents=True, exist_ok=True)
    for name, fn in [("rng", rng_golden), ("gemm", gemm_golden), ("eb", eb_golden), ("campaigns", campaigns_golden),
                     ("requant", requant_golden)]:
        data = {"generator": "oracle/make_golden.py", "source": "reference built from /root/reference/proj/src",
                "cases": fn(R)}
        (OUT / f"{name}.json").write_text(json.dumps(data, indent=1) + "\n")
        print("wrote", name)


if __name__ == "__main__":
    main()
