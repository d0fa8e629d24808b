"""numpy wrappers over the C oracle (oracle/liboracle.so) and the reference shim (oracle/_ref).

TEST INFRASTRUCTURE: used only as the checker of the CUDA library.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
_ORC = None
_REF = None


def orc():
    global _ORC
    if _ORC is None:
        _ORC = C.CDLL(str(REPO / "oracle" / "liboracle.so"))
        _ORC.orc_mod127.restype = C.c_int32
        _ORC.orc_mod127.argtypes = [C.c_int64]
        _ORC.orc_verify_checksums.restype = C.c_uint64
        _ORC.orc_packed_at.restype = C.c_int8
        _ORC.orc_pack_len.restype = C.c_size_t
        _ORC.orc_half_to_float.restype = C.c_float
        _ORC.orc_half_to_float.argtypes = [C.c_uint16]
        _ORC.orc_draw_bit_index.restype = C.c_uint
    return _ORC


def ref():
    global _REF
    if _REF is None:
        p = REPO / "oracle" / "_ref" / "libabftlp_ref.so"
        if not p.exists():
            return None
        _REF = C.CDLL(str(p))
        _REF.ref_mod127.restype = C.c_int32
        _REF.ref_mod127.argtypes = [C.c_int64]
        _REF.ref_gemm_weight_new.restype = C.c_void_p
        _REF.ref_eb_table_new.restype = C.c_void_p
    return _REF


def P(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def sz(v):
    return C.c_size_t(int(v))


# ---------------------------------------------------------------- generators (reference draw protocol)
def gen_u8(seed, stream, skip, count):
    out = np.empty(count, np.uint8)
    orc().orc_gen_u8(C.c_uint64(seed), C.c_uint64(stream), C.c_uint64(skip), C.c_uint64(count), P(out))
    return out


def gen_s8(seed, stream, skip, count):
    out = np.empty(count, np.int8)
    orc().orc_gen_s8(C.c_uint64(seed), C.c_uint64(stream), C.c_uint64(skip), C.c_uint64(count), P(out))
    return out


def gen_real_f32(seed, stream, skip, count, lo, hi):
    out = np.empty(count, np.float32)
    orc().orc_gen_real_f32(C.c_uint64(seed), C.c_uint64(stream), C.c_uint64(skip), C.c_uint64(count), C.c_double(lo),
                           C.c_double(hi), P(out))
    return out


def gen_below(seed, stream, skip, count, bound):
    out = np.empty(count, np.int64)
    orc().orc_gen_below(C.c_uint64(seed), C.c_uint64(stream), C.c_uint64(skip), C.c_uint64(count), C.c_uint64(bound),
                        P(out))
    return out


def splitmix(seed, stream, count, lib=None):
    out = np.empty(count, np.uint64)
    fn = (lib or orc()).orc_splitmix64 if lib is None else lib.ref_splitmix64
    fn(C.c_uint64(seed), C.c_uint64(stream), C.c_uint64(count), P(out))
    return out


def gemm_inputs(seed, trial, m, n, k):
    """A then B from SplitMix64(seed, 4*trial) exactly as P:src/fault_lab.cpp:180-183."""
    a = gen_u8(seed, trial * 4, 0, m * k).reshape(m, k)
    b = gen_s8(seed, trial * 4, m * k, k * n).reshape(k, n)
    return a, b


# ---------------------------------------------------------------- GEMM
def mod127(v):
    return int(orc().orc_mod127(int(v)))


def row_checksums(b):
    b = np.ascontiguousarray(b, np.int8)
    cs = np.empty(b.shape[0], np.int8)
    rc = orc().orc_compute_row_checksums(P(b), sz(b.shape[0]), sz(b.shape[1]), P(cs))
    if rc:
        raise ValueError("compute_row_checksums: empty matrix")
    return cs


def abft_gemm(a, b, cs=None):
    """-> (cTemp m x (n+1) int32, flags uint8[m], errCount)"""
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.int8)
    m, k = a.shape
    n = b.shape[1]
    ct = np.empty((m, n + 1), np.int32)
    fl = np.empty(m, np.uint8)
    err = C.c_uint64()
    csp = None if cs is None else np.ascontiguousarray(cs, np.int8)
    orc().orc_abft_gemm(P(a), sz(m), sz(k), P(b), sz(n), P(csp), P(ct), P(fl), C.byref(err))
    return ct, fl, int(err.value)


def plain_gemm(a, b):
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.int8)
    c = np.empty((a.shape[0], b.shape[1]), np.int32)
    orc().orc_plain_gemm(P(a), sz(a.shape[0]), sz(a.shape[1]), P(b), sz(b.shape[1]), P(c))
    return c


def verify(ctemp):
    ctemp = np.ascontiguousarray(ctemp, np.int32)
    fl = np.empty(ctemp.shape[0], np.uint8)
    e = orc().orc_verify_checksums(P(ctemp), sz(ctemp.shape[0]), sz(ctemp.shape[1]), P(fl))
    return int(e), fl


def pack(b, cs, rb, cb):
    b = np.ascontiguousarray(b, np.int8)
    k, n = b.shape
    buf = np.empty(orc().orc_pack_len(sz(k), sz(n), sz(rb), sz(cb)), np.int8)
    orc().orc_pack_encoded(P(b), P(np.ascontiguousarray(cs, np.int8)), sz(k), sz(n), sz(rb), sz(cb), P(buf))
    return buf


def packed_at(buf, n, rb, cb, i, j):
    return int(orc().orc_packed_at(P(buf), sz(n), sz(rb), sz(cb), sz(i), sz(j)))


def dual_product(a, b):
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.int8)
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m + 1, n + 1), np.int64)
    orc().orc_dual_encoded_product(P(a), sz(m), sz(k), P(b), sz(n), P(c))
    return c


def dual_check(c):
    c = np.ascontiguousarray(c, np.int64)
    i, j = C.c_size_t(), C.c_size_t()
    kind = orc().orc_dual_encoded_check(P(c), sz(c.shape[0] - 1), sz(c.shape[1] - 1), C.byref(i), C.byref(j))
    return kind, int(i.value), int(j.value)


# ---------------------------------------------------------------- EmbeddingBag
ELEM = {"s8": 0, "u8": 1, "u4": 2}


def row_sums(rows, elem="s8", dim=None):
    rows = np.ascontiguousarray(rows).view(np.uint8)
    R, rb = rows.shape
    d = dim or (rb * 2 if elem == "u4" else rb)
    out = np.empty(R, np.int32)
    orc().orc_precompute_row_sums(ELEM[elem], P(rows), sz(R), sz(d), sz(rb), P(out))
    return out


def eb(rows, scales, biases, offsets, indices, weights=None, elem="s8", dim=None, row_sums_=None, checked=True):
    """-> (r[B,d] f32, rsum f64[B], csum f64[B], err u8[B]); raises IndexError on out-of-range."""
    rows = np.ascontiguousarray(rows).view(np.uint8)
    R, rb = rows.shape
    d = dim or (rb * 2 if elem == "u4" else rb)
    scales = np.ascontiguousarray(scales)
    st = 1 if scales.dtype in (np.float16, np.uint16) else 0
    sc = scales.view(np.uint16) if st else scales.astype(np.float32)
    bi = np.ascontiguousarray(biases)
    bi = bi.view(np.uint16) if st else bi.astype(np.float32)
    off = np.ascontiguousarray(offsets, np.int64)
    idx = np.ascontiguousarray(indices, np.int64)
    w = None if weights is None else np.ascontiguousarray(weights, np.float32)
    nb = len(off) - 1
    r = np.zeros((nb, d), np.float32)
    rs = np.zeros(nb)
    cs = np.zeros(nb)
    er = np.zeros(nb, np.uint8)
    sums = None if row_sums_ is None else np.ascontiguousarray(row_sums_, np.int32)
    rc = orc().orc_eb_bags(ELEM[elem], st, P(rows), sz(R), sz(d), sz(rb), P(sc), P(bi), P(sums), P(off),
                           P(idx) if len(idx) else None, P(w), sz(nb), int(checked), P(r), P(rs), P(cs), P(er))
    if rc == -2:
        raise IndexError("embedding_bag: index out of range")
    return r, rs, cs, er


def half_to_float(h):
    return float(orc().orc_half_to_float(int(h)))


# ---------------------------------------------------------------- campaigns
TARGET = {"weight_b": 0, "intermediate_c": 1, "eb_table": 2, "none": 3}
MODEL = {"single_bit_flip": 0, "random_value": 1}
RANGE = {"all": 0, "high4": 1, "low4": 2}


def gemm_campaign(shapes, per, target, seed, model="single_bit_flip", rng="all", workers=8):
    sh = np.array([[m, n, k] for (m, n, k) in shapes], np.uint64).ravel()
    det = np.zeros(len(shapes) * per, np.uint8)
    rc = orc().orc_run_gemm_campaign(P(sh), sz(len(shapes)), sz(per), TARGET[target], MODEL[model], RANGE[rng],
                                     C.c_uint64(seed), sz(workers), P(det))
    assert rc == 0
    return det


def eb_campaign(R, d, pool, batch, trials, target, seed, model="single_bit_flip", rng="all", workers=8):
    det = np.zeros(trials, np.uint8)
    rc = orc().orc_run_eb_campaign(sz(R), sz(d), sz(pool), sz(batch), sz(trials), TARGET[target], MODEL[model],
                                   RANGE[rng], C.c_uint64(seed), sz(workers), P(det))
    assert rc == 0
    return det


def fnv1a64(arr: np.ndarray) -> str:
    h = 0xCBF29CE484222325
    for byte in np.ascontiguousarray(arr).view(np.uint8).tobytes():
        h ^= byte
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def sha256(arr: np.ndarray) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(arr).view(np.uint8).tobytes()).hexdigest()


# ---------------------------------------------------------------- requantization (P:src/quant.cpp:77-118)
def requantize(c, n, row_sum_a, col_sum_b, prm, k):
    """C' (m x ldc int32, only the first n columns read) -> u8 m x n; raises ValueError on scaleC <= 0."""
    c = np.ascontiguousarray(c, np.int32)
    m, ldc = c.shape
    rs = np.ascontiguousarray(row_sum_a, np.int32)
    cs = np.ascontiguousarray(col_sum_b, np.int32)
    p = np.ascontiguousarray(prm, np.float64)
    out = np.empty((m, n), np.uint8)
    rc = orc().orc_requantize(P(c), sz(ldc), sz(m), sz(n), P(rs), P(cs), P(p), C.c_uint64(int(k)), P(out), sz(n))
    if rc != 0:
        raise ValueError("requantize: scaleC must be positive")
    return out


def row_sums_u8(a):
    a = np.ascontiguousarray(a, np.uint8)
    out = np.empty(a.shape[0], np.int32)
    orc().orc_row_sums_u8(P(a), sz(a.shape[0]), sz(a.shape[1]), sz(a.shape[1]), P(out))
    return out


def col_sums_i8(b):
    b = np.ascontiguousarray(b, np.int8)
    out = np.empty(b.shape[1], np.int32)
    orc().orc_col_sums_i8(P(b), sz(b.shape[0]), sz(b.shape[1]), sz(b.shape[1]), P(out))
    return out
