"""The oracle is pinned before it is trusted (CPU only).

1. Known answers from the reference's own unit tests (P:tests/test_gemm_abft.cpp,
   P:tests/test_embedding_abft.cpp, P:tests/test_fault_lab.cpp, P:tests/acceptance.cpp).
2. Golden vectors produced by the real reference (tests/golden/*.json, oracle/make_golden.py).
3. Where oracle/_ref (the reference compiled from its sources) is present: direct comparison on
   random inputs.
"""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_api as O
from campaign_configs import CAMPAIGNS, GEMM_SHAPES

GOLD = Path(__file__).resolve().parent / "golden"


def gold(name):
    return json.loads((GOLD / f"{name}.json").read_text())["cases"]


# ------------------------------------------------------------------ known answers (reference unit tests)
def test_mod127_known_answers():  # P:tests/test_gemm_abft.cpp:31-38
    for v, r in [(0, 0), (6, 6), (200, 73), (-2, 125), (-127, 0), (381, 0)]:
        assert O.mod127(v) == r


def test_row_checksum_examples():  # P:tests/test_gemm_abft.cpp:40-51
    b = np.array([0, 0, 0, 1, 2, 3, 100, 100, 0, -1, -1, 0], np.int8).reshape(4, 3)
    assert O.row_checksums(b).tolist() == [0, 6, 73, 125]
    with pytest.raises(ValueError):
        O.row_checksums(np.zeros((0, 3), np.int8))


def test_pack_round_trip_and_padding():  # P:tests/test_gemm_abft.cpp:53-90
    rng = np.random.default_rng(11)
    for k, n, rb, cb in [(4, 4, 2, 2), (3, 5, 2, 4), (64, 17, 64, 16), (1, 1, 8, 8), (7, 129, 3, 5)]:
        b = rng.integers(-128, 128, (k, n)).astype(np.int8)
        cs = O.row_checksums(b)
        buf = O.pack(b, cs, rb, cb)
        assert len(buf) == -(-k // rb) * -(-(n + 1) // cb) * rb * cb
        for i in range(k):
            for j in range(n):
                assert O.packed_at(buf, n, rb, cb, i, j) == b[i, j]
            assert O.packed_at(buf, n, rb, cb, i, n) == cs[i]
    b = np.full((3, 5), -7, np.int8)
    buf = O.pack(b, O.row_checksums(b), 2, 4)
    assert len(buf) == 32 and int((buf == 0).sum()) == 14


def test_identity_hand_oracle_and_forced_corruption():  # P:tests/test_gemm_abft.cpp:98-116
    a = np.array([[1, 0], [0, 1]], np.uint8)
    b = np.array([[3, 4], [5, 6]], np.int8)
    ct, fl, err = O.abft_gemm(a, b)
    assert err == 0 and ct.tolist() == [[3, 4, 7], [5, 6, 11]]
    ct[0, 1] = 5
    assert O.verify(ct)[0] == 1
    ct0, _, err0 = O.abft_gemm(np.random.default_rng(12).integers(0, 256, (3, 4)).astype(np.uint8),
                               np.zeros((4, 2), np.int8))
    assert err0 == 0 and not ct0.any()


def test_verify_rows_including_aliasing():  # P:tests/test_gemm_abft.cpp:126-132
    c = np.array([[3, 4, 7], [3, 4, 6], [200, 181, 0]], np.int32)
    err, flags = O.verify(c)
    assert err == 1 and flags.tolist() == [0, 1, 0]


def test_soundness_and_residue_congruence():  # P:tests/test_gemm_abft.cpp:134-157, acceptance criterion 5
    rng = np.random.default_rng(14)
    for _ in range(300):
        m, n, k = int(rng.integers(1, 17)), int(rng.integers(1, 65)), int(rng.integers(1, 65))
        a = rng.integers(0, 256, (m, k)).astype(np.uint8)
        b = rng.integers(-128, 128, (k, n)).astype(np.int8)
        cs = O.row_checksums(b)
        ct, _, err = O.abft_gemm(a, b)
        assert err == 0
        via = a.astype(np.int64) @ cs.astype(np.int64)
        assert np.array_equal(ct[:, :n].astype(np.int64).sum(1) % 127, via % 127)
        assert np.array_equal(ct[:, n].astype(np.int64) % 127, via % 127)
        assert np.array_equal(ct[:, :n], (a.astype(np.int64) @ b.astype(np.int64)).astype(np.int32))


def test_aliasing_sweep():  # P:tests/test_gemm_abft.cpp:159-171
    rng = np.random.default_rng(15)
    a = rng.integers(0, 256, (4, 8)).astype(np.uint8)
    b = rng.integers(-128, 128, (8, 6)).astype(np.int8)
    clean, _, err = O.abft_gemm(a, b)
    assert err == 0
    for delta in range(-260, 261):
        c = clean.copy()
        c[2, 3] += delta
        assert (O.verify(c)[0] > 0) == (delta % 127 != 0)


def test_single_bit_flips_coprime_to_127():  # P:tests/test_gemm_abft.cpp:173-175
    assert all((1 << l) % 127 for l in range(32))


def test_dual_encoded_oracle_locates_single_faults():  # P:tests/test_gemm_abft.cpp:177-209
    rng = np.random.default_rng(17)
    a = rng.integers(0, 256, (5, 7)).astype(np.uint8)
    b = rng.integers(-128, 128, (7, 6)).astype(np.int8)
    pristine = O.dual_product(a, b)
    assert O.dual_check(pristine)[0] == 0
    for i in range(pristine.shape[0]):
        for j in range(pristine.shape[1]):
            c = pristine.copy()
            c[i, j] += 1
            assert O.dual_check(c) == (1, i, j)
    c = pristine.copy()
    c[1, 2] += 5
    c[3, 4] -= 9
    assert O.dual_check(c)[0] == 2


def test_eb_known_answers():  # P:tests/test_embedding_abft.cpp:44-118
    assert O.row_sums(np.zeros((3, 4), np.int8)).tolist() == [0, 0, 0]
    assert O.row_sums(np.array([[1, -1, 5]], np.int8)).tolist() == [5]
    rng = np.random.default_rng(34)
    rows = rng.integers(-128, 128, (100, 16)).astype(np.int8)
    idx = rng.integers(0, 100, 50)
    off = np.array([0, 50])
    r, rs, cs, er = O.eb(rows, np.ones(100, np.float32), np.zeros(100, np.float32), off, idx)
    assert rs[0] == cs[0] and er[0] == 0  # integer path is exact (82-90)
    r, rs, cs, er = O.eb(rows, np.ones(100, np.float32), np.zeros(100, np.float32), np.array([0, 0]),
                         np.zeros(0, np.int64))
    assert rs[0] == 0.0 and cs[0] == 0.0 and er[0] == 0 and not r.any()  # empty bag (111-118)
    with pytest.raises(IndexError):
        O.eb(rows, np.ones(100, np.float32), np.zeros(100, np.float32), np.array([0, 1]), np.array([100]))


def test_eb_sign_flip_detected_and_weights_of_one_identical():  # P:tests/test_embedding_abft.cpp:101-132
    rng = np.random.default_rng(36)
    R, d = 1000, 64
    rows = rng.integers(-128, 128, (R, d)).astype(np.int8)
    sc = rng.uniform(0.005, 0.02, R).astype(np.float32)
    bi = rng.uniform(-1, 1, R).astype(np.float32)
    idx = rng.integers(0, R, 100)
    off = np.array([0, 100])
    sums = O.row_sums(rows)
    r0, rs0, cs0, e0 = O.eb(rows, sc, bi, off, idx, row_sums_=sums)
    r1, rs1, cs1, e1 = O.eb(rows, sc, bi, off, idx, weights=np.ones(100, np.float32), row_sums_=sums)
    assert np.array_equal(r0.view(np.uint32), r1.view(np.uint32)) and rs0[0] == rs1[0] and cs0[0] == cs1[0]
    bad = rows.copy()
    bad[idx[7], 11] ^= np.int8(-128)
    assert O.eb(bad, sc, bi, off, idx, row_sums_=sums)[3][0] == 1


def test_u4_and_f16_decode_against_numpy():
    rng = np.random.default_rng(5)
    R, d = 50, 64
    packed = rng.integers(0, 256, (R, d // 2)).astype(np.uint8)
    elems = np.empty((R, d), np.int64)
    elems[:, 0::2] = packed & 0xF
    elems[:, 1::2] = packed >> 4
    assert np.array_equal(O.row_sums(packed, "u4"), elems.sum(1))
    h = rng.uniform(-2, 2, 1000).astype(np.float16)
    assert all(O.half_to_float(x) == float(v) for x, v in zip(h.view(np.uint16), h))
    for special in (0x0001, 0x03FF, 0x8000, 0x7BFF, 0xFBFF):
        assert O.half_to_float(special) == float(np.array([special], np.uint16).view(np.float16)[0])


def test_fault_lab_draws():  # P:tests/test_fault_lab.cpp:41-65
    for r in range(200):
        assert 4 <= O.orc().orc_draw_bit_index(C.c_uint64(51), C.c_uint64(r), 1, 8) <= 7
        assert O.orc().orc_draw_bit_index(C.c_uint64(51), C.c_uint64(r), 2, 8) <= 3


def test_inject_before_encoding_is_absorbed():  # P:tests/test_fault_lab.cpp:121-133
    rng = np.random.default_rng(54)
    a = rng.integers(0, 256, (4, 16)).astype(np.uint8)
    b = rng.integers(-128, 128, (16, 12)).astype(np.int8)
    rec = np.zeros(5, np.int64)
    O.orc().orc_inject_weight_B(O.P(b), O.sz(16), O.sz(12), 0, 0, 0, C.c_uint64(99), C.c_uint64(0), O.P(rec))
    assert rec[0] == 1 and rec[3] != rec[4]
    assert O.abft_gemm(a, b)[2] == 0


# ------------------------------------------------------------------ golden vectors from the reference
def test_rng_golden():
    for c in gold("rng"):
        got = O.splitmix(c["seed"], c["stream"], 8)
        assert [str(int(x)) for x in got] == c["draws"]


@pytest.mark.parametrize("case", [c for c in gold("gemm") if c["label"] != "G2"], ids=lambda c: f"{c['label']}t{c['trial']}")
def test_gemm_golden(case):
    m, n, k = case["m"], case["n"], case["k"]
    a, b = O.gemm_inputs(case["seed"], case["trial"], m, n, k)
    cs = O.row_checksums(b)
    assert cs[:8].tolist() == case["cs_head"] and O.sha256(cs) == case["cs_sha"]
    ct, _, err = O.abft_gemm(a, b)
    assert O.sha256(ct) == case["ctemp_sha"] and err == case["err"] == 0
    assert int(ct.astype(np.int64).sum()) == case["ctemp_sum"]
    if "c_fault" in case:
        f = case["c_fault"]
        rec = np.zeros(5, np.int64)
        c2 = ct.copy()
        O.orc().orc_inject_intermediate_C(O.P(c2), O.sz(m), O.sz(n + 1), 1, 0, 0, C.c_uint64(case["seed"]),
                                          C.c_uint64(case["trial"]), O.P(rec))
        assert (rec[1], rec[2], rec[3], rec[4]) == (f["i"], f["j"], f["before"], f["after"])
        assert O.verify(c2)[0] == f["err"]
        fb = case["b_fault"]
        b2 = b.copy()
        O.orc().orc_inject_weight_B(O.P(b2), O.sz(k), O.sz(n), 0, 0, 0, C.c_uint64(case["seed"]),
                                    C.c_uint64(case["trial"]), O.P(rec))
        assert (rec[1], rec[2], rec[3], rec[4]) == (fb["i"], fb["j"], fb["before"], fb["after"])
        ctb, _, errb = O.abft_gemm(a, b2, cs=cs)
        assert O.sha256(ctb) == fb["ctemp_sha"] and errb == fb["err"]


def test_eb_golden():
    cases = gold("eb")
    fp_trials = cases[-1]["control_false_positive_trials"]
    assert len(fp_trials) == 7
    for c in cases[:-1]:
        Rn, d, pool, batch, t, seed = c["R"], c["d"], c["pool"], c["batch"], c["trial"], c["seed"]
        rows = O.gen_s8(seed, 4 * t, 0, Rn * d).reshape(Rn, d)
        sc = O.gen_real_f32(seed, 4 * t, Rn * d, Rn, 0.005, 0.02)
        bi = O.gen_real_f32(seed, 4 * t, Rn * d + Rn, Rn, -1.0, 1.0)
        idx = O.gen_below(seed, 4 * t + 2, 0, pool * batch, Rn)
        assert O.sha256(rows) == c["rows_sha"] and O.sha256(sc) == c["scales_sha"] and O.sha256(idx) == c["idx_sha"]
        w = O.gen_real_f32(seed, c["weights_stream"], 0, pool * batch, 0.0, 1.0) if c["weighted"] else None
        off = np.arange(0, pool * batch + 1, pool)
        r, rs, cs, er = O.eb(rows, sc, bi, off, idx, w)
        assert O.sha256(r) == c["r_sha"]
        assert [float(x).hex() for x in rs] == c["rsum_hex"] and [float(x).hex() for x in cs] == c["csum_hex"]
        assert er.tolist() == c["err"]


@pytest.mark.parametrize("name", list(CAMPAIGNS))
def test_campaign_counts_oracle(name):
    """The C restatement reproduces the reference's campaign outcomes exactly."""
    text, (trials, detected, fp) = CAMPAIGNS[name]
    assert gold("campaigns")[name] == [trials, detected, fp]
    if name.startswith("gemm"):
        per = 20 if name == "gemm_smoke" else 200
        shapes = [(1, 32, 32), (4, 48, 16), (8, 16, 64)] if name == "gemm_smoke" else GEMM_SHAPES
        seed = 1 if name == "gemm_smoke" else 20260823
        target = {"gemm_control": "none", "gemm_bitflip_c": "intermediate_c", "gemm_bitflip_b": "weight_b",
                  "gemm_smoke": "intermediate_c"}[name]
        det = O.gemm_campaign(shapes, per, target, seed)
    else:
        target = "none" if name == "eb_control" else "eb_table"
        rng = {"eb_high4": "high4", "eb_low4": "low4"}.get(name, "all")
        det = O.eb_campaign(20000, 64, 100, 10, trials, target, 31, rng=rng)
        if name == "eb_control":
            assert np.nonzero(det)[0].tolist() == gold("eb")[-1]["control_false_positive_trials"]
    got = int(det.sum())
    assert (got if target != "none" else 0) == detected and (got if target == "none" else 0) == fp


# ------------------------------------------------------------------ direct comparison with oracle/_ref
def test_oracle_matches_reference_random(ref):
    R = O.ref()
    rng = np.random.default_rng(99)
    for _ in range(60):
        m, n, k = (int(x) for x in rng.integers(1, 40, 3))
        a = rng.integers(0, 256, (m, k)).astype(np.uint8)
        b = rng.integers(-128, 128, (k, n)).astype(np.int8)
        ct = np.empty((m, n + 1), np.int32)
        err = C.c_uint64()
        assert R.ref_abft_gemm(O.P(a), O.sz(m), O.sz(k), O.P(b), O.sz(n), O.P(ct), C.byref(err)) == 0
        mine, _, e2 = O.abft_gemm(a, b)
        assert np.array_equal(ct, mine) and err.value == e2
    for trial in range(3):
        Rn, d, nb = 3000, [16, 64, 128][trial], 40
        rows = rng.integers(-128, 128, (Rn, d)).astype(np.int8)
        sc = rng.uniform(1e-3, 1e-2, Rn).astype(np.float32)
        bi = rng.uniform(-1, 1, Rn).astype(np.float32)
        lens = rng.integers(0, 120, nb)
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        idx = rng.integers(0, Rn, off[-1]).astype(np.int64)
        w = rng.uniform(-2, 2, off[-1]).astype(np.float32) if trial == 2 else None
        r_ref = np.zeros((nb, d), np.float32)
        rs_ref, cs_ref, e_ref = np.zeros(nb), np.zeros(nb), np.zeros(nb, np.uint8)
        assert R.ref_batch_abft_eb(O.P(rows), O.sz(Rn), O.sz(d), O.P(sc), O.P(bi), None, O.P(off.astype(np.uint64)),
                                   O.P(idx.astype(np.uint64)), O.P(w), O.sz(nb), O.P(r_ref), O.P(rs_ref),
                                   O.P(cs_ref), O.P(e_ref)) == 0
        r, rs, cs, er = O.eb(rows, sc, bi, off, idx, w)
        assert np.array_equal(r.view(np.uint32), r_ref.view(np.uint32))
        assert np.array_equal(rs.view(np.uint64), rs_ref.view(np.uint64))
        assert np.array_equal(cs.view(np.uint64), cs_ref.view(np.uint64))
        assert np.array_equal(er, e_ref)


# ---------------------------------------------------------------- requantization
def _requant_case(seed):
    from golden_cases import requant_inputs
    return requant_inputs(seed)


def test_requant_known_answers():  # P:tests/test_quant.cpp:125-144, 186-202
    z = O.requantize(np.zeros((2, 2), np.int32), 2, [0, 0], [0, 0], [1, 0, 1, 0, 1, 0], 2)
    assert not z.any()
    assert O.requantize(np.zeros((1, 1), np.int32), 1, [0], [0], [1, 0, 1, 0, 1, -300.2], 1)[0, 0] == 255
    with pytest.raises(ValueError):
        O.requantize(np.zeros((2, 2), np.int32), 2, [0, 0], [0, 0], [1, 0, 1, 0, 0.0, 0], 1)
    rng = np.random.default_rng(606)
    no_cs = rng.integers(-100000, 100000, (3, 4)).astype(np.int32)
    with_cs = np.concatenate([no_cs, rng.integers(-2 ** 31, 2 ** 31, (3, 1), dtype=np.int64).astype(np.int32)], 1)
    prm = [0.01, 0.2, 0.02, -0.1, 0.5, -3.0]
    a = O.requantize(no_cs, 4, [10, 20, 30], [1, 2, 3, 4], prm, 7)
    b = O.requantize(with_cs, 4, [10, 20, 30], [1, 2, 3, 4], prm, 7)
    assert np.array_equal(a, b)


def test_requant_golden():
    g = json.loads((GOLD / "requant.json").read_text())
    for case in g["cases"]:
        m, n, k, c, rs, cs, prm = _requant_case(case["seed"])
        assert (m, n, k) == (case["m"], case["n"], case["k"])
        out = O.requantize(c, n, rs, cs, prm, k)
        assert out.reshape(-1).tolist() == case["out"], case["seed"]


def test_row_col_sums_match_reference_semantics():
    rng = np.random.default_rng(7)
    a = rng.integers(0, 256, (9, 300)).astype(np.uint8)
    b = rng.integers(-128, 128, (300, 11)).astype(np.int8)
    assert np.array_equal(O.row_sums_u8(a), a.astype(np.int64).sum(1))
    assert np.array_equal(O.col_sums_i8(b), b.astype(np.int64).sum(0))
    R = O.ref()
    if R is not None:
        rr = np.empty(9, np.int32)
        R.ref_row_sums_u8(O.P(a), O.sz(9), O.sz(300), O.P(rr))
        cc = np.empty(11, np.int32)
        R.ref_col_sums_i8(O.P(b), O.sz(300), O.sz(11), O.P(cc))
        assert np.array_equal(rr, O.row_sums_u8(a)) and np.array_equal(cc, O.col_sums_i8(b))
