"""Checked int8 GEMM on the B200 vs the oracle: bit-exact C', checksum column, per-row flags and
errCount. Mirrors P:tests/test_gemm_abft.cpp and acceptance criteria 1-5 (P:tests/acceptance.cpp)."""
import ctypes as C
import json
import os
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle_api as O

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def G():
    from paper_2103_00130_b200 import gemm
    return gemm


def rnd(seed, m, n, k):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, (m, k)).astype(np.uint8), rng.integers(-128, 128, (k, n)).astype(np.int8)


def check_against_oracle(G, a, b, **kw):
    pb = G.PackedEncodedWeight(b)
    res = G.abft_gemm(a, pb, **kw)
    ct_ref, fl_ref, err_ref = O.abft_gemm(a, b)
    ct = res.cTemp.data.cpu().numpy()
    assert np.array_equal(ct, ct_ref)
    assert np.array_equal(res.rowFlags.cpu().numpy(), fl_ref)
    assert res.errCount == err_ref
    return res


def test_known_answers(G):  # P:tests/test_gemm_abft.cpp:40-116
    b = np.array([0, 0, 0, 1, 2, 3, 100, 100, 0, -1, -1, 0], np.int8).reshape(4, 3)
    assert G.compute_row_checksums(b).values.cpu().tolist() == [0, 6, 73, 125]
    pb = G.PackedEncodedWeight(np.array([[5]], np.int8))
    assert pb.at(0, 0) == 5 and pb.at(0, 1) == 5
    res = G.abft_gemm(np.array([[1, 0], [0, 1]], np.uint8), G.PackedEncodedWeight(np.array([[3, 4], [5, 6]], np.int8)))
    assert res.errCount == 0 and res.cTemp.data.cpu().tolist() == [[3, 4, 7], [5, 6, 11]]
    res.cTemp.data[0, 1] = 5
    assert G.verify_checksums(res.cTemp) == 1
    zero = G.abft_gemm(np.random.default_rng(12).integers(0, 256, (3, 4)).astype(np.uint8),
                       G.PackedEncodedWeight(np.zeros((4, 2), np.int8)))
    assert zero.errCount == 0 and not zero.cTemp.data.any()


def test_error_paths(G):  # P:tests/test_gemm_abft.cpp:92-96, 118-132
    from paper_2103_00130_b200 import _lib
    with pytest.raises(_lib.InvalidArgument):
        G.PackedEncodedWeight(np.zeros((0, 3), np.int8))
    with pytest.raises(_lib.InvalidArgument):
        G.PackedEncodedWeight(np.ones((2, 2), np.int8), G.WeightChecksum(torch.ones(1, dtype=torch.int8)))
    a, b = rnd(13, 2, 2, 3)
    with pytest.raises(_lib.InvalidArgument):
        G.abft_gemm(a, G.PackedEncodedWeight(np.ones((4, 2), np.int8)))
    c = G.IntermediateMatrix(torch.tensor([[3, 4, 7], [3, 4, 6], [200, 181, 0]], dtype=torch.int32), True)
    assert G.verify_checksums(c) == 1
    with pytest.raises(_lib.InvalidArgument):
        G.verify_checksums(G.IntermediateMatrix(torch.tensor([[1, 2]], dtype=torch.int32), False))


def test_pack_round_trip(G):  # P:tests/test_gemm_abft.cpp:60-77 (at() contract)
    rng = np.random.default_rng(11)
    for k, n in [(4, 4), (3, 5), (64, 17), (1, 1), (7, 129), (300, 513)]:
        b = rng.integers(-128, 128, (k, n)).astype(np.int8)
        enc = G.PackedEncodedWeight(b).encoded().cpu().numpy()
        assert np.array_equal(enc[:, :n], b)
        assert np.array_equal(enc[:, n], O.row_checksums(b))


def test_encoder_tile_edges_and_reencode(G):
    """The one-kernel encoder (128 x 128 tiles, residues and arrivals in one atomic word): the checksum column's slot at
    a tile boundary (n % 128 == 0), padding rows inside the last k-block, the aligned 16-byte load path, and a second
    encode into the same handle (the scratch words reset themselves)."""
    rng = np.random.default_rng(21)
    for k, n in [(100, 128), (128, 256), (129, 128), (384, 512), (512, 384), (1000, 1024), (257, 2000)]:
        b = rng.integers(-128, 128, (k, n)).astype(np.int8)
        pb = G.PackedEncodedWeight(b)
        for _ in range(2):
            enc = pb.encoded().cpu().numpy()
            assert np.array_equal(enc[:, :n], b)
            assert np.array_equal(enc[:, n], O.row_checksums(b))
            pb.reencode(b)
    # extreme rows: every partial residue at its maximum
    b = np.full((256, 640), -128, np.int8)
    b[::2] = 127
    enc = G.PackedEncodedWeight(b).encoded().cpu().numpy()
    assert np.array_equal(enc[:, 640], O.row_checksums(b))


def test_encoder_very_wide_weight_takes_the_slab_encoder(G):
    """More than 2047 column tiles (n > 262 016) would overflow the tile encoder's arrival field: such weights are
    encoded by the one-block-per-row-slab kernel; same [B | cs]."""
    rng = np.random.default_rng(23)
    k, n = 130, 262_200
    b = rng.integers(-128, 128, (k, n)).astype(np.int8)
    enc = G.PackedEncodedWeight(b).encoded().cpu().numpy()
    assert np.array_equal(enc[:, :n], b) and np.array_equal(enc[:, n], O.row_checksums(b))


@pytest.mark.parametrize("k", [2056, 2057, 4112, 4113])
def test_row_sum_extremes_at_the_int32_bounds(G, k):
    """The epilogue sums a chunk's 32 (k <= 2056) or 16 (k <= 4112) columns in 32 bits: with every product at its
    extreme (A = 255, B = -128 or 127) those sums sit just inside int32; one k further the 64-bit path takes over."""
    for bv in (-128, 127):
        a = np.full((40, k), 255, np.uint8)
        b = np.full((k, 96), bv, np.int8)
        assert check_against_oracle(G, a, b).errCount == 0


@pytest.mark.parametrize("m,n,k,tiling", [(64, 1024, 256, "256"), (32, 256, 256, "256"), (200, 512, 1024, "128"),
                                            (300, 1024, 640, "64"), (64, 512, 512, None), (257, 768, 384, "256")])
def test_balanced_tiles_when_n_fills_its_tiles(G, m, n, k, tiling, monkeypatch):
    """n % BN == 0 at short K: the n + 1 columns split into balanced tiles narrower than BN (the MMA's N), the checksum
    column on the tensor cores; forced on and off, with faults on both sides of the checksum column."""
    a, b = rnd(3 * m + n + k, m, n, k)
    if tiling:
        monkeypatch.setenv("ABFTLP_GEMM_TILING", tiling)
    for tw in ("1", "0"):
        monkeypatch.setenv("ABFTLP_GEMM_TILEW", tw)
        assert check_against_oracle(G, a, b).errCount == 0
        pb = G.PackedEncodedWeight(b)
        for fault in ((m - 1, n - 1, 30), (0, n, 3), (m // 2, n // 2, 0)):
            res = G.abft_gemm(a, pb, fault=fault)
            ct, _, _ = O.abft_gemm(a, b)
            ct[fault[0], fault[1]] ^= np.int32(1 << fault[2])
            err_ref, fl_ref = O.verify(ct)
            assert np.array_equal(res.cTemp.data.cpu().numpy(), ct)
            assert np.array_equal(res.rowFlags.cpu().numpy(), fl_ref) and res.errCount == err_ref == 1


def test_random_small_products_bit_exact(G):  # P:tests/test_gemm_abft.cpp:134-157 / acceptance 5
    rng = np.random.default_rng(14)
    for _ in range(120):
        m, n, k = int(rng.integers(1, 17)), int(rng.integers(1, 65)), int(rng.integers(1, 65))
        a = rng.integers(0, 256, (m, k)).astype(np.uint8)
        b = rng.integers(-128, 128, (k, n)).astype(np.int8)
        res = check_against_oracle(G, a, b)
        assert res.errCount == 0


@pytest.mark.parametrize("m,n,k", [(64, 512, 512), (130, 300, 200), (256, 1024, 1024), (1, 3200, 800),
                                   (129, 257, 129), (8, 800, 3200), (300, 64, 4096), (513, 96, 48)])
def test_shapes_bit_exact(G, m, n, k):
    a, b = rnd(m * 7 + n, m, n, k)
    assert check_against_oracle(G, a, b).errCount == 0


@pytest.mark.parametrize("tiling", ["256", "128", "64", "256,2", "128,2", "64,2", "256,1", "128,1", "64,1",
                                    "128,0,2", "256,0,2", "256,1,2", "128,2,2"])
def test_g2_tilings_bit_exact(G, tiling, monkeypatch):
    """Every N-tile / split-K / epilogue variant gives the identical C' and verdicts."""
    monkeypatch.setenv("ABFTLP_GEMM_TILING", tiling)
    a, b = O.gemm_inputs(20260823, 0, 256, 4096, 4096)
    pb = G.PackedEncodedWeight(b)
    res = G.abft_gemm(a, pb)
    gold = [c for c in json.loads((GOLD / "gemm.json").read_text())["cases"] if c["label"] == "G2"][0]
    ct = res.cTemp.data.cpu().numpy()
    assert O.sha256(ct) == gold["ctemp_sha"]
    assert int(ct.astype(np.int64).sum()) == gold["ctemp_sum"]
    assert res.errCount == 0


@pytest.mark.parametrize("m,n,k,tiling", [(64, 512, 512, "128,0,2"), (130, 300, 1200, "128,0,2"),
                                          (256, 1000, 777, "64,0,2"), (33, 2049, 4096, "256,0,2"),
                                          (256, 4096, 4096, "128,0,2")])
def test_split_k_bit_exact_with_faults(G, m, n, k, tiling, monkeypatch):
    """Split-K units (partial tile handed over through L2) give the identical C', checksum column and
    verdicts, including the in-epilogue fault hook on both sides of the checksum column."""
    monkeypatch.setenv("ABFTLP_GEMM_TILING", tiling)
    a, b = rnd(m + 11 * n + k, m, n, k)
    pb = G.PackedEncodedWeight(b)
    for _ in range(2):  # the hand-over flags are self-resetting: a second call must see fresh partials
        res = G.abft_gemm(a, pb)
        ct, fl, err = O.abft_gemm(a, b)
        assert np.array_equal(res.cTemp.data.cpu().numpy(), ct) and res.errCount == err == 0
    for col in (n // 2, n):
        bad = G.abft_gemm(a, pb, fault=(m - 1, col, 30))
        assert bad.errCount == 1 and int(bad.rowFlags[m - 1].item()) == 1


def test_device_api_aligned_layout_matches_ctemp(G):
    """The perf layout (C ld n, separate csum, TMA epilogue) equals the reference layout."""
    from paper_2103_00130_b200 import _lib
    m, n, k = 256, 4096, 4096
    a, b = rnd(3, m, n, k)
    pb = G.PackedEncodedWeight(b)
    dev = torch.device("cuda")
    at = torch.from_numpy(a).to(dev)
    c = torch.empty((m, n), dtype=torch.int32, device=dev)
    cs = torch.empty(m, dtype=torch.int32, device=dev)
    fl = torch.empty(m, dtype=torch.uint8, device=dev)
    err = torch.empty(1, dtype=torch.int32, device=dev)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.call("abftlp_gemm_checked", C.c_void_p(at.data_ptr()), m, k, pb.handle, C.c_void_p(c.data_ptr()), n,
              C.c_void_p(cs.data_ptr()), 1, C.c_void_p(fl.data_ptr()), C.c_void_p(err.data_ptr()), None, st)
    ct_ref, fl_ref, err_ref = O.abft_gemm(a, b)
    assert np.array_equal(c.cpu().numpy(), ct_ref[:, :n]) and np.array_equal(cs.cpu().numpy(), ct_ref[:, n])
    assert int(err.item()) == err_ref == 0 and not fl.any()
    # unchecked kernel: same C
    c2 = torch.empty_like(c)
    _lib.call("abftlp_gemm_unchecked", C.c_void_p(at.data_ptr()), m, k, pb.handle, C.c_void_p(c2.data_ptr()), n, st)
    assert torch.equal(c, c2)
    # host-buffer (e2e) path
    ch = np.empty((m, n), np.int32)
    csh = np.empty(m, np.int32)
    flh = np.empty(m, np.uint8)
    eh = C.c_uint32()
    _lib.call("abftlp_gemm_checked_host", a.ctypes.data_as(C.c_void_p), m, k, pb.handle, ch.ctypes.data_as(C.c_void_p),
              n, csh.ctypes.data_as(C.c_void_p), flh.ctypes.data_as(C.c_void_p), C.byref(eh), st)
    assert np.array_equal(ch, ct_ref[:, :n]) and np.array_equal(csh, ct_ref[:, n]) and eh.value == 0


def test_golden_g1_trials_and_c_faults(G):
    """G1 (BASELINE config 0): reference draw protocol, odd trials flip one C' bit (in-epilogue hook)."""
    cases = [c for c in json.loads((GOLD / "gemm.json").read_text())["cases"] if c["label"] != "G2"]
    for case in cases:
        m, n, k = case["m"], case["n"], case["k"]
        a, b = O.gemm_inputs(case["seed"], case["trial"], m, n, k)
        pb = G.PackedEncodedWeight(b)
        res = G.abft_gemm(a, pb)
        assert O.sha256(res.cTemp.data.cpu().numpy()) == case["ctemp_sha"] and res.errCount == 0
        if "c_fault" in case:
            f = case["c_fault"]
            bit = int(np.log2(abs((f["after"] ^ f["before"]) & 0xFFFFFFFF)))
            hooked = G.abft_gemm(a, pb, fault=(f["i"], f["j"], bit))
            ct = hooked.cTemp.data.cpu().numpy()
            assert int(ct[f["i"], f["j"]]) == f["after"] and hooked.errCount == f["err"] == 1
            assert hooked.rowFlags.cpu().numpy().nonzero()[0].tolist() == [f["i"]]
            fb = case["b_fault"]
            bb = G.PackedEncodedWeight(b)
            bb.flip_bit(fb["i"], fb["j"], int(np.log2((fb["after"] ^ fb["before"]) & 0xFF)))
            rb = G.abft_gemm(a, bb)
            assert O.sha256(rb.cTemp.data.cpu().numpy()) == fb["ctemp_sha"] and rb.errCount == fb["err"]


def test_fault_hook_equals_post_hoc_injection(G):
    """Epilogue hook (fused) and inject-then-verify (reference protocol) give identical C' and verdicts,
    including hits on the checksum column."""
    rng = np.random.default_rng(21)
    for t in range(40):
        m, n, k = int(rng.integers(1, 300)), int(rng.integers(1, 700)), int(rng.integers(1, 700))
        a, b = rnd(t, m, n, k)
        pb = G.PackedEncodedWeight(b)
        i, j, bit = int(rng.integers(0, m)), int(rng.integers(0, n + 1)), int(rng.integers(0, 32))
        hooked = G.abft_gemm(a, pb, fault=(i, j, bit))
        post = G.abft_gemm(a, pb)
        post.cTemp.data[i, j] = int(np.int32(np.uint32(int(post.cTemp.data[i, j]) & 0xFFFFFFFF) ^ np.uint32(1 << bit)))
        assert torch.equal(hooked.cTemp.data, post.cTemp.data)
        assert hooked.errCount == G.verify_checksums(post.cTemp) == 1


def test_aliasing_sweep_on_device_verify(G):  # P:tests/test_gemm_abft.cpp:159-171
    a, b = rnd(15, 4, 6, 8)
    clean = G.abft_gemm(a, G.PackedEncodedWeight(b))
    assert clean.errCount == 0
    for delta in range(-260, 261, 3):
        c = G.IntermediateMatrix(clean.cTemp.data.clone(), True)
        c.data[2, 3] += delta
        assert (G.verify_checksums(c) > 0) == (delta % 127 != 0)


def test_plain_gemm_matches(G):
    a, b = rnd(5, 77, 333, 190)
    c = G.plain_gemm(a, b).data.cpu().numpy()
    assert np.array_equal(c, O.plain_gemm(a, b))


def test_g2_full_size_properties(G):
    """BASELINE config 1 at full size: residue identity row by row, and a fault in B' after encoding is
    caught in every row where A's value is not in {0, 127, 254} (the 3/256 aliasing law)."""
    a, b = O.gemm_inputs(20260823, 1, 256, 4096, 4096)
    pb = G.PackedEncodedWeight(b)
    res = G.abft_gemm(a, pb)
    ct = res.cTemp.data.cpu().numpy().astype(np.int64)
    assert res.errCount == 0
    assert np.array_equal(ct[:, :4096].sum(1) % 127, ct[:, 4096] % 127)
    i, j, bit = 1234, 777, 6
    pb.flip_bit(i, j, bit)
    bad = G.abft_gemm(a, pb)
    delta = int(np.int8(np.uint8(b[i, j]) ^ np.uint8(1 << bit))) - int(b[i, j])
    expect = ((a[:, i].astype(np.int64) * delta) % 127 != 0)
    assert np.array_equal(bad.rowFlags.cpu().numpy().astype(bool), expect)
    assert bad.errCount == int(expect.sum())


def test_empty_m(G):
    pb = G.PackedEncodedWeight(np.ones((4, 3), np.int8))
    res = G.abft_gemm(np.zeros((0, 4), np.uint8), pb)
    assert res.errCount == 0 and res.cTemp.data.shape == (0, 4)


@pytest.mark.parametrize("m,n,k", [(8192, 64, 2048), (4096, 200, 1000), (3000, 64, 777), (2050, 129, 640)])
def test_gemv_helpers_tall_narrow_bit_exact(G, m, n, k, monkeypatch):
    """Tall narrow shapes (the D5 MLP shards): the checksum column is computed by the pairs the tile grid
    leaves idle (gemv_helper) and added as one extra arrival per row. C', checksum column, verdicts and
    both fault sides are identical to the oracle, and identical with the helpers switched off."""
    a, b = rnd(m + 3 * n + k, m, n, k)
    pb = G.PackedEncodedWeight(b)
    ct, fl, err = O.abft_gemm(a, b)
    for helpers in ("1", "0"):
        monkeypatch.setenv("ABFTLP_GEMV_HELPERS", helpers)
        for _ in range(2):  # self-resetting row workspace
            res = G.abft_gemm(a, pb)
            assert np.array_equal(res.cTemp.data.cpu().numpy(), ct) and res.errCount == err == 0
        for col in (n // 2, n):
            bad = G.abft_gemm(a, pb, fault=(m - 1, col, 17))
            assert bad.errCount == 1 and int(bad.rowFlags[m - 1].item()) == 1


@pytest.mark.parametrize("m,n,k", [(8192, 64, 512), (1000, 100, 640), (300, 127, 1300)])
def test_single_tile_rows_bit_exact_and_workspace_clean(G, m, n, k, monkeypatch):
    """One N tile with the checksum column in the same tile (BN=128): each row has one contribution and is
    finalized without the row atomic. Verdicts with faults on both sides of the checksum column, repeated
    calls, and a following multi-tile call (which uses the shared per-row workspace) all stay exact."""
    monkeypatch.setenv("ABFTLP_GEMM_TILING", "128")
    a, b = rnd(7 * m + n + k, m, n, k)
    pb = G.PackedEncodedWeight(b)
    ct, fl, err = O.abft_gemm(a, b)
    for _ in range(2):
        res = G.abft_gemm(a, pb)
        assert np.array_equal(res.cTemp.data.cpu().numpy(), ct) and res.errCount == err == 0
    for row, col in ((0, n), (m - 1, n // 2), (m // 2, 0)):
        bad = G.abft_gemm(a, pb, fault=(row, col, 7))
        flags = bad.rowFlags.cpu().numpy()
        assert bad.errCount == 1 and flags[row] == 1 and int(flags.sum()) == 1
    monkeypatch.setenv("ABFTLP_GEMM_TILING", "64")  # n > 64: several tiles per row, row atomics again
    a2, b2 = rnd(m + 1, m, 2 * n, k)
    check_against_oracle(G, a2, b2)


def test_production_path_agrees_with_dual_encoded_oracle(G):  # P:tests/test_gemm_abft.cpp:211-236
    """50 ragged shapes (m, n, k in [1, 16]): the B200 C' equals the exact product block of the dual-encoded
    oracle (P:tests/dual_check.hpp:23-46); one bit flipped in C' is located by the dual check at its cell and
    flagged by the device verify."""
    rng = np.random.default_rng(19)
    for _ in range(50):
        m, n, k = (int(v) for v in rng.integers(1, 17, 3))
        a, b = rnd(int(rng.integers(1 << 30)), m, n, k)
        res = G.abft_gemm(a, G.PackedEncodedWeight(b))
        assert res.errCount == 0
        dual = O.dual_product(a, b)
        assert O.dual_check(dual)[0] == 0
        ct = res.cTemp.data.cpu().numpy()
        assert np.array_equal(ct[:, :n].astype(np.int64), dual[:m, :n])
        i, j, bit = int(rng.integers(m)), int(rng.integers(n)), int(rng.integers(32))
        before = int(ct[i, j])
        after = int(np.array([before], np.int32).view(np.uint32)[0] ^ np.uint32(1 << bit))
        after = int(np.array([after], np.uint32).view(np.int32)[0])
        res.cTemp.data[i, j] = after
        dual[i, j] += after - before
        assert O.dual_check(dual) == (1, i, j)
        assert G.verify_checksums(res.cTemp) > 0


@pytest.mark.parametrize("m,n,k,tiling,helpers", [(5, 300, 520, None, "1"), (16, 256, 1024, None, "1"),
                                                  (300, 512, 1000, "128", "0"), (300, 500, 1000, "128", "0"),
                                                  (8192, 64, 2048, None, "1"), (8192, 64, 2048, "64", "0")])
def test_checksum_sign_bit_flip_all_paths(G, m, n, k, tiling, helpers, monkeypatch):
    """A flipped sign bit of checksum-column elements (inject_weight_B at j == n; B' is int8, so cs becomes
    negative) multiplies as a SIGNED value on every path that forms C'[:, n]: the small-m GEMV, the epilogue's
    CUDA-core share (n % BN == 0), the tensor-core column (n % BN != 0) and the idle-pair GEMV helpers. C' and
    the verdicts equal the oracle's abft_gemm with the same corrupted checksums."""
    if tiling:
        monkeypatch.setenv("ABFTLP_GEMM_TILING", tiling)
    monkeypatch.setenv("ABFTLP_GEMV_HELPERS", helpers)
    a, b = rnd(m * 7 + n + k, m, n, k)
    pb = G.PackedEncodedWeight(b)
    cs = O.row_checksums(b).copy()
    for i in (0, k // 3, k - 1):
        pb.flip_bit(i, n, 7)
        cs[i] = np.int8(np.uint8(cs[i].view(np.uint8) ^ 0x80).view(np.int8))
        assert pb.at(i, n) == int(cs[i]) < 0
    res = G.abft_gemm(a, pb)
    ct, fl, err = O.abft_gemm(a, b, cs=cs)
    assert np.array_equal(res.cTemp.data.cpu().numpy(), ct)
    assert np.array_equal(res.rowFlags.cpu().numpy(), fl) and res.errCount == err
