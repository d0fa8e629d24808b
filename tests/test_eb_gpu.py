"""Checked EmbeddingBag on the B200 vs the oracle: pooled vectors bit-identical (tolerance 0 ULP,
tighter than north_star's 1e-5 relative), rSum/cSum bit-identical in fp64, identical verdicts.
Mirrors P:tests/test_embedding_abft.cpp and acceptance criteria 7-8."""
import os
import tempfile

import numpy as np
import pytest
import torch

import oracle_api as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    from paper_2103_00130_b200 import embedding
    return embedding


def ref_table(seed, R, d):
    rng = np.random.default_rng(seed)
    rows = rng.integers(-128, 128, (R, d)).astype(np.int8)
    return rows, rng.uniform(0.005, 0.02, R).astype(np.float32), rng.uniform(-1, 1, R).astype(np.float32)


def assert_same(out, flags, rsum, csum, ref):
    r_ref, rs_ref, cs_ref, e_ref = ref
    assert np.array_equal(out.cpu().numpy().view(np.uint32), r_ref.view(np.uint32))
    if flags is not None:
        assert np.array_equal(rsum.cpu().numpy().view(np.uint64), rs_ref.view(np.uint64))
        assert np.array_equal(csum.cpu().numpy().view(np.uint64), cs_ref.view(np.uint64))
        assert np.array_equal(flags.cpu().numpy(), e_ref)


def test_row_sums(E):  # P:tests/test_embedding_abft.cpp:44-57
    assert E.precompute_row_sums(np.zeros((3, 4), np.int8)).cpu().tolist() == [0, 0, 0]
    assert E.precompute_row_sums(np.array([[1, -1, 5]], np.int8)).cpu().tolist() == [5]
    rows = np.random.default_rng(31).integers(-128, 128, (1000, 64)).astype(np.int8)
    assert np.array_equal(E.precompute_row_sums(rows).cpu().numpy(), rows.astype(np.int64).sum(1))
    u8 = np.random.default_rng(1).integers(0, 256, (500, 128)).astype(np.uint8)
    assert np.array_equal(E.precompute_row_sums(u8, "u8").cpu().numpy(), u8.astype(np.int64).sum(1))
    u4 = np.random.default_rng(2).integers(0, 256, (500, 32)).astype(np.uint8)
    assert np.array_equal(E.precompute_row_sums(u4, "u4").cpu().numpy(), O.row_sums(u4, "u4"))


def test_empty_identity_duplicate_lookups(E):  # P:tests/test_embedding_abft.cpp:59-74
    rows, sc, bi = ref_table(32, 20, 8)
    sc[3], bi[3] = 1.0, 0.0
    t = E.QuantEmbeddingTable(rows, sc, bi)
    assert not E.embedding_bag(t, E.IndexBag()).any()
    single = E.embedding_bag(t, E.IndexBag([3])).cpu().numpy()
    assert np.array_equal(single, rows[3].astype(np.float32))
    twice = E.embedding_bag(t, E.IndexBag([3, 3])).cpu().numpy()
    assert np.array_equal(twice, 2.0 * single)


def test_out_of_range(E):  # P:tests/test_embedding_abft.cpp:76-80
    t = E.QuantEmbeddingTable(*ref_table(33, 4, 4))
    with pytest.raises(IndexError):
        E.embedding_bag(t, E.IndexBag([4]))
    with pytest.raises(IndexError):
        E.batch_abft_eb(t, [E.IndexBag([0, 1]), E.IndexBag([2 ** 40])])


def test_integer_path_exact_and_empty_bag(E):  # P:tests/test_embedding_abft.cpp:82-118
    rows, _, _ = ref_table(34, 100, 16)
    t = E.QuantEmbeddingTable(rows, np.ones(100, np.float32), np.zeros(100, np.float32))
    res = E.abft_embedding_bag(t, E.IndexBag(np.random.default_rng(3).integers(0, 100, 50)))
    assert res.rSum == res.cSum and not res.err
    e = E.abft_embedding_bag(E.QuantEmbeddingTable(*ref_table(37, 10, 4)), E.IndexBag())
    assert not e.err and e.rSum == 0.0 and e.cSum == 0.0


def test_sign_flip_and_weights(E):  # P:tests/test_embedding_abft.cpp:101-143
    rows, sc, bi = ref_table(36, 1000, 64)
    bag = E.IndexBag(np.random.default_rng(4).integers(0, 1000, 100))
    t = E.QuantEmbeddingTable(rows, sc, bi)
    plain = E.abft_embedding_bag(t, bag)
    w1 = E.abft_embedding_bag(t, E.IndexBag(bag.indices, np.ones(100, np.float32)))
    assert torch.equal(plain.r, w1.r) and plain.rSum == w1.rSum and plain.cSum == w1.cSum
    t.flip_bit(int(bag.indices[7]), 11, 7)
    assert E.abft_embedding_bag(t, bag).err
    rng = np.random.default_rng(39)
    t2 = E.QuantEmbeddingTable(*ref_table(39, 500, 64))
    for _ in range(20):
        assert not E.abft_embedding_bag(t2, E.IndexBag(rng.integers(0, 500, 60), rng.uniform(-2, 2, 60))).err


def test_batch_only_targeted_bag_flagged(E):  # P:tests/test_embedding_abft.cpp:145-169
    rows, sc, bi = ref_table(40, 2000, 64)
    rng = np.random.default_rng(41)
    bags = [E.IndexBag(rng.integers(0, 2000, 100)) for _ in range(10)]
    t = E.QuantEmbeddingTable(rows, sc, bi)
    assert not any(r.err for r in E.batch_abft_eb(t, bags))
    used = set(int(i) for b in range(10) if b != 4 for i in bags[b].indices)
    victim = next(int(i) for i in bags[4].indices if int(i) not in used)
    t.flip_bit(victim, 3, 7)
    assert [r.err for r in E.batch_abft_eb(t, bags)] == [b == 4 for b in range(10)]


@pytest.mark.parametrize("elem,scale,R,d,nb,lo,hi,weighted", [
    ("s8", "f32", 1000, 128, 64, 20, 100, False), ("u8", "f32", 1000, 128, 64, 20, 100, True),
    ("u4", "f16", 2000, 64, 64, 1, 150, True), ("s8", "f32", 500, 64, 40, 0, 100, True),
    ("u8", "f16", 3000, 128, 50, 0, 80, False), ("s8", "f32", 100, 8, 10, 0, 5, False),
    ("u4", "f32", 300, 16, 10, 1, 9, True), ("s8", "f32", 400, 256, 30, 1, 90, False),
    ("u8", "f32", 200, 32, 30, 1, 90, True), ("s8", "f32", 100, 96, 10, 3, 40, False),
    ("u4", "f16", 1000, 128, 33, 1, 200, False), ("s8", "f16", 700, 200, 20, 0, 70, True)])
def test_bit_exact_vs_oracle(E, elem, scale, R, d, nb, lo, hi, weighted):
    rng = np.random.default_rng(R + d + nb)
    rb = d // 2 if elem == "u4" else d
    rows = rng.integers(0 if elem != "s8" else -128, 256 if elem != "s8" else 128, (R, rb)).astype(
        np.int8 if elem == "s8" else np.uint8)
    sdt = np.float16 if scale == "f16" else np.float32
    sc = rng.uniform(1e-3, 1e-2, R).astype(sdt)
    bi = rng.uniform(-1, 1, R).astype(sdt)
    lens = rng.integers(lo, hi + 1, nb)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = rng.integers(0, R, off[-1]).astype(np.int64)
    w = rng.uniform(0, 1, off[-1]).astype(np.float32) if weighted else None
    t = E.QuantEmbeddingTable(rows, sc, bi, elem=elem, dim=d)
    ref = O.eb(rows, sc, bi, off, idx, w, elem=elem, dim=d)
    out, flags, rsum, csum, cnt = E.eb_csr(t, off, idx, w)
    assert_same(out, flags, rsum, csum, ref)
    assert int(cnt.item()) == int(ref[3].sum())
    out_u, *_ = E.eb_csr(t, off, idx, w, checked=False)
    assert torch.equal(out_u, out)


@pytest.mark.parametrize("cfg", ["E3", "E4"])
def test_baseline_configs_full_size(E, cfg):
    """BASELINE configs 2 and 3 at full size: 4M x 128 u8 (Zipf bags) and 8M x 64 int4 + fp16 with weights,
    bit-exact against the oracle, then a row-flip batch (0.1% of rows) with identical verdicts."""
    rng = np.random.default_rng(3 if cfg == "E3" else 4)
    if cfg == "E3":
        R, d, nb, elem, sdt = 4_000_000, 128, 2048, "u8", np.float32
        lens = rng.integers(20, 101, nb)
        ranks = np.arange(1, R + 1, dtype=np.float64)
        cdf = np.cumsum(ranks ** -1.05)
        cdf /= cdf[-1]
        perm = rng.permutation(R)
        idx = perm[np.searchsorted(cdf, rng.random(int(lens.sum())))].astype(np.int64)
        w = None
    else:
        R, d, nb, elem, sdt = 8_000_000, 64, 4096, "u4", np.float16
        lens = rng.integers(1, 151, nb)
        idx = rng.integers(0, R, int(lens.sum())).astype(np.int64)
        w = rng.uniform(0, 1, int(lens.sum())).astype(np.float32)
    rb = d if elem == "u8" else d // 2
    rows_t = torch.randint(0, 256, (R, rb), dtype=torch.uint8, device="cuda")
    rows = rows_t.cpu().numpy()
    sc = rng.uniform(1e-3, 1e-2, R).astype(sdt)
    bi = rng.uniform(-1, 1, R).astype(sdt)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    t = E.QuantEmbeddingTable(rows_t, sc, bi, elem=elem, dim=d)
    out, flags, rsum, csum, _ = E.eb_csr(t, off, idx, w)
    ref = O.eb(rows, sc, bi, off, idx, w, elem=elem, dim=d)
    assert_same(out, flags, rsum, csum, ref)
    # flip one random bit in 0.1% of the rows (after row sums), compare verdicts with the oracle
    victims = rng.choice(R, R // 1000, replace=False)
    width = 8 if elem == "u8" else 4
    cols = rng.integers(0, d, len(victims))
    bits = rng.integers(0, width, len(victims))
    for r_, c_, b_ in zip(victims[:64], cols[:64], bits[:64]):  # through the C ABI injector
        t.flip_bit(int(r_), int(c_), int(b_))
    # the rest through the batched device injector (abftlp_eb_table_flip_bits)
    t.flip_bits(victims[64:], cols[64:], bits[64:])
    torch.cuda.synchronize()
    rows2 = rows_t.cpu().numpy()  # the injector also mutates the caller's (borrowed) rows
    sums = O.row_sums(rows, elem, d)
    ref2 = O.eb(rows2, sc, bi, off, idx, w, elem=elem, dim=d, row_sums_=sums)
    out2, flags2, rsum2, csum2, _ = E.eb_csr(t, off, idx, w)
    assert_same(out2, flags2, rsum2, csum2, ref2)


def test_table_file_round_trip(E):  # P:tests/test_embedding_abft.cpp:171-195
    rows, sc, bi = ref_table(41, 64, 16)
    t = E.QuantEmbeddingTable(rows, sc, bi)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.abeb")
        E.save_table(t, p)
        lt = E.load_table(p)
        assert np.array_equal(lt.rows.cpu().numpy(), rows)
        assert np.array_equal(lt.rowSums.cpu().numpy(), O.row_sums(rows))
        stale = E.QuantEmbeddingTable(rows, sc, bi, row_sums=O.row_sums(rows) + np.eye(1, 64, 5, dtype=np.int32)[0])
        E.save_table(stale, p)
        from paper_2103_00130_b200 import _lib
        with pytest.raises(_lib.IoError):
            E.load_table(p)
        E.load_table(p, validateRowSums=False)
        with open(p, "wb") as f:
            f.write(b"NOPE")
        with pytest.raises(_lib.IoError):
            E.load_table(p)
    with pytest.raises(_lib.IoError):
        E.load_table("/nonexistent/abft.tbl")


@pytest.mark.parametrize("elem,scale,d,weighted,wpb", [("s8", "f32", 128, False, "1"), ("u4", "f16", 64, True, "1"),
                                                       ("u8", "f32", 128, True, "2"), ("s8", "f16", 256, False, "4"),
                                                       ("u8", "f32", 64, False, "2")])
def test_many_bags_per_group_bit_exact(E, elem, scale, d, weighted, wpb, monkeypatch):
    """Far more bags than resident bag groups (every group works through many bags, including empty ones and
    runs of them), on each warps-per-bag split: bit-exact against the oracle, including the flag count."""
    monkeypatch.setenv("ABFTLP_EB_WPB", wpb)
    rng = np.random.default_rng(d * 7 + int(wpb))
    R, nb = 3000, 30000
    rb = d // 2 if elem == "u4" else d
    rows = rng.integers(0 if elem != "s8" else -128, 256 if elem != "s8" else 128, (R, rb)).astype(
        np.int8 if elem == "s8" else np.uint8)
    sdt = np.float16 if scale == "f16" else np.float32
    sc = rng.uniform(1e-3, 1e-2, R).astype(sdt)
    bi = rng.uniform(-1, 1, R).astype(sdt)
    lens = rng.integers(0, 41, nb)
    lens[rng.random(nb) < 0.1] = 0  # 10 % empty bags, some consecutive
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = rng.integers(0, R, off[-1]).astype(np.int64)
    w = rng.uniform(0, 1, off[-1]).astype(np.float32) if weighted else None
    t = E.QuantEmbeddingTable(rows, sc, bi, elem=elem, dim=d)
    # corrupt a few rows after the row sums (the stored sums stay those of the clean rows), so bags are flagged
    rows_now = rows.copy().view(np.uint8)
    for r in rng.choice(R, 20, replace=False):
        col, bit = int(rng.integers(0, d)), int(rng.integers(0, 4))
        t.flip_bit(int(r), col, bit)
        if elem == "u4":
            rows_now[r, col // 2] ^= np.uint8(1 << (bit + 4 * (col & 1)))
        else:
            rows_now[r, col] ^= np.uint8(1 << bit)
    ref = O.eb(rows_now.view(rows.dtype), sc, bi, off, idx, w, elem=elem, dim=d, row_sums_=O.row_sums(rows, elem, d))
    out, flags, rsum, csum, cnt = E.eb_csr(t, off, idx, w)
    assert_same(out, flags, rsum, csum, ref)
    assert int(cnt.item()) == int(ref[3].sum()) > 0


def test_gather_probe_runs_and_validates(E):
    """abftlp_gather_probe (the bench's random-gather roof): runs on a table and rejects bad record sizes."""
    import ctypes as C
    from paper_2103_00130_b200 import _lib
    tab = torch.zeros((1000, 64), dtype=torch.uint8, device="cuda")
    idx = torch.randint(0, 1000, (5000,), dtype=torch.int64, device="cuda")
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    _lib.call("abftlp_gather_probe", vp(tab), 64, vp(idx), 5000, vp(sink), None)
    torch.cuda.synchronize()
    with pytest.raises(_lib.InvalidArgument):
        _lib.call("abftlp_gather_probe", vp(tab), 24, vp(idx), 5000, vp(sink), None)


@pytest.mark.parametrize("elem,scale,d,weighted", [("s8", "f32", 256, False), ("u8", "f16", 256, True),
                                                   ("u4", "f32", 256, True), ("s8", "f32", 128, True),
                                                   ("u4", "f16", 64, False), ("u8", "f32", 32, False)])
def test_sync_fast_path_bit_exact(E, elem, scale, d, weighted, monkeypatch):
    """The 8-byte-aligned (non-cp.async) warp-per-bag kernel, forced with ABFTLP_EB_SYNC: bit-exact against the
    oracle on 1, 2, 4 and 8 columns per lane, with faulted rows flagged."""
    monkeypatch.setenv("ABFTLP_EB_SYNC", "1")
    rng = np.random.default_rng(d * 13 + len(elem))
    R, nb = 2000, 700
    rb = d // 2 if elem == "u4" else d
    rows = rng.integers(0 if elem != "s8" else -128, 256 if elem != "s8" else 128, (R, rb)).astype(
        np.int8 if elem == "s8" else np.uint8)
    sdt = np.float16 if scale == "f16" else np.float32
    sc = rng.uniform(1e-3, 1e-2, R).astype(sdt)
    bi = rng.uniform(-1, 1, R).astype(sdt)
    lens = rng.integers(0, 90, nb)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = rng.integers(0, R, off[-1]).astype(np.int64)
    w = rng.uniform(0, 1, off[-1]).astype(np.float32) if weighted else None
    t = E.QuantEmbeddingTable(rows, sc, bi, elem=elem, dim=d)
    rows_now = rows.copy().view(np.uint8)
    for r in rng.choice(R, 10, replace=False):
        col, bit = int(rng.integers(0, d)), int(rng.integers(0, 4))
        t.flip_bit(int(r), col, bit)
        if elem == "u4":
            rows_now[r, col // 2] ^= np.uint8(1 << (bit + 4 * (col & 1)))
        else:
            rows_now[r, col] ^= np.uint8(1 << bit)
    ref = O.eb(rows_now.view(rows.dtype), sc, bi, off, idx, w, elem=elem, dim=d, row_sums_=O.row_sums(rows, elem, d))
    out, flags, rsum, csum, cnt = E.eb_csr(t, off, idx, w)
    assert_same(out, flags, rsum, csum, ref)
    assert int(cnt.item()) == int(ref[3].sum()) > 0
    out_u, *_ = E.eb_csr(t, off, idx, w, checked=False)
    assert torch.equal(out_u, out)
