"""Requantization on the B200 vs the oracle restatement of P:src/quant.cpp:77-118:
standalone kernel and the fused GEMM epilogue, bit-identical u8 outputs (tolerance 0)."""
import json
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle_api as O
from golden_cases import requant_inputs

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def Q():
    from paper_2103_00130_b200 import quant
    return quant


def _params(Q, prm, k):
    return Q.RequantParams(*[float(x) for x in prm], k=int(k))


def test_standalone_matches_golden(Q):
    from paper_2103_00130_b200.gemm import IntermediateMatrix
    g = json.loads((GOLD / "requant.json").read_text())
    for case in g["cases"]:
        m, n, k, c, rs, cs, prm = requant_inputs(case["seed"])
        out = Q.requantize(IntermediateMatrix(torch.from_numpy(c).cuda(), True), rs, cs, _params(Q, prm, k))
        assert out.cpu().numpy().reshape(-1).tolist() == case["out"], case["seed"]


def test_standalone_known_answers(Q):  # P:tests/test_quant.cpp:125-144
    from paper_2103_00130_b200 import _lib
    from paper_2103_00130_b200.gemm import IntermediateMatrix
    z = Q.requantize(IntermediateMatrix(torch.zeros((2, 2), dtype=torch.int32), False), [0, 0], [0, 0],
                     Q.RequantParams(1, 0, 1, 0, 1, 0, 2))
    assert not z.any()
    big = Q.requantize(IntermediateMatrix(torch.zeros((1, 1), dtype=torch.int32), False), [0], [0],
                       Q.RequantParams(1, 0, 1, 0, 1, -300.2, 1))
    assert int(big[0, 0]) == 255
    with pytest.raises(_lib.InvalidArgument):
        Q.requantize(IntermediateMatrix(torch.zeros((2, 2), dtype=torch.int32), False), [0, 0], [0, 0],
                     Q.RequantParams(scaleC=0.0))
    with pytest.raises(_lib.InvalidArgument):
        Q.requantize(IntermediateMatrix(torch.zeros((2, 2), dtype=torch.int32), False), [0], [0, 0],
                     Q.RequantParams())


def test_row_col_sums(Q):
    rng = np.random.default_rng(3)
    a = rng.integers(0, 256, (77, 1000)).astype(np.uint8)
    b = rng.integers(-128, 128, (1000, 300)).astype(np.int8)
    assert np.array_equal(Q.row_sums(a).cpu().numpy(), O.row_sums_u8(a))
    assert np.array_equal(Q.col_sums(b).cpu().numpy(), O.col_sums_i8(b))


@pytest.mark.parametrize("m,n,k,tiling", [(64, 512, 512, None), (256, 4096, 4096, None), (300, 700, 333, "128"),
                                          (33, 97, 64, "64"), (513, 1000, 1024, "256"), (256, 256, 128, "256,1")])
def test_fused_epilogue_matches_oracle(Q, m, n, k, tiling, monkeypatch):
    from paper_2103_00130_b200 import gemm as G
    if tiling:
        monkeypatch.setenv("ABFTLP_GEMM_TILING", tiling)
    a, b = O.gemm_inputs(20260823, 1, m, n, k)
    pb = G.PackedEncodedWeight(b)
    rs, cs = O.row_sums_u8(a), O.col_sums_i8(b)
    rng = np.random.default_rng(m + n + k)
    prm = [rng.uniform(1e-3, 0.05), rng.uniform(-0.5, 0.5), rng.uniform(1e-3, 0.05), rng.uniform(-0.5, 0.5),
           rng.uniform(1.0, 200.0), rng.uniform(-1000.0, 1000.0)]
    res, out = Q.abft_gemm_requant(a, pb, rs, cs, _params(Q, prm, k))
    ct, fl, err = O.abft_gemm(a, b)
    assert np.array_equal(res.cTemp.data.cpu().numpy(), ct) and res.errCount == err == 0
    ref = O.requantize(ct, n, rs, cs, prm, k)
    assert np.array_equal(out.cpu().numpy(), ref)
    # a fault in C' (col < n) is seen by the requantized output and flagged; C' not written when not kept
    r, col, bit = m // 2, n // 3, 17
    res2, out2 = Q.abft_gemm_requant(a, pb, rs, cs, _params(Q, prm, k), fault=(r, col, bit), keep_c=False)
    bad = ct.copy()
    bad[r, col:col + 1] = (bad[r, col:col + 1].view(np.uint32) ^ np.uint32(1 << bit)).view(np.int32)
    assert np.array_equal(out2.cpu().numpy(), O.requantize(bad, n, rs, cs, prm, k))
    assert res2.errCount == 1 and int(res2.rowFlags[r].item()) == 1
    assert not res2.cTemp.data[:, :n].any()  # int32 C' skipped


def test_dependent_chain_under_pdl_and_graph(Q):
    """GEMM i+1 consumes GEMM i's requantized u8 output as its A on the same stream, all enqueued without
    host synchronisation: the kernels overlap prologue/tail under programmatic dependent launch, so this
    checks that nothing reads A before griddepcontrol.wait. Run eagerly and as a replayed CUDA graph;
    every layer bit-exact vs the oracle."""
    import ctypes as C
    from paper_2103_00130_b200 import _lib
    from paper_2103_00130_b200 import gemm as G
    m, dims = 256, [512, 1024, 768, 512]
    rng = np.random.default_rng(77)
    a0 = rng.integers(0, 256, (m, dims[0])).astype(np.uint8)
    ws = [rng.integers(-128, 128, (dims[i], dims[i + 1])).astype(np.int8) for i in range(len(dims) - 1)]
    prm = [0.01, 0.1, 0.02, -0.05, 40.0, -20.0]
    pbs = [G.PackedEncodedWeight(w) for w in ws]
    css = [torch.from_numpy(O.col_sums_i8(w)).cuda() for w in ws]
    dev = torch.device("cuda")
    xs = [torch.from_numpy(a0).cuda()] + [torch.empty((m, dims[i + 1]), dtype=torch.uint8, device=dev)
                                          for i in range(len(ws))]
    cts = [torch.empty((m, dims[i + 1] + 1), dtype=torch.int32, device=dev) for i in range(len(ws))]
    rss = [torch.empty(m, dtype=torch.int32, device=dev) for _ in ws]
    fls = [torch.empty(m, dtype=torch.uint8, device=dev) for _ in ws]
    errs = torch.empty(len(ws) + 1, dtype=torch.int32, device=dev)
    prms = [_params(Q, prm, dims[i])._c() for i in range(len(ws))]
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    # a last plain checked GEMM reads the final requantized output directly: a GEMM -> GEMM PDL pair
    w_last = rng.integers(-128, 128, (dims[-1], 300)).astype(np.int8)
    pb_last = G.PackedEncodedWeight(w_last)
    ct_last = torch.empty((m, 301), dtype=torch.int32, device=dev)
    fl_last = torch.empty(m, dtype=torch.uint8, device=dev)

    def chain(st):
        for i, pb in enumerate(pbs):
            k, n = dims[i], dims[i + 1]
            _lib.call("abftlp_row_sums_u8", vp(xs[i]), m, k, k, vp(rss[i]), st)
            _lib.call("abftlp_gemm_checked_requant", vp(xs[i]), m, k, pb.handle, vp(cts[i]), n + 1,
                      C.c_void_p(cts[i].data_ptr() + 4 * n), n + 1, vp(fls[i]), C.c_void_p(errs.data_ptr() + 4 * i),
                      None, vp(rss[i]), vp(css[i]), C.byref(prms[i]), vp(xs[i + 1]), n, st)
        _lib.call("abftlp_gemm_checked", vp(xs[-1]), m, dims[-1], pb_last.handle, vp(ct_last), 301,
                  C.c_void_p(ct_last.data_ptr() + 4 * 300), 301, vp(fl_last), C.c_void_p(errs.data_ptr() + 4 * len(ws)),
                  None, st)

    ref_x = a0
    refs = []
    for i, w in enumerate(ws):
        ct, _, _ = O.abft_gemm(ref_x, w)
        ref_x = O.requantize(ct, w.shape[1], O.row_sums_u8(ref_x), O.col_sums_i8(w), prm, dims[i])
        refs.append((ct, ref_x))

    def check():
        torch.cuda.synchronize()
        for i, (ct, rx) in enumerate(refs):
            assert np.array_equal(cts[i].cpu().numpy(), ct), i
            assert np.array_equal(xs[i + 1].cpu().numpy(), rx), i
        assert np.array_equal(ct_last.cpu().numpy(), O.abft_gemm(refs[-1][1], w_last)[0])
        assert not errs.any()

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        chain(C.c_void_p(s.cuda_stream))
    check()
    for t in xs[1:] + cts + [ct_last]:
        t.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        chain(C.c_void_p(s.cuda_stream))
    with torch.cuda.stream(s):
        for _ in range(3):
            g.replay()
    check()


@pytest.mark.parametrize("batch,m,n,k", [(11, 64, 512, 512), (5, 256, 1024, 640), (3, 33, 97, 200), (1, 40, 256, 256)])
def test_host_batched_requant_job_matches_oracle(Q, batch, m, n, k):
    """abftlp_gemm_checked_requant_host_batched: pinned host u8 in, u8 out (the int32 product never leaves the GPU);
    every run's requantized output, checksum column, flags and count equal the oracle's abft_gemm + requantize
    (P:src/gemm_abft.cpp:93-100, P:src/quant.cpp:77-102), with row pitches that are not the staging pitches, and a
    corrupted B' (flipped after encoding) flags rows in every run."""
    import ctypes as C
    from paper_2103_00130_b200 import _lib as L
    from paper_2103_00130_b200 import gemm as G
    from paper_2103_00130_b200._device import stream_handle
    rng = np.random.default_rng(batch * 1000 + m)
    a = rng.integers(0, 256, (batch, m, k)).astype(np.uint8)
    b = rng.integers(-128, 128, (k, n)).astype(np.int8)
    prm = [rng.uniform(1e-3, 0.05), rng.uniform(-0.5, 0.5), rng.uniform(1e-3, 0.05), rng.uniform(-0.5, 0.5),
           rng.uniform(1.0, 200.0), rng.uniform(-1000.0, 1000.0)]
    pb = G.PackedEncodedWeight(b)
    lda, ldo = k + 3, n + 5
    ah = torch.zeros((batch, m, lda), dtype=torch.uint8).pin_memory()
    ah[:, :, :k] = torch.from_numpy(a)
    oh = torch.full((batch, m, ldo), 7, dtype=torch.uint8).pin_memory()
    csh = torch.zeros((batch, m), dtype=torch.int32).pin_memory()
    flh = torch.zeros((batch, m), dtype=torch.uint8).pin_memory()
    erh = torch.zeros(batch, dtype=torch.int32).pin_memory()
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731

    def run():
        L.call("abftlp_gemm_checked_requant_host_batched", vp(ah), batch, m, lda, m * lda, pb.handle,
               C.byref(_params(Q, prm, k)._c()), vp(oh), ldo, m * ldo, vp(csh), m, vp(flh), m, vp(erh), stream_handle())

    cs = O.col_sums_i8(b)
    for faulty in (False, True):
        bb = b.copy()
        if faulty:
            i, j, bit = k // 3, n // 2, 6
            pb.flip_bit(i, j, bit)
            bb[i, j] = np.int8(np.uint8(bb[i, j].view(np.uint8) ^ (1 << bit)).view(np.int8))
        run()
        for r in range(batch):
            ct, fl, err = O.abft_gemm(a[r], bb, cs=O.row_checksums(b))
            ref = O.requantize(ct, n, O.row_sums_u8(a[r]), cs if not faulty else O.col_sums_i8(bb), prm, k)
            assert np.array_equal(oh[r, :, :n].numpy(), ref), (faulty, r)
            assert (oh[r, :, n:] == 7).all()  # nothing written past a row's n bytes
            assert np.array_equal(csh[r].numpy(), ct[:, -1]) and np.array_equal(flh[r].numpy(), fl)
            assert int(erh[r]) == err and (err > 0 or not faulty or not a[r][:, k // 3].any())


@pytest.mark.parametrize("prm", [[1.0, 0.0, 1.0, 0.0, 2.0, 0.0],        # x = C/2: every odd C' sits on a boundary
                                 [1.0, 0.0, 1.0, 0.0, 4.0, 2.0],        # x = (C - 2)/4: quarters, halves, negatives
                                 [0.5, 1.0, 0.25, -2.0, 0.125, -3.0],   # exact binary fractions with row / column terms
                                 [1e6, 0.5, 1e6, -0.5, 1e3, 0.0],       # margin too wide for the fast path: all exact
                                 [1e-3, 0.0, 1e-3, 0.0, 1e-9, -1e-7]])  # tiny scaleC: saturates, margin too wide
def test_fused_epilogue_rounding_boundaries(Q, prm):
    """The fused epilogue's two-FMA fast path hands every element near a rounding boundary (and every launch whose
    error margin is not small) to the reference-order double sequence: products that land EXACTLY on j + 0.5, or on
    0 / 255.5, must give the reference's round-half-away bytes (P:src/quant.cpp:10-14, 77-102)."""
    from paper_2103_00130_b200 import gemm as G
    m, n, k = 70, 96, 16
    rng = np.random.default_rng(int(prm[4] * 1000) % 9973)
    a = rng.integers(0, 6, (m, k)).astype(np.uint8)
    b = rng.integers(-3, 7, (k, n)).astype(np.int8)
    pb = G.PackedEncodedWeight(b)
    rs, cs = O.row_sums_u8(a), O.col_sums_i8(b)
    res, out = Q.abft_gemm_requant(a, pb, rs, cs, _params(Q, prm, k))
    ct, _, _ = O.abft_gemm(a, b)
    ref = O.requantize(ct, n, rs, cs, prm, k)
    assert np.array_equal(out.cpu().numpy(), ref)
    if prm[4] == 2.0:
        assert (ct[:, :n] % 2 != 0).sum() > 1000  # the case does exercise exact halves


@pytest.mark.parametrize("m,n,k", [(300, 512, 640), (256, 4096, 4096), (70, 96, 128)])
def test_fused_epilogue_with_aligned_c_and_two_epilogue_groups(Q, m, n, k):
    """C' kept in a 16-byte-aligned layout (checksum column separate): the TMA-store epilogue, which fused-requant
    launches run with two epilogue groups splitting each tile's columns. C', checksum column, flags and the
    requantized bytes equal the oracle's (P:src/gemm_abft.cpp:93-124, P:src/quant.cpp:77-102), clean and with a C'
    fault."""
    import ctypes as C
    from paper_2103_00130_b200 import _lib as L
    from paper_2103_00130_b200 import gemm as G
    from paper_2103_00130_b200._device import stream_handle
    a, b = O.gemm_inputs(99, 2, m, n, k)
    pb = G.PackedEncodedWeight(b)
    rs, cs = O.row_sums_u8(a), O.col_sums_i8(b)
    prm = [0.013, -0.2, 0.021, 0.3, 55.0, -40.0]
    dev = torch.device("cuda")
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    ad = torch.from_numpy(a).to(dev)
    c = torch.zeros((m, n), dtype=torch.int32, device=dev)
    csum = torch.zeros(m, dtype=torch.int32, device=dev)
    fl = torch.zeros(m, dtype=torch.uint8, device=dev)
    er = torch.zeros(1, dtype=torch.int32, device=dev)
    out = torch.zeros((m, n), dtype=torch.uint8, device=dev)
    rsd, csd = torch.from_numpy(rs).to(dev), torch.from_numpy(cs).to(dev)
    ct, flr, err = O.abft_gemm(a, b)
    for fault in (None, (m // 2, n // 3, 19)):
        f = C.byref(L.Fault(1, *fault)) if fault else None
        L.call("abftlp_gemm_checked_requant", vp(ad), m, k, pb.handle, vp(c), n, vp(csum), 1, vp(fl), vp(er), f, vp(rsd),
               vp(csd), C.byref(_params(Q, prm, k)._c()), vp(out), n, stream_handle())
        torch.cuda.synchronize()
        ref_c = ct.copy()
        if fault:
            r, col, bit = fault
            ref_c[r, col:col + 1] = (ref_c[r, col:col + 1].view(np.uint32) ^ np.uint32(1 << bit)).view(np.int32)
        assert np.array_equal(c.cpu().numpy(), ref_c[:, :n]) and np.array_equal(csum.cpu().numpy(), ct[:, -1])
        assert np.array_equal(out.cpu().numpy(), O.requantize(ref_c, n, rs, cs, prm, k))
        assert int(er.item()) == (1 if fault else 0) and int(fl.sum().item()) == (1 if fault else 0)
