"""One-launch batched checked GEMM (BASELINE config 0: 100 seeded trials of m=64, k=512, n=512, each with
its own A and B under the reference's draw protocol) vs the oracle, problem by problem, bit-exact."""
import numpy as np
import pytest

import oracle_api as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nb,m,n,k", [(100, 64, 512, 512), (7, 130, 300, 200), (3, 256, 1024, 1024)])
def test_batched_matches_per_problem_oracle(nb, m, n, k):
    from paper_2103_00130_b200 import gemm as G
    a = np.stack([O.gemm_inputs(20260823, t, m, n, k)[0] for t in range(nb)])
    b = np.stack([O.gemm_inputs(20260823, t, m, n, k)[1] for t in range(nb)])
    pb = G.PackedEncodedWeightBatch(b)
    ct, err, flags = G.abft_gemm_batched(a, pb)
    ct, err, flags = ct.cpu().numpy(), err.cpu().numpy(), flags.cpu().numpy()
    for t in range(nb):
        ref, fl, e = O.abft_gemm(a[t], b[t])
        assert np.array_equal(ct[t], ref), t
        assert err[t] == e == 0 and not flags[t].any()
    # one fault in one problem (checksum column and a data column): only that problem is flagged
    for col in (n, n // 2):
        p_ = nb // 2
        ct2, err2, flags2 = G.abft_gemm_batched(a, pb, fault=(p_, m - 1, col, 5))
        err2 = err2.cpu().numpy()
        assert err2[p_] == 1 and err2.sum() == 1 and int(flags2[p_, m - 1].item()) == 1


def test_g1_trials_protocol_sum():
    """SURVEY 8c known answer: over the 100 G1 trials the clean C' sum is -81,406,600,320 and the odd
    trials' single C' bit flips (stream t*4+1 draws) are all detected, with no false positives."""
    from paper_2103_00130_b200 import gemm as G
    from paper_2103_00130_b200.rng import SplitMix64
    nb, m, n, k = 100, 64, 512, 512
    a = np.stack([O.gemm_inputs(20260823, t, m, n, k)[0] for t in range(nb)])
    b = np.stack([O.gemm_inputs(20260823, t, m, n, k)[1] for t in range(nb)])
    pb = G.PackedEncodedWeightBatch(b)
    ct, err, _ = G.abft_gemm_batched(a, pb)
    assert int(ct.cpu().numpy().astype(np.int64).sum()) == -81_406_600_320
    assert int(err.sum().item()) == 0
    detected = 0
    for t in range(1, nb, 2):
        r = SplitMix64(20260823, t * 4 + 1)
        i, j, bit = r.next_below(m), r.next_below(n + 1), r.next_below(32)
        _, e, _ = G.abft_gemm_batched(a, pb, fault=(t, i, j, bit))
        detected += int(e[t].item())
    assert detected == 50


@pytest.mark.parametrize("nb,m,n,k", [(12, 256, 1024, 1024), (5, 200, 520, 384), (32, 33, 300, 208), (8, 1, 256, 256), (24, 1, 800, 800),
                                      (40, 64, 1024, 256)])
def test_grouped_shared_weight_with_fault_list(nb, m, n, k):
    """Grouped job form (BASELINE config 1's 1000 runs against one encoded B): every problem shares ONE
    PackedEncodedWeight, several C' faults (data and checksum columns, different problems, two in one
    problem) ride in one launch's fault list; per problem, C' equals the oracle with the same bits flipped
    post hoc and the counts equal the reference's verify on it."""
    from paper_2103_00130_b200 import gemm as G
    a = np.stack([O.gemm_inputs(20260823, t, m, n, k)[0] for t in range(nb)])
    b = O.gemm_inputs(20260823, 0, m, n, k)[1]
    pb = G.PackedEncodedWeight(b)
    # (requests of fewer than 256 rows against one weight run as the row blocks of one tall GEMM: same results)
    faults = [(1, min(3, m - 1), n, 7), (4, m - 1, n // 3, 31), (4, 0, 0, 0), (nb - 1, m // 2, n - 1, 12)]
    ct, err, flags = G.abft_gemm_batched(a, pb, faults=faults)
    ct, err, flags = ct.cpu().numpy(), err.cpu().numpy(), flags.cpu().numpy()
    for t in range(nb):
        ref, _, _ = O.abft_gemm(a[t], b)
        ref = ref.copy()
        for (p_, i, j, bit) in faults:
            if p_ == t:
                ref[i, j] = np.int32(np.uint32(ref[i, j].view(np.uint32) ^ np.uint32(1 << bit)).view(np.int32))
        assert np.array_equal(ct[t], ref), t
        e_ref, fl_ref = O.verify(ref)  # the reference's verify_checksums on the post-hoc faulted C'
        assert err[t] == e_ref == len({i for (p_, i, _, _) in faults if p_ == t}), t
        assert np.array_equal(flags[t], fl_ref), t


def test_grouped_fault_list_limits():
    from paper_2103_00130_b200 import _lib
    from paper_2103_00130_b200 import gemm as G
    a = np.zeros((2, 8, 128), np.uint8)
    pb = G.PackedEncodedWeight(np.ones((128, 64), np.int8))
    with pytest.raises(_lib.InvalidArgument):
        G.abft_gemm_batched(a, pb, faults=[(0, 0, 0, 0)] * 9)
    with pytest.raises(_lib.InvalidArgument):  # out_of_range -> ABFTLP_ERR_INVALID_ARGUMENT
        G.abft_gemm_batched(a, pb, faults=[(2, 0, 0, 0)])


@pytest.mark.parametrize("nb,m,n,k", [(21, 256, 512, 384), (3, 40, 130, 200), (1, 7, 64, 128)])
def test_host_batched_job_matches_oracle(nb, m, n, k):
    """abftlp_gemm_checked_host_batched (pinned host buffers, pipelined copy-in / grouped launch / copy-out):
    every run's C', checksum column, flags and count equal the oracle's abft_gemm on that run."""
    import ctypes as C
    import torch
    from paper_2103_00130_b200 import _lib
    from paper_2103_00130_b200 import gemm as G
    a = np.stack([O.gemm_inputs(20260823, t, m, n, k)[0] for t in range(nb)])
    b = O.gemm_inputs(20260823, 0, m, n, k)[1]
    pb = G.PackedEncodedWeight(b)
    ah = torch.from_numpy(a).pin_memory()
    ch = torch.zeros((nb, m, n), dtype=torch.int32).pin_memory()
    csh = torch.zeros((nb, m), dtype=torch.int32).pin_memory()
    flh = torch.ones((nb, m), dtype=torch.uint8).pin_memory()
    eh = torch.full((nb,), 7, dtype=torch.int32).pin_memory()
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    _lib.call("abftlp_gemm_checked_host_batched", vp(ah), nb, m, k, m * k, pb.handle, vp(ch), n, m * n, vp(csh), m,
              vp(flh), m, vp(eh), None)
    for t in range(nb):
        ref, fl, e = O.abft_gemm(a[t], b)
        assert np.array_equal(ch[t].numpy(), ref[:, :n]), t
        assert np.array_equal(csh[t].numpy(), ref[:, n]), t
        assert not flh[t].numpy().any() and int(eh[t]) == e == 0, t


def test_batched_weight_flip_bit_only_hits_its_problem():
    """abftlp_gemm_weight_flip_bit_batched: inject_weight_B into one problem of a batched weight after encoding
    (clean checksums): that problem's C' equals the oracle product with the corrupted B and the clean checksum
    column, and only its rows can be flagged; the other problems are untouched."""
    import ctypes as C
    from paper_2103_00130_b200 import _lib
    from paper_2103_00130_b200 import gemm as G
    nb, m, n, k = 3, 256, 512, 384
    a = np.stack([O.gemm_inputs(20260823, t, m, n, k)[0] for t in range(nb)])
    b = np.stack([O.gemm_inputs(20260823, t, m, n, k)[1] for t in range(nb)])
    pb = G.PackedEncodedWeightBatch(b)
    p_, i, j, bit = 1, 100, 200, 6
    _lib.call("abftlp_gemm_weight_flip_bit_batched", pb.handle, p_, i, j, bit, None)
    ct, err, flags = G.abft_gemm_batched(a, pb)
    ct, err = ct.cpu().numpy(), err.cpu().numpy()
    for t in range(nb):
        bt = b[t].copy()
        if t == p_:
            bt.view(np.uint8)[i, j] ^= np.uint8(1 << bit)
        ref, fl, e = O.abft_gemm(a[t], bt, cs=O.row_checksums(b[t]))
        assert np.array_equal(ct[t], ref), t
        assert err[t] == e, t
    assert err[p_] >= 1 and err[0] == err[2] == 0
    with pytest.raises(_lib.InvalidArgument):
        _lib.call("abftlp_gemm_weight_flip_bit_batched", pb.handle, nb, 0, 0, 0, None)


@pytest.mark.parametrize("ew", ["4", "8"])
@pytest.mark.parametrize("nb,m,n,k", [(6, 64, 512, 512), (3, 256, 1024, 1024), (4, 130, 300, 1000)])
def test_epilogue_warp_counts_bit_exact(nb, m, n, k, ew, monkeypatch):
    """The checked epilogue with one group of 4 warps or two groups of 4 splitting each tile's columns (one row
    arrival per group): identical C', checksum column, flags and counts, with C' faults on both sides."""
    from paper_2103_00130_b200 import gemm as G
    monkeypatch.setenv("ABFTLP_GEMM_EW", ew)
    a = np.stack([O.gemm_inputs(20260823, t, m, n, k)[0] for t in range(nb)])
    b = np.stack([O.gemm_inputs(20260823, t, m, n, k)[1] for t in range(nb)])
    pb = G.PackedEncodedWeightBatch(b)
    faults = [(0, m - 1, n, 3), (nb - 1, 1, n // 2, 30)]
    for fl_ in (None, faults):
        ct, err, flags = G.abft_gemm_batched(a, pb, faults=fl_) if fl_ else G.abft_gemm_batched(a, pb)
        ct, err = ct.cpu().numpy(), err.cpu().numpy()
        for t in range(nb):
            ref, _, _ = O.abft_gemm(a[t], b[t])
            ref = ref.copy()
            for (p_, i, j, bit) in (fl_ or []):
                if p_ == t:
                    ref[i, j] = np.int32(np.uint32(ref[i, j].view(np.uint32) ^ np.uint32(1 << bit)).view(np.int32))
            e_ref, _ = O.verify(ref)
            assert np.array_equal(ct[t], ref), t
            assert err[t] == e_ref, t
