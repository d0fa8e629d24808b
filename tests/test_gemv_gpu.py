"""Small-m checked GEMM (GEMV class) vs the oracle and vs the tensor-core path: the 28
DLRM shapes of P:data/shapes.txt (m in {1, 8, 32, 64}; m <= 16 take the GEMV path) plus ragged shapes and
the fault hook on both sides of the checksum column."""
import numpy as np
import pytest

import oracle_api as O

pytestmark = pytest.mark.gpu

# P:data/shapes.txt (m x n x k): 7 (n, k) pairs for each m
NK = [(256, 256), (800, 800), (1024, 1024), (3200, 3200), (800, 3200), (3200, 800), (1024, 256)]
SHAPES = [(m, n, k) for m in (1, 8, 32, 64) for n, k in NK]


@pytest.mark.parametrize("m,n,k", SHAPES)
def test_dlrm_shapes_bit_exact(m, n, k):
    from paper_2103_00130_b200 import gemm as G
    a, b = O.gemm_inputs(20260823, m + n + k, m, n, k)
    res = G.abft_gemm(a, G.PackedEncodedWeight(b))
    ct, fl, err = O.abft_gemm(a, b)
    assert np.array_equal(res.cTemp.data.cpu().numpy(), ct) and res.errCount == err == 0


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (2, 33, 17), (3, 100, 130), (13, 257, 1000), (16, 4095, 4096),
                                   (7, 64, 4097)])
def test_ragged_and_faults_match_tensor_core_path(m, n, k, monkeypatch):
    from paper_2103_00130_b200 import gemm as G
    a, b = O.gemm_inputs(7, m * 1000 + n, m, n, k)
    pb = G.PackedEncodedWeight(b)
    res = G.abft_gemm(a, pb)
    ct, fl, err = O.abft_gemm(a, b)
    assert np.array_equal(res.cTemp.data.cpu().numpy(), ct) and res.errCount == err == 0
    for col in (n - 1, n):
        bad = G.abft_gemm(a, pb, fault=(m - 1, col, 3))
        assert bad.errCount == 1 and int(bad.rowFlags[m - 1].item()) == 1
        monkeypatch.setenv("ABFTLP_GEMV_MAX_ROWS", "0")  # same call on the tensor-core path
        tc = G.abft_gemm(a, pb, fault=(m - 1, col, 3))
        monkeypatch.delenv("ABFTLP_GEMV_MAX_ROWS")
        assert np.array_equal(bad.cTemp.data.cpu().numpy(), tc.cTemp.data.cpu().numpy())
    plain = G.plain_gemm(a, b)
    assert np.array_equal(plain.data.cpu().numpy(), ct[:, :n])


@pytest.mark.parametrize("m,n,k", [(1, 256, 256), (3, 1000, 700), (8, 800, 800), (16, 256, 1024), (5, 64, 130),
                                   (8, 3200, 256)])
def test_single_cluster_gemv_matches_multiblock_and_oracle(m, n, k, monkeypatch):
    """The one-cluster GEMV (no global atomics: residues and checksum shares meet in the leader's shared memory)
    and the multi-block GEMV give the oracle's C', checksum column and verdicts, with C' faults on both sides of the
    checksum column."""
    from paper_2103_00130_b200 import gemm as G
    a, b = O.gemm_inputs(11, m * 31 + n + k, m, n, k)
    pb = G.PackedEncodedWeight(b)
    ct, fl, err = O.abft_gemm(a, b)
    for cl in ("1", "0"):
        monkeypatch.setenv("ABFTLP_GEMV_CLUSTER", cl)
        monkeypatch.setenv("ABFTLP_GEMV_CLUSTER_BYTES", str(8 << 20))
        for _ in range(2):
            res = G.abft_gemm(a, pb)
            assert np.array_equal(res.cTemp.data.cpu().numpy(), ct) and res.errCount == err == 0
            assert np.array_equal(res.rowFlags.cpu().numpy(), fl)
        for row, col, bit in ((m - 1, n, 30), (0, n // 2, 3), (m // 2, 0, 31)):
            bad = G.abft_gemm(a, pb, fault=(row, col, bit))
            flags = bad.rowFlags.cpu().numpy()
            assert bad.errCount == 1 and flags[row] == 1 and int(flags.sum()) == 1
            c2 = ct.copy()
            c2[row, col:col + 1] = (c2[row, col:col + 1].view(np.uint32) ^ np.uint32(1 << bit)).view(np.int32)
            assert np.array_equal(bad.cTemp.data.cpu().numpy(), c2)
