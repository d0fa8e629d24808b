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
