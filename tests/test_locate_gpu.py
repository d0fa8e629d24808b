"""Dual-encoded locate / correct on the GPU (abftlp_gemm_locate): the cell the reference's dual-encoded oracle
(P:tests/dual_check.hpp:23-73, restated in the oracle) locates is the cell the device finds, the repair restores the
clean product bit for bit, a hit checksum column is recomputed, and several errors are reported as not locatable."""
import numpy as np
import pytest
import torch

import oracle_api as O

pytestmark = pytest.mark.gpu


def _flip(v, bit):
    return int(np.array([np.uint32(np.int32(v).view(np.uint32)) ^ np.uint32(1 << bit)], np.uint32).view(np.int32)[0])


@pytest.mark.parametrize("m,n,k", [(5, 37, 70), (64, 512, 512), (300, 1000, 640), (8, 3200, 800), (1, 256, 256)])
def test_locate_and_correct_single_cell(m, n, k):
    from paper_2103_00130_b200 import gemm as G
    rng = np.random.default_rng(m + n + k)
    a = rng.integers(0, 256, (m, k)).astype(np.uint8)
    b = rng.integers(-128, 128, (k, n)).astype(np.int8)
    pb = G.PackedEncodedWeight(b)
    ct, _, _ = O.abft_gemm(a, b)
    clean = G.abft_gemm(a, pb)
    assert G.locate_and_correct(a, pb, clean).status == 0
    for _ in range(3):
        i, j, bit = int(rng.integers(m)), int(rng.integers(n)), int(rng.integers(32))
        bad = G.abft_gemm(a, pb, fault=(i, j, bit))
        assert bad.errCount == 1
        # the dual-encoded oracle (CPU) locates the same cell in the corrupted product
        dual = O.dual_product(a, b)
        dual[i, j] += _flip(int(ct[i, j]), bit) - int(ct[i, j])
        assert O.dual_check(dual) == (1, i, j)
        r = G.locate_and_correct(a, pb, bad)
        assert (r.status, r.row, r.col) == (1, i, j)
        assert r.delta == _flip(int(ct[i, j]), bit) - int(ct[i, j])
        assert np.array_equal(bad.cTemp.data.cpu().numpy(), ct)  # repaired bit for bit
        assert bad.errCount == 0 and not bad.rowFlags.any()


def test_locate_checksum_column_and_multiple_errors():
    from paper_2103_00130_b200 import gemm as G
    rng = np.random.default_rng(3)
    m, n, k = 40, 300, 256
    a = rng.integers(0, 256, (m, k)).astype(np.uint8)
    b = rng.integers(-128, 128, (k, n)).astype(np.int8)
    pb = G.PackedEncodedWeight(b)
    ct, _, _ = O.abft_gemm(a, b)
    bad = G.abft_gemm(a, pb, fault=(7, n, 12))  # the checksum column C'[7][n]
    r = G.locate_and_correct(a, pb, bad)
    assert (r.status, r.row, r.col) == (2, 7, n)
    assert np.array_equal(bad.cTemp.data.cpu().numpy(), ct) and bad.errCount == 0
    bad = G.abft_gemm(a, pb, fault=(3, 10, 5))
    bad.cTemp.data[20, 100] += 1  # a second error in another row and column
    bad.errCount = G.verify_checksums(bad.cTemp, bad.rowFlags)
    r = G.locate_and_correct(a, pb, bad)
    assert r.status == 3 and r.rows_flagged == 2 and r.cols_mismatched == 2
