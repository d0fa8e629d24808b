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
