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
