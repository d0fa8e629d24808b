"""Deterministic input generators shared by oracle/make_golden.py and the tests (fixtures are
regenerated from these; TEST INFRASTRUCTURE)."""
import numpy as np


def requant_inputs(seed):
    """Deterministic requantization case: C' (m x (n+1), junk checksum column), row/col sums, params."""
    rng = np.random.default_rng(seed)
    m, n, k = int(rng.integers(1, 13)), int(rng.integers(1, 13)), int(rng.integers(1, 4097))
    c = rng.integers(-2 ** 31, 2 ** 31, (m, n + 1), dtype=np.int64).astype(np.int32)
    if seed % 3 == 0:  # realistic magnitudes as well as full-range words
        c = rng.integers(-3_000_000, 3_000_000, (m, n + 1)).astype(np.int32)
    rs = rng.integers(0, 255 * k + 1, m).astype(np.int32)
    cs = rng.integers(-128 * k, 127 * k + 1, n).astype(np.int32)
    prm = np.array([rng.uniform(1e-4, 0.05), rng.uniform(-0.5, 0.5), rng.uniform(1e-4, 0.05),
                    rng.uniform(-0.5, 0.5), rng.uniform(0.01, 50.0), rng.uniform(-100.0, 100.0)])
    return m, n, k, c, rs, cs, prm
