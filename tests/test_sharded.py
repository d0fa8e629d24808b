"""Multi-process (gloo, world size 2, CPU) tests of the sharding host logic (paper_2103_00130_b200/sharded.py,
SURVEY 8e): N-column GEMM shards with OR-reduced verdicts, table-wise EmbeddingBag shards with the
all-to-all to batch-sharded layout. The per-shard compute is the CPU oracle here (test infrastructure);
on GPUs the same classes run the CUDA library (tests/test_sharded_gpu.py covers the scatter kernel)."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))

from paper_2103_00130_b200 import sharded as S  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# ---------------------------------------------------------------- oracle-backed shard compute (CPU)
class OracleGemmBackend:
    def encode(self, b_shard):
        return np.ascontiguousarray(b_shard.numpy() if torch.is_tensor(b_shard) else b_shard, dtype=np.int8)

    def run(self, a, w, fault=None):
        import oracle_api as O
        ct, fl, _ = O.abft_gemm(a, w)
        if fault is not None:  # post-hoc flip of C'(row, col) and the reference's row check
            r, c, bit = fault
            ct = ct.copy()
            ct[r, c:c + 1] = (ct[r, c:c + 1].view(np.uint32) ^ np.uint32(1 << bit)).view(np.int32)
            _, fl = O.verify(ct)
        return torch.from_numpy(ct), torch.from_numpy(np.asarray(fl, dtype=np.uint8))


class OracleEbBackend:
    """Writes the exchange buffer exactly as the GPU grouped scatter launch does: x[g, b, slot, :d] = pooled vector
    of sample g*Bg + b, byte 4*d of x[g, b, slot] = its verdict (the flag quad)."""

    def pool_into(self, tables, bags, x, d, stream=None):
        import oracle_api as O
        G, Bg = x.shape[0], x.shape[1]
        xb = x.view(torch.uint8)
        for slot, (table, (offsets, indices, weights)) in enumerate(zip(tables, bags)):
            rows, sc, bi, sums = table
            r, _, _, e = O.eb(rows, sc, bi, offsets, indices, weights, row_sums_=sums)
            x[:, :, slot, :d] = torch.from_numpy(r).view(G, Bg, d)
            xb[:, :, slot, 4 * d] = torch.from_numpy(np.asarray(e, dtype=np.uint8)).view(G, Bg)

    def raise_on_status(self):
        pass


# ---------------------------------------------------------------- workers
M, K, N = 33, 70, 37


def _gemm_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle_api as O
        a, b = O.gemm_inputs(20260823, 0, M, N, K)
        n0, n1 = S.column_shard(N, world, rank)
        g = S.ShardedAbftGemm(b[:, n0:n1], N, backend=OracleGemmBackend())
        clean = g(a)
        # rank 1 flips bit 9 of its local C'(5, 2); every rank must see row 5 flagged
        bad = g(a, fault=(5, 2, 9) if rank == 1 else None)
        shards = [None] * world
        dist.all_gather_object(shards, (n0, n1, clean.cTemp.numpy()))
        q.put((rank, clean.errCount, clean.rowFlags.numpy(), bad.errCount, bad.rowFlags.numpy(), shards))
    finally:
        dist.destroy_process_group()


T, B, D, R = 5, 6, 16, 50


def _eb_inputs(t):
    rng = np.random.default_rng(100 + t)
    rows = rng.integers(-128, 128, (R, D)).astype(np.int8)
    sc = rng.uniform(1e-3, 1e-2, R).astype(np.float32)
    bi = rng.uniform(-1, 1, R).astype(np.float32)
    lens = rng.integers(0, 12, B)
    lens[t % B] = 0  # an empty bag somewhere
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = rng.integers(0, R, int(off[-1])).astype(np.int64)
    w = rng.uniform(0, 1, int(off[-1])).astype(np.float32) if t % 2 else None
    return rows, sc, bi, off, idx, w


def _eb_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tables, bags = {}, {}
        for t in S.local_tables(T, world, rank):
            rows, sc, bi, off, idx, w = _eb_inputs(t)
            sums = rows.astype(np.int32).sum(axis=1).astype(np.int32)  # row sums of the pristine table
            if t == 3:  # fault after row sums: flip the sign bit of an element pooled by sample 1's bag
                rows = rows.copy()
                i = int(idx[off[1]]) if off[2] > off[1] else int(idx[0])
                rows[i, 4] ^= np.int8(-128)
            tables[t] = (rows, sc, bi, sums)
            bags[t] = (off, idx, w)
        eb = S.ShardedEmbeddingBags(tables, T, B, D, backend=OracleEbBackend(), device="cpu")
        out, flags = eb(bags)
        q.put((rank, out.numpy(), flags.numpy()))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r[0])


# ---------------------------------------------------------------- tests
def test_column_shard_partition():
    for n in (1, 2, 7, 37, 4096):
        for world in (1, 2, 3, 8):
            if n < world:
                continue
            ranges = [S.column_shard(n, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
            widths = [b - a for a, b in ranges]
            assert max(widths) - min(widths) <= 1


def test_table_ownership():
    assert [S.table_owner(t, 3) for t in range(7)] == [0, 1, 2, 0, 1, 2, 0]
    assert S.local_tables(7, 3, 1) == [1, 4]
    assert sorted(sum((S.local_tables(64, 8, r) for r in range(8)), [])) == list(range(64))


def test_sharded_gemm_gloo_world2():
    import oracle_api as O
    res = _spawn(_gemm_worker)
    a, b = O.gemm_inputs(20260823, 0, M, N, K)
    full, fl_full, _ = O.abft_gemm(a, b)
    for rank, clean_err, clean_fl, bad_err, bad_fl, shards in res:
        assert clean_err == 0 and not clean_fl.any()
        # C shards reassemble the single-GPU product bit for bit; each shard's own checksum column is the
        # reference's abft_gemm on that shard (not comparable to the global column n)
        cat = np.concatenate([s[2][:, :-1] for s in sorted(shards, key=lambda s: s[0])], axis=1)
        assert np.array_equal(cat, full[:, :N])
        for n0, n1, ct in shards:
            ref_ct, _, _ = O.abft_gemm(a, np.ascontiguousarray(b[:, n0:n1]))
            assert np.array_equal(ct, ref_ct)
        # the verdict for a fault in rank 1's shard equals the reference's global check
        n0_1 = S.column_shard(N, 2, 1)[0]
        g = full.copy()
        c = n0_1 + 2
        g[5, c:c + 1] = (g[5, c:c + 1].view(np.uint32) ^ np.uint32(1 << 9)).view(np.int32)
        e, fl = O.verify(g)
        assert bad_err == e == 1
        assert np.array_equal(bad_fl, np.asarray(fl, dtype=np.uint8))


def test_sharded_eb_gloo_world2():
    import oracle_api as O
    res = _spawn(_eb_worker)
    Bg = B // 2
    for rank, out, flags in res:
        assert out.shape == (Bg, T, D) and flags.shape == (Bg, T)
        for t in range(T):
            rows, sc, bi, off, idx, w = _eb_inputs(t)
            sums = rows.astype(np.int32).sum(axis=1).astype(np.int32)
            if t == 3:
                rows = rows.copy()
                i = int(idx[off[1]]) if off[2] > off[1] else int(idx[0])
                rows[i, 4] ^= np.int8(-128)
            r, _, _, e = O.eb(rows, sc, bi, off, idx, w, row_sums_=sums)
            sl = S.sample_slice(B, 2, rank)
            assert np.array_equal(out[:, t].view(np.uint32), r[sl].view(np.uint32)), (rank, t)
            assert np.array_equal(flags[:, t], np.asarray(e, dtype=np.uint8)[sl]), (rank, t)
    flagged = np.concatenate([r[2] for r in res], axis=0)
    assert flagged[:, 3].any() and not np.delete(flagged, 3, axis=1).any()


def test_sharded_eb_rejects_wrong_ownership():
    with pytest.raises(ValueError):
        S.ShardedEmbeddingBags({1: None}, 4, 8, 16, backend=OracleEbBackend(), device="cpu")
