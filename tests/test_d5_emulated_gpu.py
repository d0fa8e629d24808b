"""The D5 exchange (BASELINE configs[4]) on ONE GPU with G = 8 emulated ranks: every emulated rank's
tables go through the same grouped lookup launch (abftlp_eb_group_checked_scatter) and the same destination
address arithmetic the multi-rank classes use (paper_2103_00130_b200/sharded.py), the NCCL all-to-all is replaced
by the equivalent chunk copies, and the reassembled [B/G, T, d] outputs of every emulated rank are compared
bit-exactly with the CPU oracle for all 64 tables. The emulated ranks run one after another on one GPU (no rank
waits on another), which is the single-GPU stand-in for the 8-GPU exchange."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle_api as O

pytestmark = pytest.mark.gpu

G, T, R, D, B, POOL = 8, 64, 20_000, 128, 512, 80


def _zipf_bags(rng, n):
    ranks = np.arange(1, R + 1, dtype=np.float64)
    cdf = np.cumsum(ranks ** -1.05)
    cdf /= cdf[-1]
    return rng.permutation(R)[np.searchsorted(cdf, rng.random(n))].astype(np.int64)


@pytest.fixture(scope="module")
def d5_tables():
    """64 int8-rowwise tables (fp32 scale/bias), a few rows corrupted after the row sums, Zipf(1.05) bags of 80."""
    from paper_2103_00130_b200 import embedding as E
    tabs, host, bags = {}, {}, {}
    dev = torch.device("cuda")
    for t in range(T):
        rng = np.random.default_rng(1000 + t)
        rows = rng.integers(-128, 128, (R, D), dtype=np.int8)
        sc = rng.uniform(1e-3, 1e-2, R).astype(np.float32)
        bi = rng.uniform(-1, 1, R).astype(np.float32)
        tab = E.QuantEmbeddingTable(rows, sc, bi, elem="s8", dim=D)
        sums = O.row_sums(rows, "s8", D)
        idx = _zipf_bags(rng, B * POOL)
        off = np.arange(0, B * POOL + 1, POOL, dtype=np.int64)
        if t % 5 == 0:  # corrupt a looked-up row after the row sums: its bags must be flagged
            r, col, bit = int(idx[POOL * (t % B)]), int(rng.integers(0, D)), 6
            tab.flip_bit(r, col, bit)
            rows.view(np.uint8)[r, col] ^= np.uint8(1 << bit)
        tabs[t] = tab
        ref = O.eb(rows, sc, bi, off, idx, None, elem="s8", dim=D, row_sums_=sums)
        host[t] = (ref[0], np.asarray(ref[3], dtype=np.uint8))
        bags[t] = (torch.from_numpy(off).to(dev), torch.from_numpy(idx).to(dev), None)
    return tabs, host, bags


def _check_rank(g, out, flags, host):
    Bg = B // G
    assert tuple(out.shape) == (Bg, T, D) and tuple(flags.shape) == (Bg, T)
    o, f = out.cpu().numpy(), flags.cpu().numpy()
    for t in range(T):
        r_ref, e_ref = host[t]
        assert np.array_equal(o[:, t].view(np.uint32), r_ref[g * Bg:(g + 1) * Bg].view(np.uint32)), (g, t)
        assert np.array_equal(f[:, t], e_ref[g * Bg:(g + 1) * Bg]), (g, t)


def test_emulated_g8_nccl_exchange_matches_oracle(d5_tables):
    """NCCL path: emulated rank r pools its 8 tables into its exchange buffer [G, B/G, Tg, d+4] (vectors + flag
    quads) in one grouped launch; the all-to-all is recv_g[r] = send_r[g]; unpack_exchange reorders to table
    order. All 64 tables of all 8 emulated ranks equal the oracle bit for bit."""
    from paper_2103_00130_b200 import sharded as S
    tabs, host, bags = d5_tables
    Bg, Tg = B // G, T // G
    sends = []
    for r in range(G):
        mine = S.local_tables(T, G, r)
        x = torch.full((G, Bg, Tg, D + S.FLAG_QUAD), float("nan"), dtype=torch.float32, device="cuda")
        x.view(torch.uint8)[..., 4 * D:].zero_()
        be = S.GpuEbBackend()
        be.pool_into([tabs[t] for t in mine], [bags[t] for t in mine], x, D)
        be.raise_on_status()
        sends.append(x)
    total_flags = 0
    for g in range(G):
        recv = torch.stack([sends[r][g] for r in range(G)])  # all_to_all_single: chunk g of every sender
        out, flags = S.unpack_exchange(recv, T, D)
        _check_rank(g, out, flags, host)
        total_flags += int(flags.to(torch.int64).sum().item())
    assert total_flags == sum(int(h[1].sum()) for h in host.values()) > 0


def test_emulated_g8_peer_exchange_matches_oracle(d5_tables):
    """Peer path: emulated rank r's grouped launch writes bag b of table t straight into destination rank
    b // (B/G)'s FINAL buffers out[b % (B/G), t] / flags[...] (the PeerExchange address arithmetic over 8
    buffers standing in for the peers' symmetric memory). No reassembly step."""
    from paper_2103_00130_b200 import sharded as S
    tabs, host, bags = d5_tables
    Bg = B // G
    outs = [torch.full((Bg, T, D), float("nan"), dtype=torch.float32, device="cuda") for _ in range(G)]
    fls = [torch.full((Bg, T), 7, dtype=torch.uint8, device="cuda") for _ in range(G)]
    for r in range(G):
        mine = S.local_tables(T, G, r)
        be = S.GpuEbBackend()
        od = [[outs[g].data_ptr() + t * D * 4 for g in range(G)] for t in mine]
        fd = [[fls[g].data_ptr() + t for g in range(G)] for t in mine]
        be.pool([tabs[t] for t in mine], [bags[t] for t in mine], od, fd, ld_out=T * D, flag_ld=T, bags_per_dest=Bg)
        be.raise_on_status()
    for g in range(G):
        _check_rank(g, outs[g], fls[g], host)


def test_group_plan_rebinds_bags(d5_tables):
    """A persistent plan re-pointed at new bags (abftlp_eb_group_set_bags) pools exactly what a fresh plan pools."""
    from paper_2103_00130_b200 import embedding as E
    tabs, _, bags = d5_tables
    ts = [tabs[t] for t in range(4)]
    n = 100
    out = [torch.empty((n, 4, D), dtype=torch.float32, device="cuda") for _ in range(2)]
    fl = [torch.empty((n, 4), dtype=torch.uint8, device="cuda") for _ in range(2)]
    mk = lambda k: E.EbGroupPlan(ts, [[out[k].data_ptr() + t * D * 4] for t in range(4)],  # noqa: E731
                                 [[fl[k].data_ptr() + t] for t in range(4)], ld_out=4 * D, flag_ld=4, bags_per_dest=n)
    plan = mk(0)
    rng = np.random.default_rng(3)
    first = [(o[:n + 1].clone(), i.clone(), None) for o, i, _ in (bags[t] for t in range(4))]
    plan(first)
    for step in range(2):
        new = []
        for _ in range(4):
            lens = rng.integers(0, 50, n)
            off = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)).cuda()
            new.append((off, torch.from_numpy(rng.integers(0, R, int(lens.sum()))).cuda(), None))
        c0 = int(plan(new).item())
        c1 = int(mk(1)(new).item())
        torch.cuda.synchronize()
        assert torch.equal(out[0].view(torch.int32), out[1].view(torch.int32)) and torch.equal(fl[0], fl[1])
        assert c0 == c1


@pytest.mark.parametrize("d,force", [(40, False), (72, False), (128, True)])
def test_group_unfused_fallback(d, force, monkeypatch):
    """Tables the fused grouped kernel cannot take (dim % 32 != 0, rows not 16-byte aligned) run as one scatter
    launch per table behind the same group API: same outputs and flag count as the oracle (d = 128 forces the
    per-table form with ABFTLP_EB_GROUP_UNFUSED)."""
    from paper_2103_00130_b200 import embedding as E
    if force:
        monkeypatch.setenv("ABFTLP_EB_GROUP_UNFUSED", "1")
    rng = np.random.default_rng(d)
    n, Rr, nt = 64, 3000, 3
    tabs, bags, refs = [], [], []
    for t in range(nt):
        rows = rng.integers(-128, 128, (Rr, d)).astype(np.int8)
        sc = rng.uniform(1e-3, 1e-2, Rr).astype(np.float32)
        bi = rng.uniform(-1, 1, Rr).astype(np.float32)
        tab = E.QuantEmbeddingTable(rows, sc, bi, elem="s8", dim=d)
        tab.flip_bit(int(rng.integers(0, Rr)), 3, 7)
        rows2 = tab.rows.cpu().numpy().view(np.int8)
        lens = rng.integers(0, 60, n)
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        idx = rng.integers(0, Rr, int(off[-1])).astype(np.int64)
        tabs.append(tab)
        bags.append((off, idx, None))
        refs.append(O.eb(rows2, sc, bi, off, idx, None, elem="s8", dim=d, row_sums_=O.row_sums(rows, "s8", d)))
    out = torch.full((n, nt, d), float("nan"), dtype=torch.float32, device="cuda")
    fl = torch.full((n, nt), 7, dtype=torch.uint8, device="cuda")
    plan = E.EbGroupPlan(tabs, [[out.data_ptr() + t * d * 4] for t in range(nt)], [[fl.data_ptr() + t] for t in range(nt)],
                         ld_out=nt * d, flag_ld=nt, bags_per_dest=n)
    cnt = int(plan(bags).item())
    o, f = out.cpu().numpy(), fl.cpu().numpy()
    for t in range(nt):
        assert np.array_equal(o[:, t].view(np.uint32), refs[t][0].view(np.uint32))
        assert np.array_equal(f[:, t], refs[t][3])
    assert cnt == int(sum(np.asarray(r[3]).sum() for r in refs))


def _world2_worker(rank, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=2, device_id=torch.device("cuda", rank))
    try:
        from paper_2103_00130_b200 import embedding as E
        from paper_2103_00130_b200 import sharded as S
        Tn, Bn, d, Rr = 6, 32, 128, 4000
        tables, bags = {}, {}
        for t in S.local_tables(Tn, 2, rank):
            rng = np.random.default_rng(500 + t)
            rows = rng.integers(-128, 128, (Rr, d)).astype(np.int8)
            tab = E.QuantEmbeddingTable(rows, rng.uniform(1e-3, 1e-2, Rr).astype(np.float32),
                                        rng.uniform(-1, 1, Rr).astype(np.float32), elem="s8", dim=d)
            off = np.concatenate([[0], np.cumsum(rng.integers(0, 40, Bn))]).astype(np.int64)
            tables[t], bags[t] = tab, (off, rng.integers(0, Rr, int(off[-1])).astype(np.int64), None)
        res = {}
        for ex in ("nccl", "peer"):
            try:
                out, fl = S.ShardedEmbeddingBags(tables, Tn, Bn, d, exchange=ex)(bags)
                res[ex] = (out.cpu().numpy().copy(), fl.cpu().numpy().copy())
            except RuntimeError as e:
                res[ex] = str(e)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_world2_nccl_and_peer_match_oracle():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ps = [ctx.Process(target=_world2_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    Tn, Bn, d, Rr = 6, 32, 128, 4000
    for t in range(Tn):
        rng = np.random.default_rng(500 + t)
        rows = rng.integers(-128, 128, (Rr, d)).astype(np.int8)
        sc, bi = rng.uniform(1e-3, 1e-2, Rr).astype(np.float32), rng.uniform(-1, 1, Rr).astype(np.float32)
        off = np.concatenate([[0], np.cumsum(rng.integers(0, 40, Bn))]).astype(np.int64)
        idx = rng.integers(0, Rr, int(off[-1])).astype(np.int64)
        r_ref, _, _, e_ref = O.eb(rows, sc, bi, off, idx, None, elem="s8", dim=d)
        for rank in range(2):
            for ex, v in got[rank].items():
                if isinstance(v, str):
                    assert ex == "peer", v  # symmetric memory may be unavailable; NCCL must work
                    continue
                sl = slice(rank * Bn // 2, (rank + 1) * Bn // 2)
                assert np.array_equal(v[0][:, t].view(np.uint32), r_ref[sl].view(np.uint32)), (rank, ex, t)
                assert np.array_equal(v[1][:, t], np.asarray(e_ref, dtype=np.uint8)[sl]), (rank, ex, t)
