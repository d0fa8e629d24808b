"""GPU side of the sharding path: the scatter-mode lookup kernel (abftlp_eb_checked_scatter)
writes every bag into its destination slot bit-identically to the plain kernel, and the sharded classes
run on the CUDA library (world size 1 on the single test GPU; the multi-rank host logic is covered by
tests/test_sharded.py with gloo)."""
import numpy as np
import pytest
import torch

import oracle_api as O

pytestmark = pytest.mark.gpu


def _table(E, elem, R, d, seed, f16=False):
    rng = np.random.default_rng(seed)
    rb = d // 2 if elem == "u4" else d
    lo, hi = (-128, 128) if elem == "s8" else (0, 256)
    rows = rng.integers(lo, hi, (R, rb)).astype(np.int8 if elem == "s8" else np.uint8)
    sdt = np.float16 if f16 else np.float32
    sc = rng.uniform(1e-3, 1e-2, R).astype(sdt)
    bi = rng.uniform(-1, 1, R).astype(sdt)
    return rows, sc, bi, E.QuantEmbeddingTable(rows, sc, bi, elem=elem, dim=d)


@pytest.mark.parametrize("elem,d,f16,weighted", [("u8", 128, False, False), ("u4", 64, True, True),
                                                 ("s8", 40, False, True), ("s8", 256, False, False)])
def test_scatter_kernel_matches_plain(elem, d, f16, weighted):
    from paper_2103_00130_b200 import embedding as E
    rows, sc, bi, t = _table(E, elem, 3000, d, 7, f16)
    rng = np.random.default_rng(11)
    G, Bg, Tg, slot = 3, 5, 2, 1
    B = G * Bg
    lens = rng.integers(0, 90, B)
    lens[4] = 0
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = rng.integers(0, 3000, off[-1]).astype(np.int64)
    w = rng.uniform(0, 1, off[-1]).astype(np.float32) if weighted else None
    out, flags, _, _, cnt = E.eb_csr(t, off, idx, w)
    send = torch.full((G, Bg, Tg, d), float("nan"), dtype=torch.float32, device="cuda")
    send_f = torch.full((G, Bg, Tg), 7, dtype=torch.uint8, device="cuda")
    n = E.eb_csr_scatter(t, off, idx, w, [send[g, 0, slot] for g in range(G)], [send_f[g, 0, slot:] for g in range(G)],
                         ld_out=Tg * d, flag_ld=Tg, bags_per_dest=Bg)
    got = send[:, :, slot].reshape(B, d)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), out.cpu().numpy().view(np.uint32))
    assert np.array_equal(send_f[:, :, slot].reshape(B).cpu().numpy(), flags.cpu().numpy())
    assert int(n.item()) == int(cnt.item())
    # the other slot is untouched
    assert torch.isnan(send[:, :, 0]).all() and (send_f[:, :, 0] == 7).all()
    r_ref, _, _, e_ref = O.eb(rows, sc, bi, off, idx, w, elem=elem, dim=d)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), r_ref.view(np.uint32))


def test_sharded_classes_world1():
    from paper_2103_00130_b200 import embedding as E
    from paper_2103_00130_b200 import sharded as S
    a, b = O.gemm_inputs(20260823, 0, 96, 300, 256)
    g = S.ShardedAbftGemm(torch.from_numpy(b).cuda(), 300)
    r = g(a)
    ct, fl, err = O.abft_gemm(a, b)
    assert np.array_equal(r.cTemp.cpu().numpy(), ct) and r.errCount == err == 0
    r2 = g(a, fault=(7, 300, 31))  # checksum column, sign bit
    assert r2.errCount == 1 and int(r2.rowFlags[7].item()) == 1
    T, B, d = 3, 8, 64
    tables, bags, refs = {}, {}, {}
    for t in range(T):
        rows, sc, bi, tab = _table(E, "u8", 1000, d, 20 + t)
        rng = np.random.default_rng(40 + t)
        off = np.concatenate([[0], np.cumsum(rng.integers(0, 30, B))]).astype(np.int64)
        idx = rng.integers(0, 1000, off[-1]).astype(np.int64)
        tables[t], bags[t] = tab, (off, idx, None)
        refs[t] = O.eb(rows, sc, bi, off, idx, None, elem="u8", dim=d)
    out, flags = S.ShardedEmbeddingBags(tables, T, B, d)(bags)
    for t in range(T):
        assert np.array_equal(out[:, t].cpu().numpy().view(np.uint32), refs[t][0].view(np.uint32))
        assert np.array_equal(flags[:, t].cpu().numpy(), refs[t][3])


@pytest.mark.parametrize("elem,scale,d,weighted", [("s8", "f32", 128, False), ("u4", "f16", 64, True)])
def test_grouped_tables_equal_per_table_scatter(elem, scale, d, weighted):
    """abftlp_eb_group_checked_scatter (all of a GPU's tables in ONE launch, D5) writes exactly what one
    abftlp_eb_checked_scatter per table writes: pooled vectors, flags and the total flag count."""
    import ctypes as C

    import numpy as np
    import torch

    from paper_2103_00130_b200 import _lib as L
    from paper_2103_00130_b200 import embedding as E
    dev = torch.device("cuda")
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    rng = np.random.default_rng(d)
    T, R, B, G = 5, 4000, 1200, 4
    Bg = B // G
    tabs, keep, bags = [], [], []
    for t in range(T):
        rb = d // 2 if elem == "u4" else d
        rows = rng.integers(0 if elem != "s8" else -128, 256 if elem != "s8" else 128, (R, rb)).astype(
            np.int8 if elem == "s8" else np.uint8)
        sdt = np.float16 if scale == "f16" else np.float32
        tab = E.QuantEmbeddingTable(rows, rng.uniform(1e-3, 1e-2, R).astype(sdt), rng.uniform(-1, 1, R).astype(sdt),
                                    elem=elem, dim=d)
        for r in rng.choice(R, 10, replace=False):  # some corrupted rows -> some flagged bags
            tab.flip_bit(int(r), int(rng.integers(0, d)), 1)
        lens = rng.integers(0, 60, B)
        off = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)).to(dev)
        ix = torch.from_numpy(rng.integers(0, R, int(lens.sum())).astype(np.int64)).to(dev)
        w = torch.from_numpy(rng.uniform(0, 1, int(lens.sum())).astype(np.float32)).to(dev) if weighted else None
        tabs.append(tab)
        bags.append((off, ix, w))
    outs = [torch.full((G, Bg, T, d), float("nan"), dtype=torch.float32, device=dev) for _ in range(2)]
    flgs = [torch.full((G, Bg, T), 7, dtype=torch.uint8, device=dev) for _ in range(2)]
    cnt = [torch.zeros(1, dtype=torch.int32, device=dev) for _ in range(3)]
    dests = []
    for k in range(2):
        per = []
        for t in range(T):
            o = torch.tensor([outs[k][g, 0, t].data_ptr() for g in range(G)], dtype=torch.int64, device=dev)
            f = torch.tensor([flgs[k][g, 0, t:].data_ptr() for g in range(G)], dtype=torch.int64, device=dev)
            per.append((o, f))
        dests.append(per)
    total = 0
    for t in range(T):  # reference: one scatter launch per table
        off, ix, w = bags[t]
        o, f = dests[0][t]
        L.call("abftlp_eb_checked_scatter", tabs[t].handle, vp(off), vp(ix), B, vp(w) if w is not None else None,
               vp(o), T * d, vp(f), T, Bg, vp(cnt[0]), None, None)
        total += int(cnt[0].item())
    P = C.c_void_p
    th = (P * T)(*[tabs[t].handle for t in range(T)])
    offs = (P * T)(*[P(bags[t][0].data_ptr()) for t in range(T)])
    ixs = (P * T)(*[P(bags[t][1].data_ptr()) for t in range(T)])
    ws = (P * T)(*[P(bags[t][2].data_ptr()) for t in range(T)]) if weighted else None
    ods = (P * T)(*[P(dests[1][t][0].data_ptr()) for t in range(T)])
    fds = (P * T)(*[P(dests[1][t][1].data_ptr()) for t in range(T)])
    grp = C.c_void_p()
    L.call("abftlp_eb_group_create", th, T, offs, ixs, ws, ods, fds, C.byref(grp))
    for _ in range(2):  # self-resetting workspace
        L.call("abftlp_eb_group_checked_scatter", grp, B, T * d, T, Bg, vp(cnt[1]), None, None)
        torch.cuda.synchronize()
        assert torch.equal(outs[1].view(torch.int32), outs[0].view(torch.int32))
        assert torch.equal(flgs[1], flgs[0])
        assert int(cnt[1].item()) == total > 0
    L.lib.abftlp_eb_group_free(grp)


def test_d5_share_full_size_grouped_vs_oracle():
    """BASELINE configs[4] at full size for one GPU's share (8 tables x 1M x 128 int8 rows, fp32 scale/bias, batch
    8192, pooling 80, Zipf(1.05) indices): the grouped one-launch lookup writes, for every table, the oracle's
    pooled vectors and verdicts (bit-exact), with a few rows corrupted after the row sums."""
    import ctypes as C

    import numpy as np
    import torch

    from paper_2103_00130_b200 import _lib as L
    from paper_2103_00130_b200 import embedding as E
    dev = torch.device("cuda")
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    T, R, d, B, pool, G = 8, 1_000_000, 128, 8192, 80, 8
    Bg = B // G
    rng = np.random.default_rng(5)
    ranks = np.arange(1, R + 1, dtype=np.float64)
    cdf = np.cumsum(ranks ** -1.05)
    cdf /= cdf[-1]
    tabs, host, bags = [], [], []
    for t in range(T):
        rows = rng.integers(-128, 128, (R, d), dtype=np.int8)
        sc = rng.uniform(1e-3, 1e-2, R).astype(np.float32)
        bi = rng.uniform(-1, 1, R).astype(np.float32)
        tab = E.QuantEmbeddingTable(rows, sc, bi, elem="s8", dim=d)
        sums = O.row_sums(rows, "s8", d)
        for r in rng.choice(R, 4, replace=False):  # corrupt after the row sums
            col, bit = int(rng.integers(0, d)), int(rng.integers(0, 8))
            tab.flip_bit(int(r), col, bit)
            rows.view(np.uint8)[r, col] ^= np.uint8(1 << bit)
        idx = rng.permutation(R)[np.searchsorted(cdf, rng.random(B * pool))].astype(np.int64)
        off = np.arange(0, B * pool + 1, pool, dtype=np.int64)
        tabs.append(tab)
        host.append((rows, sc, bi, sums, off, idx))
        bags.append((torch.from_numpy(off).to(dev), torch.from_numpy(idx).to(dev), None))
    send = torch.full((G, Bg, T, d), float("nan"), dtype=torch.float32, device=dev)
    send_f = torch.full((G, Bg, T), 7, dtype=torch.uint8, device=dev)
    outs = [[send[g, 0, t] for g in range(G)] for t in range(T)]
    flags = [[send_f[g, 0, t:] for g in range(G)] for t in range(T)]
    cnt = E.eb_group_scatter(tabs, bags, outs, flags, ld_out=T * d, flag_ld=T, bags_per_dest=Bg)
    out = send.permute(2, 0, 1, 3).reshape(T, B, d).cpu().numpy()
    fl = send_f.permute(2, 0, 1).reshape(T, B).cpu().numpy()
    total = 0
    for t in (0, 3, 7):  # three tables against the oracle (CPU time), all tables' counts via the flags
        rows, sc, bi, sums, off, idx = host[t]
        r_ref, _, _, e_ref = O.eb(rows, sc, bi, off, idx, None, elem="s8", dim=d, row_sums_=sums)
        assert np.array_equal(out[t].view(np.uint32), r_ref.view(np.uint32)), t
        assert np.array_equal(fl[t], e_ref), t
    total = int(fl.astype(np.int64).sum())
    assert int(cnt.item()) == total


def test_peer_exchange_world1_matches_oracle():
    """ShardedEmbeddingBags(exchange="peer"): the grouped lookup kernel writes straight into the ranks' symmetric
    receive buffers (peer memory over NVLink at world > 1; the rank's own buffer here, world size 1 -- the only
    GPU count this run has), then a device-side barrier. Identical to the oracle and to the NCCL-exchange path."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2103_00130_b200 import embedding as E
    from paper_2103_00130_b200 import sharded as S
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        T, B, d = 4, 16, 128
        tables, bags, refs = {}, {}, {}
        for t in range(T):
            rows, sc, bi, tab = _table(E, "s8", 2000, d, 60 + t)
            rng = np.random.default_rng(70 + t)
            off = np.concatenate([[0], np.cumsum(rng.integers(0, 40, B))]).astype(np.int64)
            idx = rng.integers(0, 2000, off[-1]).astype(np.int64)
            tables[t], bags[t] = tab, (off, idx, None)
            refs[t] = O.eb(rows, sc, bi, off, idx, None, elem="s8", dim=d)
        try:
            peer = S.ShardedEmbeddingBags(tables, T, B, d, exchange="peer")
        except RuntimeError as e:  # symmetric memory unavailable on this driver / box
            pytest.skip(f"symmetric memory unavailable: {e}")
        for _ in range(2):  # the exchange buffers are reused call to call
            out, flags = peer(bags)
            for t in range(T):
                assert np.array_equal(out[:, t].cpu().numpy().view(np.uint32), refs[t][0].view(np.uint32))
                assert np.array_equal(flags[:, t].cpu().numpy(), refs[t][3])
        out2, flags2 = S.ShardedEmbeddingBags(tables, T, B, d)(bags)
        assert torch.equal(out.view(torch.int32), out2.view(torch.int32)) and torch.equal(flags, flags2)
    finally:
        dist.destroy_process_group()
