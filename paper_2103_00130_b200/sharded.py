"""Multi-GPU sharding of the ABFT path. One process per GPU, torch.distributed
for the plumbing (NCCL on GPUs; gloo in the CPU tests).

* GEMM shards by N columns. Rank g encodes ITS OWN shard B[:, n0:n1] -- its own mod-127 checksums,
  never exchanged -- and runs the checked kernel on it. The only collective is the OR of the per-row
  verdicts (all-reduce MAX on uint8[m]); for a single fault this equals the reference's global check
  (P:src/gemm_abft.cpp:113-124) because the fault perturbs only its shard's row sum. C stays sharded.
* EmbeddingBag shards table-wise: table t lives on rank t % G with its row sums. Each rank pools its
  tables for the whole batch, and the pooled vectors + verdicts are transposed to batch-sharded
  [B/G, T, d] by ONE all_to_all_single of a buffer carrying both. On the GPU one grouped lookup launch
  writes every bag straight into its destination slot of that buffer (abftlp_eb_group_checked_scatter),
  so no gather/copy kernel sits between the lookups and the collective; with exchange="peer" the same
  launch writes into the owning ranks' final buffers over NVLink and there is no collective at all.
  Per-bag math is unchanged by sharding, so outputs and verdicts are bit-identical to one GPU.

The compute backend is pluggable only so the host logic can be tested on CPU processes; the default
backends are the CUDA library (there is no CPU fallback in the product path).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import torch
import torch.distributed as dist


def _world(group) -> tuple[int, int]:
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


# ---------------------------------------------------------------- GEMM (N-column shards)
def column_shard(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous N range [n0, n1) of `rank` (first n % world ranks take one extra column)."""
    if n <= 0 or world <= 0 or not 0 <= rank < world:
        raise ValueError("column_shard: bad arguments")
    base, rem = divmod(n, world)
    n0 = rank * base + min(rank, rem)
    return n0, n0 + base + (1 if rank < rem else 0)


class GpuGemmBackend:
    """The CUDA library: encode once, checked GEMM with per-row flags."""

    def encode(self, b_shard):
        from . import gemm
        return gemm.PackedEncodedWeight(b_shard)

    def run(self, a, w, fault=None):
        from . import gemm
        res = gemm.abft_gemm(a, w, fault=fault)
        return res.cTemp.data, res.rowFlags


@dataclass
class ShardedGemmResult:
    cTemp: torch.Tensor      # this rank's C' shard: m x (n1 - n0 + 1), its own checksum column last
    rowFlags: torch.Tensor   # global verdicts (OR over shards), uint8[m]
    errCount: int            # rows flagged anywhere
    n0: int
    n1: int


class ShardedAbftGemm:
    """Checked GEMM over an N-column-sharded weight. `b_shard` is this rank's B[:, n0:n1]."""

    def __init__(self, b_shard, n_total: int, group=None, backend=None):
        self.group = group
        self.world, self.rank = _world(group)
        self.n0, self.n1 = column_shard(n_total, self.world, self.rank)
        if int(b_shard.shape[1]) != self.n1 - self.n0:
            raise ValueError("ShardedAbftGemm: b_shard width does not match this rank's column range")
        self.backend = backend or GpuGemmBackend()
        self.w = self.backend.encode(b_shard)

    def __call__(self, a, fault=None) -> ShardedGemmResult:
        c, flags = self.backend.run(a, self.w, fault)
        flags = flags.to(torch.uint8).contiguous()
        if self.world > 1:
            dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=self.group)
        return ShardedGemmResult(c, flags, int(flags.to(torch.int64).sum().item()), self.n0, self.n1)


# ---------------------------------------------------------------- EmbeddingBag (table-wise shards)
def table_owner(t: int, world: int) -> int:
    return t % world


def local_tables(num_tables: int, world: int, rank: int) -> list[int]:
    return list(range(rank, num_tables, world))


# The exchange buffer of the NCCL path carries each pooled vector followed by a 16-byte "flag quad" whose first
# byte is the bag's verdict, so ONE all-to-all moves vectors and verdicts together and the rows stay 16-byte
# aligned: x[g, b, slot, :d] = pooled vector, byte 4*d of x[g, b, slot] = flag.
FLAG_QUAD = 4  # floats


class GpuEbBackend:
    """The CUDA library: a rank's tables in ONE persistent grouped launch (abftlp_eb_group_*) whose kernel writes
    every bag straight into its destination slot -- the NCCL exchange buffer, or the peers' final buffers."""

    def __init__(self):
        self.plan = None

    def pool(self, tables: list, bags: list, out_dests: list, flag_dests: list, ld_out: int, flag_ld: int,
             bags_per_dest: int, stream=None):
        from .embedding import EbGroupPlan
        if self.plan is None:
            self.plan = EbGroupPlan(tables, out_dests, flag_dests, ld_out, flag_ld, bags_per_dest)
        self.plan.bind(bags, stream)
        self.plan.launch(True, stream)

    def raise_on_status(self):
        if self.plan is not None:
            self.plan.raise_on_status()

    # NCCL path: slot s of this rank -> x[g, :, s] for every destination rank g
    def pool_into(self, tables: list, bags: list, x: torch.Tensor, d: int, stream=None):
        G, Bg, Tg, D4 = (int(v) for v in x.shape)
        base = x.data_ptr()
        row = lambda g, s: base + ((g * Bg * Tg) + s) * D4 * 4  # noqa: E731  (byte address of x[g, 0, s, 0])
        outs = [[row(g, s) for g in range(G)] for s in range(len(tables))]
        flags = [[row(g, s) + 4 * d for g in range(G)] for s in range(len(tables))]
        self.pool(tables, bags, outs, flags, ld_out=Tg * D4, flag_ld=Tg * D4 * 4, bags_per_dest=Bg, stream=stream)


class PeerExchange:
    """The table-wise all-to-all fused into the lookups over NVLink peer memory: every rank's FINAL
    buffers -- pooled vectors [B/G, T, d] and verdicts [B/G, T] of its samples -- live in symmetric memory, and
    rank r's grouped lookup kernel writes bag b of table t straight into rank g = b // (B/G)'s out[b % (B/G), t]:
    no send buffer, no collective, no reassembly. One device-side barrier before the launch (every peer has
    consumed the previous step's outputs) and one after (all peers' writes landed) order the exchange."""

    def __init__(self, Bg: int, T: int, d: int, group, device):
        import torch.distributed._symmetric_memory as symm
        self.Bg, self.T, self.d = Bg, T, d
        self.out = symm.empty(Bg, T, d, dtype=torch.float32, device=device)
        self.flags = symm.empty(Bg, T, dtype=torch.uint8, device=device)
        name = (group or dist.group.WORLD).group_name
        self.h = symm.rendezvous(self.out, name)
        self.hf = symm.rendezvous(self.flags, name)
        self.rank = self.h.rank

    def destinations(self, t: int):
        """Per destination rank g: the address of peer g's out[0, t] (pooled rows) and flags[0, t] (verdicts)."""
        return ([int(p) + t * self.d * 4 for p in self.h.buffer_ptrs],
                [int(p) + t for p in self.hf.buffer_ptrs])

    def barrier(self):
        self.h.barrier()


class ShardedEmbeddingBags:
    """Table-wise sharded checked EmbeddingBag for a batch of `batch` samples over `num_tables` tables.
    `tables` maps this rank's table ids (t % G == rank) to their tables. Returns, for this rank's slice of
    the batch (samples [rank*B/G, (rank+1)*B/G)), pooled outputs [B/G, T, d] and verdicts [B/G, T].

    exchange="nccl": the grouped lookup kernel writes into a persistent exchange buffer [G, B/G, Tg, d + 4]
    (vector + flag quad), ONE all_to_all_single moves it, and one copy kernel reorders the received slots into
    table order (table t = slot * G + g). exchange="peer": the kernel writes into the owners' final buffers over
    NVLink (PeerExchange); the returned tensors are views of those buffers, valid until the next call."""

    def __init__(self, tables: dict, num_tables: int, batch: int, dim: int, group=None, backend=None,
                 device: torch.device | str | None = None, exchange: str = "nccl"):
        self.group = group
        self.world, self.rank = _world(group)
        if batch % self.world:
            raise ValueError("ShardedEmbeddingBags: batch must be divisible by the world size")
        mine = local_tables(num_tables, self.world, self.rank)
        if sorted(tables) != mine:
            raise ValueError(f"ShardedEmbeddingBags: rank {self.rank} must own tables {mine}")
        self.tables, self.T, self.B, self.d = tables, num_tables, batch, dim
        self.order = sorted(tables)
        self.Tg = -(-num_tables // self.world)  # slots per rank (padded when T % G != 0)
        self.backend = backend or GpuEbBackend()
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        if exchange not in ("nccl", "peer"):
            raise ValueError("ShardedEmbeddingBags: exchange must be 'nccl' or 'peer'")
        G, Bg = self.world, self.B // self.world
        self.peer = None
        self.local = None
        if exchange == "peer":  # lookups write straight into the destination ranks' final buffers (GPU backend only)
            self.peer = PeerExchange(Bg, num_tables, dim, group, self.device)
        elif G == 1 and hasattr(self.backend, "pool"):  # one rank: the lookups write the final layout directly
            self.local = (torch.empty((Bg, num_tables, dim), dtype=torch.float32, device=self.device),
                          torch.empty((Bg, num_tables), dtype=torch.uint8, device=self.device))
        else:  # persistent exchange buffers; flag quads zeroed once (only their first byte is ever written)
            self.xsend = torch.zeros((G, Bg, self.Tg, dim + FLAG_QUAD), dtype=torch.float32, device=self.device)
            self.xrecv = torch.zeros_like(self.xsend) if G > 1 else self.xsend
            self.out = torch.empty((Bg, self.Tg, G, dim), dtype=torch.float32, device=self.device)
            self.flags = torch.empty((Bg, self.Tg, G), dtype=torch.uint8, device=self.device)

    def __call__(self, bags: dict, stream=None) -> tuple[torch.Tensor, torch.Tensor]:
        """bags[t] = (offsets[B+1], indices, weights-or-None) for every local table t."""
        try:
            return self.launch(bags, stream)
        finally:
            self.backend.raise_on_status()  # (after the exchange: a failing rank never strands its peers)

    def launch(self, bags: dict, stream=None) -> tuple[torch.Tensor, torch.Tensor]:
        """The step without any host synchronisation (CUDA-graph capturable once bound): lookups, exchange and
        reordering are enqueued; index errors are left in the backend's status word."""
        for t in self.order:
            if len(bags[t][0]) != self.B + 1:
                raise ValueError("ShardedEmbeddingBags: every table needs one bag per sample")
        tabs = [self.tables[t] for t in self.order]
        tbags = [bags[t] for t in self.order]
        if self.local is not None:  # world size 1: no exchange, bag b of table t -> out[b, t]
            out, flags = self.local
            self.backend.pool(tabs, tbags, [[out.data_ptr() + t * self.d * 4] for t in self.order],
                              [[flags.data_ptr() + t] for t in self.order], ld_out=self.T * self.d, flag_ld=self.T,
                              bags_per_dest=self.B, stream=stream)
            return out, flags
        if self.peer is not None:  # lookups + exchange in one grouped launch over peer memory
            dst = [self.peer.destinations(t) for t in self.order]
            self.peer.barrier()  # every peer has consumed its previous exchange before it is overwritten
            try:
                self.backend.pool(tabs, tbags, [o for o, _ in dst], [f for _, f in dst], ld_out=self.T * self.d,
                                  flag_ld=self.T, bags_per_dest=self.B // self.world, stream=stream)
            finally:
                self.peer.barrier()  # always reached, so a failing rank cannot strand its peers in the barrier
            return self.peer.out, self.peer.flags
        self.backend.pool_into(tabs, tbags, self.xsend, self.d, stream=stream)
        if self.world > 1:
            dist.all_to_all_single(self.xrecv, self.xsend, group=self.group)
        return unpack_exchange(self.xrecv, self.T, self.d, self.out, self.flags)


def unpack_exchange(x: torch.Tensor, T: int, d: int, out: torch.Tensor | None = None,
                    flags: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """Received exchange buffer [G, B/G, Tg, d + 4] (slot s of sender g = table s * G + g) -> this rank's samples
    [B/G, T, d] and verdicts [B/G, T] in table order: the (slot, g) -> t transpose is one permuted copy each."""
    G, Bg, Tg = (int(v) for v in x.shape[:3])
    if out is None:
        out = torch.empty((Bg, Tg, G, d), dtype=torch.float32, device=x.device)
    if flags is None:
        flags = torch.empty((Bg, Tg, G), dtype=torch.uint8, device=x.device)
    out.copy_(x[..., :d].permute(1, 2, 0, 3))
    flags.copy_(x.view(torch.uint8)[..., 4 * d].permute(1, 2, 0))
    o, f = out.view(Bg, Tg * G, d), flags.view(Bg, Tg * G)
    if Tg * G != T:
        o, f = o[:, :T], f[:, :T]
    return o, f


def sample_slice(batch: int, world: int, rank: int) -> slice:
    bg = batch // world
    return slice(rank * bg, (rank + 1) * bg)


__all__: Sequence[str] = ["column_shard", "ShardedAbftGemm", "ShardedGemmResult", "GpuGemmBackend", "table_owner",
                          "local_tables", "GpuEbBackend", "PeerExchange", "ShardedEmbeddingBags", "sample_slice",
                          "FLAG_QUAD", "unpack_exchange"]
