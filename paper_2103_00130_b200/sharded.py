"""Multi-GPU sharding of the ABFT path. One process per GPU, torch.distributed
for the plumbing (NCCL on GPUs; gloo in the CPU tests).

* GEMM shards by N columns. Rank g encodes ITS OWN shard B[:, n0:n1] -- its own mod-127 checksums,
  never exchanged -- and runs the checked kernel on it. The only collective is the OR of the per-row
  verdicts (all-reduce MAX on uint8[m]); for a single fault this equals the reference's global check
  (P:src/gemm_abft.cpp:113-124) because the fault perturbs only its shard's row sum. C stays sharded.
* EmbeddingBag shards table-wise: table t lives on rank t % G with its row sums. Each rank pools its
  tables for the whole batch, and the pooled vectors + verdicts are transposed to batch-sharded
  [B/G, T, d] by ONE all_to_all_single. On the GPU the lookup kernel writes every bag straight into its
  destination slot of the exchange buffer (abftlp_eb_checked_scatter), so no gather/copy kernel sits
  between the lookups and the collective; with NVLink peer mappings the same kernel can target the
  peers' receive buffers directly. Per-bag math is unchanged by sharding, so outputs and verdicts are
  bit-identical to one GPU.

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


class GpuEbBackend:
    """The CUDA library. `run_into` pools one table's bags straight into the exchange buffer slots."""

    def run_into(self, table, offsets, indices, weights, send, send_flags, slot: int) -> None:
        from .embedding import eb_csr_scatter
        G, Bg, Tg, d = (int(s) for s in send.shape)
        outs = [send[g, 0, slot] for g in range(G)]
        flags = [send_flags[g, 0, slot:] for g in range(G)]
        eb_csr_scatter(table, offsets, indices, weights, outs, flags, ld_out=Tg * d, flag_ld=Tg, bags_per_dest=Bg)

    def run_all_into(self, tables: list, bags: list, send, send_flags) -> None:
        """All local tables (slot order) in ONE launch when they share type and dim (abftlp_eb_group_*)."""
        from .embedding import eb_group_scatter
        G, Bg, Tg, d = (int(s) for s in send.shape)
        same = len({(t.elem, t.scale_dtype, t.dim()) for t in tables}) == 1 and \
            len({w is None for _, _, w in bags}) == 1
        if len(tables) < 2 or not same:
            for slot, (table, (off, idx, w)) in enumerate(zip(tables, bags)):
                self.run_into(table, off, idx, w, send, send_flags, slot)
            return
        outs = [[send[g, 0, slot] for g in range(G)] for slot in range(len(tables))]
        flags = [[send_flags[g, 0, slot:] for g in range(G)] for slot in range(len(tables))]
        eb_group_scatter(tables, bags, outs, flags, ld_out=Tg * d, flag_ld=Tg, bags_per_dest=Bg)


class PeerExchange:
    """The table-wise all-to-all fused into the lookups over NVLink peer memory: every rank's receive
    buffers [G, B/G, Tg, d] (+ flags) live in symmetric memory, and rank r's grouped lookup kernel writes bag b of
    its table slot s straight into destination rank g = b // (B/G)'s buffer at [r, b % (B/G), s] -- no send buffer,
    no separate all-to-all; one device-side barrier orders the peers' writes before the consumer reads."""

    def __init__(self, G: int, Bg: int, Tg: int, d: int, group, device):
        import torch.distributed._symmetric_memory as symm
        self.G, self.Bg, self.Tg, self.d = G, Bg, Tg, d
        self.recv = symm.empty(G, Bg, Tg, d, dtype=torch.float32, device=device)
        self.recv_f = symm.empty(G, Bg, Tg, dtype=torch.uint8, device=device)
        name = (group or dist.group.WORLD).group_name
        self.h = symm.rendezvous(self.recv, name)
        self.hf = symm.rendezvous(self.recv_f, name)
        self.rank = self.h.rank

    def destinations(self, slot: int):
        """Per destination rank g: the address of peer g's recv[rank, 0, slot] (pooled rows) and recv_f[...] (flags)."""
        r, Bg, Tg, d = self.rank, self.Bg, self.Tg, self.d
        outs = [int(p) + ((r * Bg) * Tg + slot) * d * 4 for p in self.h.buffer_ptrs]
        flags = [int(p) + (r * Bg) * Tg + slot for p in self.hf.buffer_ptrs]
        return outs, flags

    def barrier(self):
        self.h.barrier()


class ShardedEmbeddingBags:
    """Table-wise sharded checked EmbeddingBag for a batch of `batch` samples over `num_tables` tables.
    `tables` maps this rank's table ids (t % G == rank) to their tables. Returns, for this rank's slice of
    the batch (samples [rank*B/G, (rank+1)*B/G)), pooled outputs [B/G, T, d] and verdicts [B/G, T]."""

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
        self.Tg = -(-num_tables // self.world)  # slots per rank (padded when T % G != 0)
        self.backend = backend or GpuEbBackend()
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        if exchange not in ("nccl", "peer"):
            raise ValueError("ShardedEmbeddingBags: exchange must be 'nccl' or 'peer'")
        # "peer": lookups write straight into the destination ranks' symmetric buffers (GPU backend only)
        self.peer = PeerExchange(self.world, self.B // self.world, self.Tg, dim, group, self.device) \
            if exchange == "peer" else None

    def __call__(self, bags: dict) -> tuple[torch.Tensor, torch.Tensor]:
        """bags[t] = (offsets[B+1], indices, weights-or-None) for every local table t."""
        G, Bg, Tg, d = self.world, self.B // self.world, self.Tg, self.d
        order = sorted(self.tables)
        for t in order:
            if len(bags[t][0]) != self.B + 1:
                raise ValueError("ShardedEmbeddingBags: every table needs one bag per sample")
        if self.peer is not None:  # lookups + exchange in one grouped launch over peer memory
            from .embedding import eb_group_scatter
            dst = [self.peer.destinations(slot) for slot in range(len(order))]
            self.peer.barrier()  # every peer has consumed its previous exchange before it is overwritten
            eb_group_scatter([self.tables[t] for t in order], [bags[t] for t in order], [o for o, _ in dst],
                             [f for _, f in dst], ld_out=Tg * d, flag_ld=Tg, bags_per_dest=Bg)
            self.peer.barrier()
            return self._gather(self.peer.recv, self.peer.recv_f)
        send = torch.zeros((G, Bg, Tg, d), dtype=torch.float32, device=self.device)
        send_f = torch.zeros((G, Bg, Tg), dtype=torch.uint8, device=self.device)
        if hasattr(self.backend, "run_all_into"):  # all local tables in one launch
            self.backend.run_all_into([self.tables[t] for t in order], [bags[t] for t in order], send, send_f)
        else:
            for slot, t in enumerate(order):
                off, idx, w = bags[t]
                self.backend.run_into(self.tables[t], off, idx, w, send, send_f, slot)
        if G > 1:
            recv = torch.empty_like(send)
            recv_f = torch.empty_like(send_f)
            dist.all_to_all_single(recv, send, group=self.group)
            dist.all_to_all_single(recv_f, send_f, group=self.group)
        else:
            recv, recv_f = send, send_f
        return self._gather(recv, recv_f)

    def _gather(self, recv, recv_f):
        """[G, B/G, Tg, d] received slots -> this rank's samples [B/G, T, d] in table order."""
        G, Bg, d = self.world, self.B // self.world, self.d
        out = torch.empty((Bg, self.T, d), dtype=torch.float32, device=self.device)
        flags = torch.empty((Bg, self.T), dtype=torch.uint8, device=self.device)
        for g in range(G):
            for slot, t in enumerate(local_tables(self.T, G, g)):
                out[:, t] = recv[g, :, slot]
                flags[:, t] = recv_f[g, :, slot]
        return out, flags


def sample_slice(batch: int, world: int, rank: int) -> slice:
    bg = batch // world
    return slice(rank * bg, (rank + 1) * bg)


__all__: Sequence[str] = ["column_shard", "ShardedAbftGemm", "ShardedGemmResult", "GpuGemmBackend", "table_owner",
                          "local_tables", "GpuEbBackend", "ShardedEmbeddingBags", "sample_slice"]
