"""Host mirror of the reference's checked EmbeddingBag API (P:src/embedding_abft.hpp:12-52).

Tables live on the GPU: 8-bit signed rows (the reference's type), plus the BASELINE variants
uint8 and packed 4-bit rows, with fp32 or fp16 per-row scale/bias. Lookups run in the
warp-per-bag kernel through the C ABI; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._device import device, ptr, stream_handle, to_device

kEbRelativeBound = 1e-5
ELEM = {"s8": 0, "u8": 1, "u4": 2}
SCALE = {"f32": 0, "f16": 1}


@dataclass
class IndexBag:
    """Multiset of row indices with optional per-lookup weights (P:src/embedding_abft.hpp:24-27)."""
    indices: Sequence[int] = field(default_factory=list)
    weights: Optional[Sequence[float]] = None


@dataclass
class EbCheckedResult:
    """Pooled vector (fp32), the fp64 sums used by the check, and the verdict (P:src/embedding_abft.hpp:29-34)."""
    r: torch.Tensor
    rSum: float
    cSum: float
    err: bool


class QuantEmbeddingTable:
    """Row-wise quantized table with per-row scale/bias and device-computed int32 row sums.

    ``rows``: R x row_bytes (row_bytes = d for s8/u8, d/2 for u4; element j of a u4 row is
    (byte[j/2] >> 4*(j&1)) & 0xF). The rows are kept alive by this object (the C ABI borrows
    them). ``row_sums`` overrides the computed sums (stale-sum experiments,
    load_table(validate=False) semantics).
    """

    def __init__(self, rows, scales, biases, elem: str = "s8", dim: int | None = None, row_sums=None,
                 scale_dtype: str | None = None, stream=None):
        if elem not in ELEM:
            raise ValueError(f"unknown element type {elem!r}")
        rt = to_device(rows, torch.int8 if elem == "s8" else torch.uint8, ndim=2)
        R, row_bytes = (int(s) for s in rt.shape)
        if dim is None:
            dim = row_bytes * 2 if elem == "u4" else row_bytes
        if scale_dtype is None:
            scale_dtype = "f16" if (isinstance(scales, torch.Tensor) and scales.dtype == torch.float16) or \
                (isinstance(scales, np.ndarray) and scales.dtype == np.float16) else "f32"
        sdt = torch.float16 if scale_dtype == "f16" else torch.float32
        st = to_device(scales, sdt)
        bt = to_device(biases, sdt)
        if st.numel() != R or bt.numel() != R:
            raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "table: scale/bias length mismatch")
        rs = None
        if row_sums is not None:
            rs = to_device(row_sums, torch.int32)
            if rs.numel() != R:
                raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "table: row-sum length mismatch")
        h = C.c_void_p()
        _lib.call("abftlp_eb_table_create", ELEM[elem], ptr(rt) if rt.numel() else C.c_void_p(1), R, dim, row_bytes,
                  SCALE[scale_dtype], ptr(st) if R else C.c_void_p(1), ptr(bt) if R else C.c_void_p(1), ptr(rs),
                  stream_handle(stream), C.byref(h))
        self._h = h
        self.rows, self.scales, self.biases, self._given_sums = rt, st, bt, rs
        self.elem, self.scale_dtype = elem, scale_dtype
        self._R, self._d = R, int(dim)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib.lib.abftlp_eb_table_free(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def numRows(self) -> int:
        return self._R

    def dim(self) -> int:
        return self._d

    @property
    def rowSums(self) -> torch.Tensor:
        """Stored row sums (the given ones if supplied, else the device-computed ones)."""
        if self._given_sums is not None:
            return self._given_sums
        out = torch.empty(self._R, dtype=torch.int32, device=device())
        _lib.call("abftlp_eb_table_row_sums", self._h, ptr(out), stream_handle())
        return out

    def validate(self) -> int:
        """Rows whose stored sum disagrees with the contents (0 when sums were computed here)."""
        if self._given_sums is None:
            return 0
        out = C.c_uint64()
        _lib.call("abftlp_eb_table_validate", self._h, ptr(self._given_sums), stream_handle(), C.byref(out))
        return int(out.value)

    def flip_bit(self, row: int, col: int, bit: int, stream=None) -> None:
        """Corrupt element (row, col) after the row sums were taken (inject_eb_table's point)."""
        _lib.call("abftlp_eb_table_flip_bit", self._h, row, col, bit, stream_handle(stream))

    def flip_bits(self, rows, cols, bits, stream=None) -> None:
        """Batched inject_eb_table: flip bits[i] of element (rows[i], cols[i]) for every i, on the device."""
        r = to_device(rows, torch.int64)
        c = to_device(cols, torch.int64)
        b = to_device(bits, torch.int32)
        if not (r.numel() == c.numel() == b.numel()):
            raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "flip_bits: length mismatch")
        status = torch.zeros(1, dtype=torch.int32, device=device())
        _lib.call("abftlp_eb_table_flip_bits", self._h, ptr(r), ptr(c), ptr(b), r.numel(), ptr(status),
                  stream_handle(stream))
        if int(status.item()) & 2:
            raise IndexError("inject_eb_table: coordinates out of range")


def precompute_row_sums(rows, elem: str = "s8", dim: int | None = None) -> torch.Tensor:
    """int32 per-row element sums (P:src/embedding_abft.cpp:39-45), computed on the device."""
    rt = to_device(rows, torch.int8 if elem == "s8" else torch.uint8, ndim=2)
    R = int(rt.shape[0])
    if R == 0:
        return torch.zeros(0, dtype=torch.int32, device=device())
    ones = torch.ones(R, dtype=torch.float32, device=device())
    return QuantEmbeddingTable(rt, ones, torch.zeros_like(ones), elem=elem, dim=dim).rowSums


def _csr(bags: Sequence[IndexBag]):
    lens = [len(b.indices) for b in bags]
    offsets = np.zeros(len(bags) + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    idx = np.concatenate([np.asarray(b.indices, dtype=np.uint64).astype(np.int64) for b in bags]) if bags and \
        offsets[-1] else np.zeros(0, dtype=np.int64)
    weighted = any(b.weights is not None for b in bags)
    w = None
    if weighted:
        parts = []
        for b in bags:
            if b.weights is not None:
                if len(b.weights) != len(b.indices):
                    raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "embedding_bag: weights length mismatch")
                parts.append(np.asarray(b.weights, dtype=np.float32))
            else:  # 1.0f weights are bit-identical to the unweighted path (P:tests/test_embedding_abft.cpp:120-132)
                parts.append(np.ones(len(b.indices), dtype=np.float32))
        w = np.concatenate(parts) if parts else np.zeros(0, np.float32)
    return offsets, idx, w


def eb_csr(table: QuantEmbeddingTable, offsets, indices, weights=None, checked: bool = True, stream=None):
    """Pooled lookups over CSR bags in one launch. Returns (out[B, d], flags[B], rsum[B], csum[B],
    flag_count) as device tensors (flags/sums/count are None when unchecked)."""
    off = to_device(offsets, torch.int64)
    idx = to_device(indices, torch.int64)
    w = None if weights is None else to_device(weights, torch.float32)
    nb = int(off.numel()) - 1
    d = table.dim()
    dev = device()
    out = torch.zeros((max(nb, 0), d), dtype=torch.float32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    if checked:
        flags = torch.zeros(max(nb, 0), dtype=torch.uint8, device=dev)
        rsum = torch.zeros(max(nb, 0), dtype=torch.float64, device=dev)
        csum = torch.zeros(max(nb, 0), dtype=torch.float64, device=dev)
        cnt = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("abftlp_eb_checked", table.handle, ptr(off), ptr(idx) if idx.numel() else C.c_void_p(8), nb, ptr(w),
                  ptr(out), d, ptr(flags), ptr(rsum), ptr(csum), ptr(cnt), ptr(status), stream_handle(stream))
    else:
        flags = rsum = csum = cnt = None
        _lib.call("abftlp_eb_unchecked", table.handle, ptr(off), ptr(idx) if idx.numel() else C.c_void_p(8), nb,
                  ptr(w), ptr(out), d, ptr(status), stream_handle(stream))
    if int(status.item()) & 1:
        raise IndexError("embedding_bag: index out of range")
    return out, flags, rsum, csum, cnt


def eb_csr_scatter(table: QuantEmbeddingTable, offsets, indices, weights, out_dests, flag_dests, ld_out: int,
                   flag_ld: int, bags_per_dest: int, stream=None) -> torch.Tensor:
    """Checked lookups writing bag b to ``out_dests[b // bags_per_dest]`` row ``b % bags_per_dest`` (row
    stride ``ld_out`` floats) and its flag to ``flag_dests[...]`` (stride ``flag_ld``): the sharded
    exchange fused into the lookup kernel (abftlp_eb_checked_scatter). ``out_dests``/``flag_dests`` are
    device tensors (views) whose first element is the destination base. Returns the flag count."""
    off = to_device(offsets, torch.int64)
    idx = to_device(indices, torch.int64)
    w = None if weights is None else to_device(weights, torch.float32)
    nb = int(off.numel()) - 1
    dev = device()
    optrs = torch.tensor([t.data_ptr() for t in out_dests], dtype=torch.int64, device=dev)
    fptrs = torch.tensor([t.data_ptr() for t in flag_dests], dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("abftlp_eb_checked_scatter", table.handle, ptr(off), ptr(idx) if idx.numel() else C.c_void_p(8), nb,
              ptr(w), ptr(optrs), ld_out, ptr(fptrs), flag_ld, bags_per_dest, ptr(cnt), ptr(status),
              stream_handle(stream))
    if int(status.item()) & 1:
        raise IndexError("embedding_bag: index out of range")
    return cnt


def eb_group_scatter(tables: list, bags: list, out_dests: list, flag_dests: list, ld_out: int, flag_ld: int,
                     bags_per_dest: int, stream=None) -> torch.Tensor:
    """eb_csr_scatter for several tables (one element type, scale type and dim; the same bag count each) in ONE
    launch (abftlp_eb_group_checked_scatter). ``bags[i] = (offsets, indices, weights-or-None)`` of table i;
    ``out_dests[i]`` / ``flag_dests[i]`` are table i's destination lists. Returns the total flag count."""
    T = len(tables)
    dev = device()
    csr = [(to_device(o, torch.int64), to_device(i, torch.int64), None if w is None else to_device(w, torch.float32))
           for o, i, w in bags]
    nb = int(csr[0][0].numel()) - 1
    if any(int(o.numel()) - 1 != nb for o, _, _ in csr):
        raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "eb_group: every table needs the same bag count")
    # destinations: tensors (their first element) or raw device addresses (e.g. peer GPUs' symmetric buffers)
    addr = lambda t: t.data_ptr() if torch.is_tensor(t) else int(t)  # noqa: E731
    optrs = [torch.tensor([addr(t) for t in od], dtype=torch.int64, device=dev) for od in out_dests]
    fptrs = [torch.tensor([addr(t) for t in fd], dtype=torch.int64, device=dev) for fd in flag_dests]
    P = C.c_void_p
    arr = lambda xs: (P * T)(*xs)  # noqa: E731
    weights = None if csr[0][2] is None else arr([P(w.data_ptr()) for _, _, w in csr])
    grp = C.c_void_p()
    _lib.call("abftlp_eb_group_create", arr([t.handle for t in tables]), T, arr([P(o.data_ptr()) for o, _, _ in csr]),
              arr([P(i.data_ptr()) if i.numel() else P(8) for _, i, _ in csr]), weights,
              arr([P(o.data_ptr()) for o in optrs]), arr([P(f.data_ptr()) for f in fptrs]), C.byref(grp))
    try:
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        cnt = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("abftlp_eb_group_checked_scatter", grp, nb, ld_out, flag_ld, bags_per_dest, ptr(cnt), ptr(status),
                  stream_handle(stream))
        if int(status.item()) & 1:
            raise IndexError("embedding_bag: index out of range")
    finally:
        _lib.lib.abftlp_eb_group_free(grp)
    return cnt


class EbGroupPlan:
    """A GPU's tables pooled in ONE launch into FIXED destinations (abftlp_eb_group_*), for a step that repeats:
    built once, then every call only re-points the tables at that call's bags (abftlp_eb_group_set_bags, a
    stream-ordered descriptor copy) when their device addresses changed. ``out_dests[i]`` / ``flag_dests[i]`` are
    table i's per-destination device addresses (ints or tensors: their first element); bag b of table i goes to
    destination ``b // bags_per_dest``, row ``b % bags_per_dest`` (stride ``ld_out`` floats / ``flag_ld`` bytes)."""

    def __init__(self, tables: list, out_dests: list, flag_dests: list, ld_out: int, flag_ld: int, bags_per_dest: int):
        self.tables = list(tables)
        self.ld_out, self.flag_ld, self.bags_per_dest = int(ld_out), int(flag_ld), int(bags_per_dest)
        dev = device()
        addr = lambda t: t.data_ptr() if torch.is_tensor(t) else int(t)  # noqa: E731
        self._optrs = [torch.tensor([addr(t) for t in od], dtype=torch.int64, device=dev) for od in out_dests]
        self._fptrs = [torch.tensor([addr(t) for t in fd], dtype=torch.int64, device=dev) for fd in flag_dests]
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.count = torch.zeros(1, dtype=torch.int32, device=dev)
        self._grp = None
        self._key = None
        self._csr = None

    def _arr(self, xs):
        return (C.c_void_p * len(self.tables))(*xs)

    def bind(self, bags: list, stream=None) -> int:
        """Point the plan at `bags[i] = (offsets, indices, weights-or-None)` (device tensors are used in place)."""
        csr = [(to_device(o, torch.int64), to_device(i, torch.int64), None if w is None else to_device(w, torch.float32))
               for o, i, w in bags]
        nb = int(csr[0][0].numel()) - 1
        if len(csr) != len(self.tables) or any(int(o.numel()) - 1 != nb for o, _, _ in csr):
            raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "eb_group: every table needs the same bag count")
        P = C.c_void_p
        key = tuple((o.data_ptr(), i.data_ptr(), 0 if w is None else w.data_ptr()) for o, i, w in csr)
        offs = self._arr([P(o.data_ptr()) for o, _, _ in csr])
        idxs = self._arr([P(i.data_ptr()) if i.numel() else P(8) for _, i, _ in csr])
        wts = None if csr[0][2] is None else self._arr([P(w.data_ptr()) for _, _, w in csr])
        if self._grp is None:
            grp = C.c_void_p()
            _lib.call("abftlp_eb_group_create", self._arr([t.handle for t in self.tables]), len(self.tables), offs, idxs,
                      wts, self._arr([P(o.data_ptr()) for o in self._optrs]),
                      self._arr([P(f.data_ptr()) for f in self._fptrs]), C.byref(grp))
            self._grp = grp
        elif key != self._key:
            _lib.call("abftlp_eb_group_set_bags", self._grp, offs, idxs, wts, stream_handle(stream))
        self._key, self._csr, self.nb = key, csr, nb  # keep the bags alive while the plan points at them
        return nb

    def launch(self, checked: bool = True, stream=None) -> None:
        """Pool the bound bags (no host synchronisation; errors are reported in ``status``)."""
        if checked:
            _lib.call("abftlp_eb_group_checked_scatter", self._grp, self.nb, self.ld_out, self.flag_ld,
                      self.bags_per_dest, ptr(self.count), ptr(self.status), stream_handle(stream))
        else:
            _lib.call("abftlp_eb_group_unchecked_scatter", self._grp, self.nb, self.ld_out, self.bags_per_dest,
                      ptr(self.status), stream_handle(stream))

    def raise_on_status(self) -> None:
        if int(self.status.item()) & 1:
            self.status.zero_()
            raise IndexError("embedding_bag: index out of range")

    def __call__(self, bags: list, checked: bool = True, stream=None) -> torch.Tensor:
        self.bind(bags, stream)
        self.launch(checked, stream)
        self.raise_on_status()
        return self.count

    def __del__(self):
        if getattr(self, "_grp", None) is not None and _lib.lib is not None:
            _lib.lib.abftlp_eb_group_free(self._grp)
            self._grp = None


def embedding_bag(table: QuantEmbeddingTable, bag: IndexBag) -> torch.Tensor:
    """Plain pooled lookup, fp32 accumulation (P:src/embedding_abft.cpp:47-60)."""
    off, idx, w = _csr([bag])
    return eb_csr(table, off, idx, w, checked=False)[0][0]


def batch_abft_eb(table: QuantEmbeddingTable, bags: Sequence[IndexBag]) -> list[EbCheckedResult]:
    """Independent checked lookups for every bag, one kernel launch (P:src/embedding_abft.cpp:85-91)."""
    if not bags:
        return []
    off, idx, w = _csr(bags)
    out, flags, rsum, csum, _ = eb_csr(table, off, idx, w, checked=True)
    f, rs, cs = flags.cpu().numpy(), rsum.cpu().numpy(), csum.cpu().numpy()
    return [EbCheckedResult(out[b], float(rs[b]), float(cs[b]), bool(f[b])) for b in range(len(bags))]


def abft_embedding_bag(table: QuantEmbeddingTable, bag: IndexBag) -> EbCheckedResult:
    """Lookup plus the row-sum check at the 1e-5 relative bound (P:src/embedding_abft.cpp:62-83)."""
    return batch_abft_eb(table, [bag])[0]


# ---------------------------------------------------------------- ABEB files (P:src/embedding_abft.cpp:93-145)
_MAGIC = b"ABEB"


def save_table(table: QuantEmbeddingTable, path: str) -> None:
    """Binary container: "ABEB", u16 version 1, u64 R, u32 d, R x (d int8, f32 scale, f32 bias), R x i32."""
    if table.elem != "s8" or table.scale_dtype != "f32":
        raise ValueError("ABEB stores int8 rows with fp32 scale/bias")
    rows = table.rows.cpu().numpy().view(np.int8)
    sc = table.scales.cpu().numpy().astype(np.float32)
    bi = table.biases.cpu().numpy().astype(np.float32)
    sums = table.rowSums.cpu().numpy().astype(np.int32)
    R, d = rows.shape
    rec = np.zeros(R, dtype=[("q", np.int8, (d,)), ("s", "<f4"), ("b", "<f4")])
    rec["q"], rec["s"], rec["b"] = rows, sc, bi
    try:
        with open(path, "wb") as f:
            f.write(_MAGIC + struct.pack("<HQI", 1, R, d))
            f.write(rec.tobytes())
            f.write(sums.astype("<i4").tobytes())
    except OSError as e:
        raise _lib.IoError(_lib.ERR_IO, f"cannot open table file for writing: {path}") from e


def load_table(path: str, validateRowSums: bool = True) -> QuantEmbeddingTable:
    """Load an ABEB file onto the device; validation recomputes the sums on the GPU."""
    try:
        with open(path, "rb") as f:
            blob = f.read()
    except OSError as e:
        raise _lib.IoError(_lib.ERR_IO, f"cannot open table file: {path}") from e
    if len(blob) < 4 or blob[:4] != _MAGIC:
        raise _lib.IoError(_lib.ERR_IO, f"not an embedding table file: {path}")
    if len(blob) < 18:
        raise _lib.IoError(_lib.ERR_IO, "table file truncated")
    ver, R, d = struct.unpack_from("<HQI", blob, 4)
    if ver != 1:
        raise _lib.IoError(_lib.ERR_IO, "unsupported table file version")
    if R == 0 or d == 0:
        raise _lib.IoError(_lib.ERR_IO, "table file has empty dimensions")
    need = 18 + R * (d + 8) + 4 * R
    if len(blob) < need:
        raise _lib.IoError(_lib.ERR_IO, "table file truncated")
    rec = np.frombuffer(blob, dtype=[("q", np.int8, (d,)), ("s", "<f4"), ("b", "<f4")], count=R, offset=18)
    sums = np.frombuffer(blob, dtype="<i4", count=R, offset=18 + R * (d + 8))
    t = QuantEmbeddingTable(np.ascontiguousarray(rec["q"]), np.ascontiguousarray(rec["s"]),
                            np.ascontiguousarray(rec["b"]), elem="s8", row_sums=sums.copy())
    if validateRowSums and t.validate() != 0:
        raise _lib.IoError(_lib.ERR_IO, "table row-sum checksums do not match contents")
    return t
