"""Host mirror of the reference's ABFT GEMM API (P:src/gemm_abft.hpp:10-74) over the B200 library.

Same names and argument meaning as the reference; every operator runs on the GPU through the C ABI
(include/abftlp_b200.h). Inputs may be numpy arrays or torch tensors; results are device tensors.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import torch

from . import _lib
from ._device import device, ptr, stream_handle, to_device

kChecksumMod = 127


def mod127(v: int) -> int:
    """Least non-negative residue (P:src/gemm_abft.hpp:13-16)."""
    return int(v) % kChecksumMod


@dataclass
class WeightChecksum:
    """Per-row sums of B mod 127, int8 in [0, 126] (P:src/gemm_abft.hpp:19-21)."""
    values: torch.Tensor


@dataclass
class IntermediateMatrix:
    """32-bit product; the last column is the checksum column when present (P:src/quant.hpp:36-44)."""
    data: torch.Tensor
    hasChecksumColumn: bool = False

    def rows(self) -> int:
        return int(self.data.shape[0])

    def logicalCols(self) -> int:
        return int(self.data.shape[1]) - (1 if self.hasChecksumColumn else 0)


@dataclass
class AbftGemmResult:
    """cTemp m x (n+1) with the checksum column last, number of flagged rows, and the per-row flags
    the B200 epilogue also emits (P:src/gemm_abft.hpp:61-64)."""
    cTemp: IntermediateMatrix
    errCount: int
    rowFlags: torch.Tensor


class PackedEncodedWeight:
    """B encoded once: mod-127 checksums + B' in the GEMM's K-major layout (P:src/gemm_abft.hpp:30-59).

    ``cs`` defaults to the checksums of ``b``; passing a WeightChecksum packs those values instead
    (e.g. the pristine checksums next to a B corrupted after encoding, P:src/fault_lab.cpp:186-189).
    """

    def __init__(self, b, cs: WeightChecksum | None = None, stream=None):
        bt = to_device(b, torch.int8)
        if bt.dim() != 2:
            raise ValueError("PackedEncodedWeight: B must be 2-D")
        k, n = (int(s) for s in bt.shape)
        handle = C.c_void_p()
        _lib.call("abftlp_gemm_encode", ptr(bt) if bt.numel() else C.c_void_p(1), k, n, max(n, 1),
                  stream_handle(stream), C.byref(handle))
        self._h = handle
        self._k, self._n = k, n
        if cs is not None:
            vals = to_device(cs.values, torch.int8)
            if vals.numel() != k:
                raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "PackedEncodedWeight: checksum length mismatch")
            _lib.call("abftlp_gemm_weight_set_checksums", self._h, ptr(vals), stream_handle(stream))
        self._view = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib.lib.abftlp_gemm_weight_free(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def k(self) -> int:
        return self._k

    def n(self) -> int:
        """Original columns, checksum excluded."""
        return self._n

    def checksum(self) -> WeightChecksum:
        out = torch.empty(self._k, dtype=torch.int8, device=device())
        _lib.call("abftlp_gemm_weight_checksums", self._h, ptr(out), stream_handle())
        return WeightChecksum(out)

    def reencode(self, b, stream=None) -> None:
        """Encode a new B of the same shape into this handle, in place (abftlp_gemm_reencode; no allocation)."""
        bt = to_device(b, torch.int8)
        if tuple(int(s) for s in bt.shape) != (self._k, self._n):
            raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "PackedEncodedWeight.reencode: shape mismatch")
        _lib.call("abftlp_gemm_reencode", self._h, ptr(bt), max(self._n, 1), stream_handle(stream))
        self._view = None

    def encoded(self) -> torch.Tensor:
        """Logical k x (n+1) matrix [B | cs]."""
        out = torch.empty((self._k, self._n + 1), dtype=torch.int8, device=device())
        _lib.call("abftlp_gemm_weight_read", self._h, ptr(out), stream_handle())
        return out

    def at(self, i: int, j: int) -> int:
        """Element of the logical k x (n+1) encoded matrix (P:src/gemm_abft.cpp:87-91)."""
        if self._view is None:
            self._view = self.encoded().cpu()
        return int(self._view[i, j])

    def flip_bit(self, i: int, j: int, bit: int, stream=None) -> None:
        """Corrupt B'(i, j) after encoding (j == n hits the checksum column)."""
        _lib.call("abftlp_gemm_weight_flip_bit", self._h, i, j, bit, stream_handle(stream))
        self._view = None


def compute_row_checksums(b) -> WeightChecksum:
    """P:src/gemm_abft.cpp:60-71 (computed by the device encoder)."""
    return PackedEncodedWeight(b).checksum()


def abft_gemm(a, pb: PackedEncodedWeight, fault: tuple[int, int, int] | None = None, stream=None) -> AbftGemmResult:
    """Row-checksum verified product (P:src/gemm_abft.cpp:93-100). ``fault=(row, col, bit)`` flips one
    bit of C' inside the epilogue, after the product and before verification."""
    at = to_device(a, torch.uint8)
    if at.dim() != 2:
        raise ValueError("abft_gemm: A must be 2-D")
    m, k = (int(s) for s in at.shape)
    if k != pb.k():
        raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "abft_gemm: dimension mismatch")
    n = pb.n()
    ctemp = torch.zeros((m, n + 1), dtype=torch.int32, device=device())
    flags = torch.zeros(m, dtype=torch.uint8, device=device())
    err = torch.zeros(1, dtype=torch.int32, device=device())
    f = None
    if fault is not None:
        f = C.byref(_lib.Fault(1, fault[0], fault[1], fault[2]))
    csum_ptr = C.c_void_p(ctemp.data_ptr() + 4 * n) if m else None
    _lib.call("abftlp_gemm_checked", ptr(at) if m else None, m, max(k, 1), pb.handle, ptr(ctemp) if m else None,
              n + 1, csum_ptr, n + 1, ptr(flags), ptr(err), f, stream_handle(stream))
    return AbftGemmResult(IntermediateMatrix(ctemp, True), int(err.item()), flags)


def locate_and_correct(a, pb: PackedEncodedWeight, res: AbftGemmResult, correct: bool = True, stream=None):
    """Dual-encoded locate (and repair) of a flagged checked result in place (abftlp_gemm_locate; the reference's
    dual-encoded oracle P:tests/dual_check.hpp:23-73 as a device operation). Returns the abftlp_locate_result."""
    at = to_device(a, torch.uint8)
    m, k = (int(s) for s in at.shape)
    n = pb.n()
    data = res.cTemp.data
    out = _lib.LocateResult()
    _lib.call("abftlp_gemm_locate", ptr(at), m, k, pb.handle, ptr(data), n + 1, C.c_void_p(data.data_ptr() + 4 * n),
              n + 1, ptr(res.rowFlags), 1 if correct else 0, C.byref(out), stream_handle(stream))
    if correct and out.status in (1, 2):
        res.errCount = int(res.rowFlags.to(torch.int64).sum().item())
    return out


def plain_gemm(a, b) -> IntermediateMatrix:
    """Unchecked baseline (P:src/gemm_abft.cpp:102-111): the same kernel with checking compiled out."""
    at = to_device(a, torch.uint8)
    bt = to_device(b, torch.int8)
    if at.shape[1] != bt.shape[0]:
        raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "plain_gemm: dimension mismatch")
    pb = PackedEncodedWeight(bt)
    m, n = int(at.shape[0]), int(bt.shape[1])
    c = torch.zeros((m, n), dtype=torch.int32, device=device())
    _lib.call("abftlp_gemm_unchecked", ptr(at) if m else None, m, max(int(at.shape[1]), 1), pb.handle,
              ptr(c) if m else None, n, stream_handle())
    return IntermediateMatrix(c, False)


def verify_checksums(c: IntermediateMatrix, flags: torch.Tensor | None = None) -> int:
    """Number of rows whose residue disagrees with the checksum column (P:src/gemm_abft.cpp:113-124)."""
    if not c.hasChecksumColumn:
        raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "verify_checksums: missing checksum column")
    data = to_device(c.data, torch.int32)
    m, cols = (int(s) for s in data.shape)
    n = cols - 1
    err = torch.zeros(1, dtype=torch.int32, device=device())
    csum = C.c_void_p(data.data_ptr() + 4 * n) if m else None
    _lib.call("abftlp_gemm_verify", ptr(data) if m else None, cols, csum, cols, m, n, ptr(flags), ptr(err),
              stream_handle())
    return int(err.item())


class PackedEncodedWeightBatch:
    """`batch` independent encoded weights of one shape (abftlp_gemm_encode_batched): the operand of the
    one-launch batched GEMM (e.g. the reference's seeded trials, each with its own A and B)."""

    def __init__(self, b, stream=None):
        bt = to_device(b, torch.int8)
        if bt.dim() != 3:
            raise ValueError("PackedEncodedWeightBatch: B must be [batch, k, n]")
        self._batch, self._k, self._n = (int(s) for s in bt.shape)
        self._h = C.c_void_p()
        _lib.call("abftlp_gemm_encode_batched", ptr(bt), self._batch, self._k, self._n, self._n, self._k * self._n,
                  stream_handle(stream), C.byref(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib.lib.abftlp_gemm_weight_free(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def batch(self) -> int:
        return self._batch

    def k(self) -> int:
        return self._k

    def n(self) -> int:
        return self._n


def abft_gemm_batched(a, pb, fault: tuple[int, int, int, int] | None = None, stream=None,
                      faults: list[tuple[int, int, int, int]] | None = None):
    """`batch` checked GEMMs in one launch: a is [batch, m, k] u8; ``pb`` is a PackedEncodedWeightBatch (one
    weight per problem) or a single PackedEncodedWeight shared by every problem (a grouped job). Returns
    (cTemp [batch, m, n+1] int32 with the checksum column last, errCount [batch] int32, rowFlags [batch, m]
    u8) as device tensors. ``fault=(problem, row, col, bit)`` flips one bit of that problem's C' in the
    epilogue; ``faults`` is a list of such tuples (at most 8 per call)."""
    at = to_device(a, torch.uint8)
    nb_w = pb.batch() if isinstance(pb, PackedEncodedWeightBatch) else None
    if at.dim() != 3 or (nb_w is not None and int(at.shape[0]) != nb_w) or int(at.shape[2]) != pb.k():
        raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "abft_gemm: dimension mismatch")
    nb, m, k = (int(s) for s in at.shape)
    n = pb.n()
    dev = device()
    ctemp = torch.zeros((nb, m, n + 1), dtype=torch.int32, device=dev)
    flags = torch.zeros((nb, m), dtype=torch.uint8, device=dev)
    err = torch.zeros(nb, dtype=torch.int32, device=dev)
    args = (ptr(at), nb, m, k, m * k, pb.handle, ptr(ctemp), n + 1, m * (n + 1),
            C.c_void_p(ctemp.data_ptr() + 4 * n), n + 1, m * (n + 1), ptr(flags), m, ptr(err))
    if faults is not None:
        arr = (_lib.BatchFault * max(1, len(faults)))(*[_lib.BatchFault(1, *f) for f in faults])
        _lib.call("abftlp_gemm_checked_batched_faults", *args, arr, len(faults), stream_handle(stream))
    else:
        f = C.byref(_lib.BatchFault(1, *fault)) if fault is not None else None
        _lib.call("abftlp_gemm_checked_batched", *args, f, stream_handle(stream))
    return ctemp, err, flags


class AbftGemmGroup:
    """Several checked (or plain) GEMMs of different shapes in ONE persistent launch (abftlp_gemm_group_*): the
    layers of a DLRM MLP, each ``(A, PackedEncodedWeight)``. Each problem writes its own C (m x n), checksum column,
    row flags and flag count -- exactly what one abft_gemm per problem writes (P:src/gemm_abft.cpp:93-124). The
    plan (tile table, tensor maps) is built once; ``run()`` only launches."""

    def __init__(self, problems: Sequence, checked: bool = True):
        self.checked = checked
        self._keep = []
        arr = (_lib.GemmProblem * len(problems))()
        self.outputs = []
        for i, (a, pb) in enumerate(problems):
            at = to_device(a, torch.uint8)
            m, k = (int(s) for s in at.shape)
            if k != pb.k():
                raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "abft_gemm: dimension mismatch")
            n = pb.n()
            c = torch.zeros((m, n), dtype=torch.int32, device=device())
            cs = torch.zeros(m, dtype=torch.int32, device=device()) if checked else None
            fl = torch.zeros(m, dtype=torch.uint8, device=device()) if checked else None
            err = torch.zeros(1, dtype=torch.int32, device=device()) if checked else None
            arr[i] = _lib.GemmProblem(at.data_ptr(), m, k, pb.handle.value, c.data_ptr(), n,
                                      cs.data_ptr() if checked else None, 1, fl.data_ptr() if checked else None,
                                      err.data_ptr() if checked else None)
            self._keep += [at, pb]
            self.outputs.append((c, cs, fl, err))
        h = C.c_void_p()
        _lib.call("abftlp_gemm_group_create", arr, len(problems), 1 if checked else 0, C.byref(h))
        self._h = h

    def run(self, stream=None):
        _lib.call("abftlp_gemm_group_run", self._h, stream_handle(stream))
        return self.outputs

    def __del__(self):
        if getattr(self, "_h", None) is not None and _lib.lib is not None:
            _lib.lib.abftlp_gemm_group_free(self._h)
            self._h = None
