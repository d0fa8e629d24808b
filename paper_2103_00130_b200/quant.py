"""Host mirror of the reference's requantization API (P:src/quant.hpp:24-71) over the B200 library.

``requantize`` replaces the CPU loop of P:src/quant.cpp:77-102 with a CUDA kernel; ``abft_gemm_requant``
is the fused form (the checked GEMM's epilogue writes the u8 C_I straight from TMEM).
Results are bit-identical to the reference (same double operations, same order).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._device import device, ptr, stream_handle, to_device
from .gemm import AbftGemmResult, IntermediateMatrix, PackedEncodedWeight


@dataclass
class RequantParams:
    """RequantParams (P:src/quant.hpp:24-32)."""
    scaleA: float = 1.0
    biasA: float = 0.0
    scaleB: float = 1.0
    biasB: float = 0.0
    scaleC: float = 1.0
    biasC: float = 0.0
    k: int = 1

    def _c(self) -> _lib.RequantParams:
        return _lib.RequantParams(self.scaleA, self.biasA, self.scaleB, self.biasB, self.scaleC, self.biasC, int(self.k))


def row_sums(a) -> torch.Tensor:
    """int32 row sums of a u8 matrix (P:src/quant.cpp:104-110), on the device."""
    at = to_device(a, torch.uint8, ndim=2)
    m, k = (int(s) for s in at.shape)
    out = torch.empty(m, dtype=torch.int32, device=device())
    _lib.call("abftlp_row_sums_u8", ptr(at) if m else None, m, k, max(k, 1), ptr(out), stream_handle())
    return out


def col_sums(b) -> torch.Tensor:
    """int32 column sums of an s8 weight (P:src/quant.cpp:112-118); accepts B or its PackedEncodedWeight."""
    pb = b if isinstance(b, PackedEncodedWeight) else PackedEncodedWeight(b)
    out = torch.empty(pb.n(), dtype=torch.int32, device=device())
    _lib.call("abftlp_gemm_weight_col_sums", pb.handle, ptr(out), stream_handle())
    return out


def requantize(c: IntermediateMatrix, rowSumA, colSumB, p: RequantParams) -> torch.Tensor:
    """u8 m x logicalCols requantized product (P:src/quant.cpp:77-102); the checksum column is never read."""
    data = to_device(c.data, torch.int32, ndim=2)
    m, cols = (int(s) for s in data.shape)
    n = c.logicalCols()
    rs = to_device(rowSumA, torch.int32)
    cs = to_device(colSumB, torch.int32)
    if rs.numel() != m:
        raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "requantize: rowSumA length mismatch")
    if cs.numel() != n:
        raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "requantize: colSumB length mismatch")
    out = torch.empty((m, n), dtype=torch.uint8, device=device())
    prm = p._c()
    _lib.call("abftlp_requantize", ptr(data) if m else None, max(cols, 1), m, n, ptr(rs), ptr(cs), C.byref(prm),
              ptr(out) if m and n else None, max(n, 1), stream_handle())
    return out


def abft_gemm_requant(a, pb: PackedEncodedWeight, rowSumA, colSumB, p: RequantParams,
                      fault: tuple[int, int, int] | None = None, keep_c: bool = True):
    """Checked GEMM + fused requantization: returns (AbftGemmResult | None, u8 C_I [m, n]). With
    ``keep_c=False`` the int32 C' is not written (the verdicts still are)."""
    at = to_device(a, torch.uint8, ndim=2)
    m, k = (int(s) for s in at.shape)
    if k != pb.k():
        raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "abft_gemm: dimension mismatch")
    n = pb.n()
    dev = device()
    rs = to_device(rowSumA, torch.int32)
    cs = to_device(colSumB, torch.int32)
    ctemp = torch.zeros((m, n + 1), dtype=torch.int32, device=dev)
    flags = torch.zeros(m, dtype=torch.uint8, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    out = torch.empty((m, n), dtype=torch.uint8, device=dev)
    f = C.byref(_lib.Fault(1, fault[0], fault[1], fault[2])) if fault is not None else None
    prm = p._c()
    c_ptr = ptr(ctemp) if (m and keep_c) else None
    csum_ptr = C.c_void_p(ctemp.data_ptr() + 4 * n) if m else None
    _lib.call("abftlp_gemm_checked_requant", ptr(at) if m else None, m, max(k, 1), pb.handle, c_ptr, n + 1, csum_ptr,
              n + 1, ptr(flags), ptr(err), f, ptr(rs), ptr(cs), C.byref(prm), ptr(out) if m else None, n,
              stream_handle())
    res = AbftGemmResult(IntermediateMatrix(ctemp, True), int(err.item()), flags)
    return res, out
