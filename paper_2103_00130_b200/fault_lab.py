"""Host mirror of the reference's fault lab (P:src/fault_lab.hpp:15-121) and the tooling C ABI.

Injectors draw their coordinates with the reference's SplitMix64 streams (seed, 4*trial + 1) and
apply the mutation on the device; campaigns run entirely on the GPU through
``abftlp_campaign_run`` and reproduce the reference's reports draw for draw.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import IntEnum
from typing import Sequence

import numpy as np
import torch

from . import _lib
from ._device import ptr, stream_handle
from .embedding import IndexBag, QuantEmbeddingTable
from .gemm import AbftGemmResult, IntermediateMatrix, PackedEncodedWeight
from .rng import SplitMix64


class FaultTarget(IntEnum):
    weight_B = 0
    intermediate_C = 1
    eb_table = 2
    none = 3


class FaultModel(IntEnum):
    single_bit_flip = 0
    random_value = 1


class BitRange(IntEnum):
    all = 0
    high4 = 1
    low4 = 2


@dataclass
class FaultSpec:
    target: FaultTarget = FaultTarget.none
    model: FaultModel = FaultModel.single_bit_flip
    bitRange: BitRange = BitRange.all
    seed: int = 0


@dataclass
class FaultRecord:
    injected: bool = False
    position: str = ""
    before: int = 0
    after: int = 0


kData, kInject, kBags, kStride = 0, 1, 2, 4


def trial_rng(seed: int, trial: int, role: int) -> SplitMix64:
    """Per-trial stream (P:src/fault_lab.cpp:19-21)."""
    return SplitMix64(seed, trial * kStride + role)


def flip_bit(value: int, bit: int, width: int) -> int:
    """XOR one bit of a `width`-bit two's-complement integer (P:src/fault_lab.hpp:87-93)."""
    if bit >= width:
        raise IndexError("flip_bit: bit index out of range")
    u = (value & ((1 << width) - 1)) ^ (1 << bit)
    return u - (1 << width) if u >= 1 << (width - 1) else u


def draw_bit_index(rng: SplitMix64, rng_range: BitRange, width: int) -> int:
    """P:src/fault_lab.cpp:89-96."""
    if rng_range == BitRange.high4:
        return width - 4 + rng.next_below(4)
    if rng_range == BitRange.low4:
        return rng.next_below(4)
    return rng.next_below(width)


def _redraw(rng: SplitMix64, cur: int, width: int) -> int:
    while True:
        nv = rng.next_int(-128, 127) if width == 8 else _to_i32(rng.next())
        if nv != cur:
            return nv


def _to_i32(u: int) -> int:
    u &= 0xFFFFFFFF
    return u - (1 << 32) if u >= 1 << 31 else u


def inject_weight_B(pb: PackedEncodedWeight, spec: FaultSpec, trial: int) -> FaultRecord:
    """Corrupt one element of B after encoding, checksum column excluded (P:src/fault_lab.cpp:98-115)."""
    if spec.target == FaultTarget.none:
        return FaultRecord()
    rng = trial_rng(spec.seed, trial, kInject)
    i, j = rng.next_below(pb.k()), rng.next_below(pb.n())
    before = pb.at(i, j)
    if spec.model == FaultModel.single_bit_flip:
        pb.flip_bit(i, j, draw_bit_index(rng, spec.bitRange, 8))
    else:
        nv = _redraw(rng, before, 8)
        for bit in range(8):  # reach the new value through bit flips of the device element
            if ((before ^ nv) >> bit) & 1:
                pb.flip_bit(i, j, bit)
    return FaultRecord(True, f"({i},{j})", before, pb.at(i, j))


def inject_intermediate_C(c: AbftGemmResult | IntermediateMatrix, spec: FaultSpec, trial: int) -> FaultRecord:
    """Corrupt one int32 of C' (any column, checksum included) (P:src/fault_lab.cpp:117-137)."""
    if spec.target == FaultTarget.none:
        return FaultRecord()
    im = c.cTemp if isinstance(c, AbftGemmResult) else c
    rows, cols = (int(s) for s in im.data.shape)
    rng = trial_rng(spec.seed, trial, kInject)
    i, j = rng.next_below(rows), rng.next_below(cols)
    before = int(im.data[i, j].item())
    if spec.model == FaultModel.single_bit_flip:
        bit = draw_bit_index(rng, spec.bitRange, 32)
        _lib.call("abftlp_flip_bit", ptr(im.data), 4, i * cols + j, bit, stream_handle())
    else:
        im.data[i, j] = _redraw(rng, before, 32)
    return FaultRecord(True, f"({i},{j})", before, int(im.data[i, j].item()))


def inject_eb_table(table: QuantEmbeddingTable, bags: Sequence[IndexBag], spec: FaultSpec, trial: int) -> FaultRecord:
    """Corrupt one element of a row pooled by a non-empty bag (P:src/fault_lab.cpp:139-166)."""
    if spec.target == FaultTarget.none:
        return FaultRecord()
    rng = trial_rng(spec.seed, trial, kInject)
    usable = [b for b in range(len(bags)) if len(bags[b].indices)]
    if not usable:
        raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "inject_eb_table: all bags empty")
    bag = bags[usable[rng.next_below(len(usable))]]
    row = int(bag.indices[rng.next_below(len(bag.indices))])
    col = rng.next_below(table.dim())
    width = 4 if table.elem == "u4" else 8

    def read() -> int:
        if table.elem == "u4":
            return (int(table.rows[row, col // 2].item()) >> (4 * (col & 1))) & 0xF
        return int(table.rows[row, col].item())
    before = read()
    if spec.model == FaultModel.single_bit_flip:
        table.flip_bit(row, col, draw_bit_index(rng, spec.bitRange, width))
    else:
        nv = _redraw(rng, before, 8) if width == 8 else None
        if nv is None:
            raise ValueError("random_value model is defined for 8-bit tables")
        for bit in range(8):
            if ((before ^ nv) >> bit) & 1:
                table.flip_bit(row, col, bit)
    return FaultRecord(True, f"({row},{col})", before, read())


# ---------------------------------------------------------------- campaigns over the C ABI
class CampaignReport:
    """Owned abftlp_report handle (P:src/fault_lab.hpp:66-80 accessors)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib.lib.abftlp_report_free(h)
            self._h = None

    @property
    def trials(self) -> int:
        return int(_lib.lib.abftlp_report_trials(self._h))

    @property
    def detected(self) -> int:
        return int(_lib.lib.abftlp_report_detected(self._h))

    @property
    def falsePositives(self) -> int:
        return int(_lib.lib.abftlp_report_false_positives(self._h))

    @property
    def notDetected(self) -> int:
        return self.trials - self.detected

    def detectionRate(self) -> float:
        return float(_lib.lib.abftlp_report_detection_rate(self._h))

    def write_csv(self, path: str) -> None:
        _lib.call("abftlp_report_write_csv", self._h, path.encode())

    def render(self) -> str:
        out = C.c_void_p()
        _lib.call("abftlp_report_render", self._h, C.byref(out))
        try:
            return C.string_at(out).decode()
        finally:
            _lib.lib.abftlp_string_free(out)


class Campaign:
    """Owned abftlp_campaign handle: parse (text) or load (path), then run on the GPU."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    @classmethod
    def parse(cls, text: str) -> "Campaign":
        h = C.c_void_p()
        _lib.call("abftlp_campaign_parse", text.encode(), C.byref(h))
        return cls(h)

    @classmethod
    def load(cls, path: str) -> "Campaign":
        h = C.c_void_p()
        _lib.call("abftlp_campaign_load", path.encode(), C.byref(h))
        return cls(h)

    def run(self) -> CampaignReport:
        r = C.c_void_p()
        _lib.call("abftlp_campaign_run", self._h, C.byref(r))
        return CampaignReport(r)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib.lib.abftlp_campaign_free(h)
            self._h = None


def run_campaign(config_text: str) -> CampaignReport:
    return Campaign.parse(config_text).run()


def analyze(m: int, n: int, k: int, d: int, pool: int) -> dict:
    """Closed-form overheads and detection probabilities (abftlp_analyze)."""
    a = _lib.Analysis()
    _lib.call("abftlp_analyze", m, n, k, d, pool, C.byref(a))
    return {name: getattr(a, name) for name, _ in _lib.Analysis._fields_}


def bench_gemm(m: int, n: int, k: int, repetitions: int = 5, seed: int = 0) -> dict:
    r = _lib.BenchResult()
    _lib.call("abftlp_bench_gemm", m, n, k, repetitions, seed, C.byref(r))
    return {"baseline_ns": r.baseline_ns, "abft_ns": r.abft_ns, "overhead_fraction": r.overhead_fraction}


def bench_eb(table_rows: int, dim: int, pooling: int, batch: int, repetitions: int = 5, seed: int = 0) -> dict:
    r = _lib.BenchResult()
    _lib.call("abftlp_bench_eb", table_rows, dim, pooling, batch, repetitions, seed, C.byref(r))
    return {"baseline_ns": r.baseline_ns, "abft_ns": r.abft_ns, "overhead_fraction": r.overhead_fraction}


def eb_check_files(table_path: str, indices_path: str, skip_validation: bool = False) -> tuple[int, int, str]:
    """(bags, flagged, rendered lines) for an ABEB table and a bag file (abftlp_eb_check_files)."""
    bags, flagged, out = C.c_uint64(), C.c_uint64(), C.c_void_p()
    _lib.call("abftlp_eb_check_files", table_path.encode(), indices_path.encode(), int(bool(skip_validation)),
              C.byref(bags), C.byref(flagged), C.byref(out))
    try:
        text = C.string_at(out).decode() if out.value else ""
    finally:
        if out.value:
            _lib.lib.abftlp_string_free(out)
    return int(bags.value), int(flagged.value), text


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("C", "np", "torch", "dataclass", "IntEnum",
                                                                       "Sequence", "annotations")]
