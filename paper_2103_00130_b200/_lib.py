"""ctypes binding of libabftlp_b200.so (include/abftlp.h + include/abftlp_b200.h).

The shared library is the only compute path: if it is missing this module raises at import
time -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("ABFTLP_B200_LIB", _PKG / "libabftlp_b200.so"))

OK, ERR_INVALID_ARGUMENT, ERR_IO, ERR_PARSE, ERR_INTERNAL = 0, -1, -2, -3, -4


class AbftError(RuntimeError):
    """Non-OK status from the C ABI; ``status`` is the abftlp status code."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


class InvalidArgument(AbftError, ValueError):
    pass


class IoError(AbftError, OSError):
    pass


class ParseError(AbftError, ValueError):
    pass


class InternalError(AbftError):
    pass


_ERRORS = {ERR_INVALID_ARGUMENT: InvalidArgument, ERR_IO: IoError, ERR_PARSE: ParseError, ERR_INTERNAL: InternalError}

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(the B200 path has no CPU fallback)")

lib = C.CDLL(str(LIB_PATH))

vp, u64, i64, u32, i32, f64 = C.c_void_p, C.c_uint64, C.c_int64, C.c_uint32, C.c_int32, C.c_double
P = C.POINTER


class Analysis(C.Structure):
    _fields_ = [(n, f64) for n in ("encode_overhead_a", "encode_overhead_b", "p_detect_b_bitflip",
                                   "p_detect_b_random", "p_detect_c_bitflip", "p_detect_c_random",
                                   "eb_overhead", "eb_memory_overhead")]


class BenchResult(C.Structure):
    _fields_ = [("baseline_ns", f64), ("abft_ns", f64), ("overhead_fraction", f64)]


class RequantParams(C.Structure):
    """abftlp_requant_params (RequantParams, P:src/quant.hpp:24-32)."""
    _fields_ = [("scaleA", C.c_double), ("biasA", C.c_double), ("scaleB", C.c_double), ("biasB", C.c_double),
                ("scaleC", C.c_double), ("biasC", C.c_double), ("k", C.c_uint64)]


class BatchFault(C.Structure):
    """abftlp_batch_fault."""
    _fields_ = [("active", C.c_int32), ("batch", C.c_uint64), ("row", C.c_uint64), ("col", C.c_uint64),
                ("bit", C.c_uint32)]


class GemmProblem(C.Structure):
    """abftlp_gemm_problem (one problem of a heterogeneous grouped GEMM)."""
    _fields_ = [("d_a", C.c_void_p), ("m", C.c_uint64), ("lda", C.c_uint64), ("w", C.c_void_p), ("d_c", C.c_void_p),
                ("ldc", C.c_uint64), ("d_csum", C.c_void_p), ("csum_ld", C.c_uint64), ("d_row_flags", C.c_void_p),
                ("d_err_count", C.c_void_p)]


class LocateResult(C.Structure):
    """abftlp_locate_result."""
    _fields_ = [("status", C.c_int32), ("row", C.c_int64), ("col", C.c_int64), ("delta", C.c_int64),
                ("rows_flagged", C.c_uint64), ("cols_mismatched", C.c_uint64)]


class Fault(C.Structure):
    _fields_ = [("active", i32), ("row", u64), ("col", u64), ("bit", u32)]


_SIGS = {
    # reference-compatible surface
    "abftlp_status_str": (C.c_char_p, [i32]),
    "abftlp_last_error": (C.c_char_p, []),
    "abftlp_campaign_load": (i32, [C.c_char_p, P(vp)]),
    "abftlp_campaign_parse": (i32, [C.c_char_p, P(vp)]),
    "abftlp_campaign_free": (None, [vp]),
    "abftlp_campaign_run": (i32, [vp, P(vp)]),
    "abftlp_report_free": (None, [vp]),
    "abftlp_report_trials": (u64, [vp]),
    "abftlp_report_detected": (u64, [vp]),
    "abftlp_report_false_positives": (u64, [vp]),
    "abftlp_report_detection_rate": (f64, [vp]),
    "abftlp_report_write_csv": (i32, [vp, C.c_char_p]),
    "abftlp_report_render": (i32, [vp, P(vp)]),
    "abftlp_string_free": (None, [vp]),
    "abftlp_analyze": (i32, [u64, u64, u64, u64, u64, P(Analysis)]),
    "abftlp_bench_gemm": (i32, [u64, u64, u64, u32, u64, P(BenchResult)]),
    "abftlp_bench_eb": (i32, [u64, u64, u64, u64, u32, u64, P(BenchResult)]),
    "abftlp_eb_check_files": (i32, [C.c_char_p, C.c_char_p, C.c_int, P(u64), P(u64), P(vp)]),
    # device operators
    "abftlp_gemm_encode": (i32, [vp, u64, u64, u64, vp, P(vp)]),
    "abftlp_gemm_weight_free": (None, [vp]),
    "abftlp_gemm_weight_dims": (i32, [vp, P(u64), P(u64)]),
    "abftlp_gemm_weight_checksums": (i32, [vp, vp, vp]),
    "abftlp_gemm_weight_set_checksums": (i32, [vp, vp, vp]),
    "abftlp_gemm_weight_read": (i32, [vp, vp, vp]),
    "abftlp_gemm_checked": (i32, [vp, u64, u64, vp, vp, u64, vp, u64, vp, vp, P(Fault), vp]),
    "abftlp_gemm_unchecked": (i32, [vp, u64, u64, vp, vp, u64, vp]),
    "abftlp_gemm_verify": (i32, [vp, u64, vp, u64, u64, u64, vp, vp, vp]),
    "abftlp_gemm_checked_host": (i32, [vp, u64, u64, vp, vp, u64, vp, vp, vp, vp]),
    "abftlp_eb_table_create": (i32, [i32, vp, u64, u64, u64, i32, vp, vp, vp, vp, P(vp)]),
    "abftlp_eb_table_free": (None, [vp]),
    "abftlp_eb_group_free": (None, [vp]),
    "abftlp_eb_table_validate": (i32, [vp, vp, vp, P(u64)]),
    "abftlp_eb_table_row_sums": (i32, [vp, vp, vp]),
    "abftlp_eb_checked": (i32, [vp, vp, vp, u64, vp, vp, u64, vp, vp, vp, vp, vp, vp]),
    "abftlp_eb_unchecked": (i32, [vp, vp, vp, u64, vp, vp, u64, vp, vp]),
    "abftlp_gemm_encode_batched": (i32, [vp, u64, u64, u64, u64, u64, vp, vp]),
    "abftlp_gemm_checked_batched": (i32, [vp, u64, u64, u64, u64, vp, vp, u64, u64, vp, u64, u64, vp, u64, vp, vp, vp]),
    "abftlp_gemm_checked_host_batched": (i32, [vp, u64, u64, u64, u64, vp, vp, u64, u64, vp, u64, vp, u64, vp, vp]),
    "abftlp_gemm_weight_flip_bit_batched": (i32, [vp, u64, u64, u64, u32, vp]),
    "abftlp_gemm_reencode": (i32, [vp, vp, u64, vp]),
    "abftlp_gemm_checked_batched_faults": (i32, [vp, u64, u64, u64, u64, vp, vp, u64, u64, vp, u64, u64, vp, u64, vp, vp, u64, vp]),
    "abftlp_gemm_unchecked_batched": (i32, [vp, u64, u64, u64, u64, vp, vp, u64, u64, vp]),
    "abftlp_gemm_checked_requant": (i32, [vp, u64, u64, vp, vp, u64, vp, u64, vp, vp, vp, vp, vp, vp, vp, u64, vp]),
    "abftlp_gemm_checked_requant_host_batched": (i32, [vp, u64, u64, u64, u64, vp, vp, vp, u64, u64, vp, u64, vp, u64, vp, vp]),
    "abftlp_requantize": (i32, [vp, u64, u64, u64, vp, vp, vp, vp, u64, vp]),
    "abftlp_row_sums_u8": (i32, [vp, u64, u64, u64, vp, vp]),
    "abftlp_gemm_weight_col_sums": (i32, [vp, vp, vp]),
    "abftlp_eb_group_create": (i32, [vp, u32, vp, vp, vp, vp, vp, vp]),
    "abftlp_gemm_group_create": (i32, [vp, u32, i32, P(vp)]),
    "abftlp_gemm_group_run": (i32, [vp, vp]),
    "abftlp_gemm_locate": (i32, [vp, u64, u64, vp, vp, u64, vp, u64, vp, i32, vp, vp]),
    "abftlp_gemm_group_free": (None, [vp]),
    "abftlp_eb_group_checked_scatter": (i32, [vp, u64, u64, u64, u64, vp, vp, vp]),
    "abftlp_eb_group_unchecked_scatter": (i32, [vp, u64, u64, u64, vp, vp]),
    "abftlp_eb_group_set_bags": (i32, [vp, vp, vp, vp, vp]),
    "abftlp_eb_checked_scatter": (i32, [vp, vp, vp, u64, vp, vp, u64, vp, u64, u64, vp, vp, vp]),
    "abftlp_flip_bit": (i32, [vp, u32, u64, u32, vp]),
    "abftlp_gemm_weight_flip_bit": (i32, [vp, u64, u64, u32, vp]),
    "abftlp_eb_table_flip_bit": (i32, [vp, u64, u64, u32, vp]),
    "abftlp_eb_table_flip_bits": (i32, [vp, vp, vp, vp, u64, vp, vp]),
    "abftlp_generate": (i32, [vp, u64, u64, u64, u64, i32, f64, f64, u64, vp]),
    "abftlp_l2_flush": (i32, [vp, u64, i32, vp]),
    "abftlp_gather_probe": (i32, [vp, u64, vp, u64, vp, vp]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)


def last_error() -> str:
    return (lib.abftlp_last_error() or b"").decode()


def check(status: int) -> None:
    """Raise the Python exception matching a non-OK abftlp status."""
    if status != OK:
        raise _ERRORS.get(status, AbftError)(status, last_error())


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args))
