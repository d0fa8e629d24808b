"""Device-memory plumbing for the Python host layer (torch is only the allocator/stream owner)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 ABFT operators need a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream=None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> C.c_void_p | None:
    return None if t is None else C.c_void_p(t.data_ptr())


def to_device(x, dtype: torch.dtype, ndim: int | None = None) -> torch.Tensor:
    """Contiguous device tensor of `dtype` (bit-preserving for same-width integer views)."""
    if isinstance(x, torch.Tensor):
        t = x
    else:
        arr = np.asarray(x)
        np_dtype = {torch.int8: np.int8, torch.uint8: np.uint8, torch.int32: np.int32, torch.int64: np.int64,
                    torch.float32: np.float32, torch.float16: np.float16}[dtype]
        if arr.dtype != np_dtype:
            arr = arr.astype(np_dtype)
        t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.dtype != dtype:
        if t.element_size() == torch.empty((), dtype=dtype).element_size() and not t.is_floating_point() \
                and not torch.empty((), dtype=dtype).is_floating_point():
            t = t.view(dtype)
        else:
            t = t.to(dtype)
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"expected a {ndim}-D array, got shape {tuple(t.shape)}")
    return t.to(device()).contiguous()
