"""SplitMix64 with (seed, stream) splitting -- the reference's generator (P:src/rng.hpp:10-43).

Counter-based: draw ``e`` (0-based) of stream ``(seed, stream)`` is ``mix(state0 + (e+1)*gamma)``,
which is what lets the device generators (csrc/lab.cu) reproduce host draw sequences.
"""
from __future__ import annotations

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


def mix(z: int) -> int:
    z &= MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


class SplitMix64:
    def __init__(self, seed: int, stream: int = 0):
        self.state = mix((seed & MASK) ^ mix((stream + GAMMA) & MASK))

    def next(self) -> int:
        self.state = (self.state + GAMMA) & MASK
        return mix(self.state)

    def next_below(self, bound: int) -> int:
        return self.next() % bound

    def next_int(self, lo: int, hi: int) -> int:
        return lo + self.next_below(hi - lo + 1)

    def next_double(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def next_real(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_double()


def _mix_np(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def draws(seed: int, stream: int, offset: int, count: int) -> np.ndarray:
    """Raw draws ``offset .. offset+count-1`` of the stream as uint64 (vectorised)."""
    s0 = np.uint64(SplitMix64(seed, stream).state)
    e = np.arange(offset + 1, offset + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix_np(s0 + e * np.uint64(GAMMA))
