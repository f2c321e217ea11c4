"""SplitMix64 stream and its device fill (pkg/src/flashwin/tensor.py:74-138).

``Rng`` is the reference's generator (same state update, mixing and
``split``). ``fill_uniform`` draws on the GPU with the same counter formula, so
the values are the reference's float64 draws rounded f64 -> f32 -> dtype: the
CPU oracle reproduces them bit for bit.
"""

from __future__ import annotations

import math

import torch

from . import ops
from .errors import InvalidRangeError, ShapeError

GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1


class Rng:
    __slots__ = ("_state",)

    def __init__(self, seed: int):
        self._state = int(seed) & MASK64

    @property
    def state(self) -> int:
        return self._state

    def next_u64(self) -> int:
        self._state = (self._state + GOLDEN) & MASK64
        z = self._state
        z = ((z ^ (z >> 30)) * MIX1) & MASK64
        z = ((z ^ (z >> 27)) * MIX2) & MASK64
        return z ^ (z >> 31)

    def next_float(self) -> float:
        return (self.next_u64() >> 11) * 2.0**-53

    def split(self) -> "Rng":
        return Rng(self.next_u64())


def fill_uniform(rng: Rng, shape, lo: float = -1.0, hi: float = 1.0, dtype=torch.float32,
                 device="cuda") -> torch.Tensor:
    """Device tensor of i.i.d. U[lo, hi) draws; consumes one draw per element."""
    shape = tuple(int(e) for e in shape)
    if not shape or any(e < 1 for e in shape):
        raise ShapeError(f"all extents must be >= 1, got {shape}")
    if not (math.isfinite(lo) and math.isfinite(hi)) or lo >= hi:
        raise InvalidRangeError(f"need lo < hi, got lo={lo}, hi={hi}")
    out = torch.empty(shape, dtype=dtype, device=device)
    ops.fill_uniform_(out, rng._state, lo, hi)
    rng._state = (rng._state + math.prod(shape) * GOLDEN) & MASK64
    return out


def fill_uniform_at(state: int, offset: int, shape, lo: float = -1.0, hi: float = 1.0,
                    dtype=torch.float32, device="cuda") -> torch.Tensor:
    """Elements [offset, offset + prod(shape)) of the stream a fill_uniform from ``state``
    would draw: a rank fills only its shard of a global tensor, bit-identical to the
    corresponding slice of the whole draw (SplitMix64 is counter-based)."""
    shape = tuple(int(e) for e in shape)
    if not shape or any(e < 1 for e in shape):
        raise ShapeError(f"all extents must be >= 1, got {shape}")
    if not (math.isfinite(lo) and math.isfinite(hi)) or lo >= hi:
        raise InvalidRangeError(f"need lo < hi, got lo={lo}, hi={hi}")
    out = torch.empty(shape, dtype=dtype, device=device)
    ops.fill_uniform_(out, (int(state) + int(offset) * GOLDEN) & MASK64, lo, hi)
    return out
