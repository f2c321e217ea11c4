"""Tiling configuration, footprint closed forms, the budget object and traffic reports.

Mirrors the reference's boundary types so callers keep their code:

* ``TileConfig``            — pkg/src/flashwin/flash.py:41-71
* ``peak_sram_forward/backward`` — flash.py:84-95
* ``ScratchpadArena``       — memory.py:29-67 (only the budget contract: capacity,
  live/peak bytes and ``CapacityError`` before any work; the on-chip simulator
  itself is replaced by the real SMEM/TMEM of the B200 kernels)
* ``TrafficReport`` / ``merge_reports`` — memory.py:70-98
* ``FlashContext``          — flash.py:74-81 (references, not copies)

On B200, ``r`` (the feature-chunk count) is validated exactly like the
reference but only acts as a tiling hint: the kernels chunk features by the
MMA K-step (16 for fp16/bf16) or 32 (SIMT path); results are r-invariant
(acceptance criterion 9).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Any, Iterable, Optional

from .errors import CapacityError, FlashwinError, InvalidRangeError, ShapeError

DEFAULT_CAPACITY_BYTES = 131072  # memory.py:26


@dataclass(frozen=True)
class TileConfig:
    """Feature-tiling parameters: chunk count r, softmax scale, accounting bytes (flash.py:41-55)."""

    r: int
    scale: float = 1.0
    elem_bytes: int = 4

    def __post_init__(self):
        if self.r < 1:
            raise InvalidRangeError(f"chunk count must be >= 1, got {self.r}")
        if self.elem_bytes not in (4, 8):
            raise InvalidRangeError(f"elem_bytes must be 4 or 8, got {self.elem_bytes}")
        if not math.isfinite(self.scale) or self.scale <= 0:
            raise InvalidRangeError(f"scale must be finite and > 0, got {self.scale}")

    def chunk_width(self, C: int) -> int:
        """Widest chunk, ceil(C/r); validates that r chunks of C features exist (flash.py:57-66)."""
        if self.r > C:
            raise ShapeError(f"chunk count {self.r} exceeds feature count {C}")
        cw = -(-C // self.r)
        if cw * (self.r - 1) >= C:
            raise ShapeError(f"chunk count {self.r} leaves an empty chunk for {C} features")
        return cw

    def chunk_spans(self, C: int) -> list[tuple[int, int]]:
        """Half-open feature spans of the r chunks (flash.py:68-71)."""
        cw = self.chunk_width(C)
        return [(i * cw, min((i + 1) * cw, C)) for i in range(self.r)]


def resolve_r(value, C: int) -> int:
    """'auto' means one chunk per 16 features (harness.py:115-119)."""
    if value == "auto":
        return max(1, C // 16)
    return int(value)


def peak_sram_forward(L: int, C: int, cfg: TileConfig) -> int:
    """(L^2 + 2*L*cw) * elem_bytes (flash.py:84-88)."""
    if L < 1 or C < 1:
        raise ShapeError(f"L and C must be >= 1, got L={L}, C={C}")
    return (L * L + 2 * L * cfg.chunk_width(C)) * cfg.elem_bytes


def peak_sram_backward(L: int, C: int, cfg: TileConfig) -> int:
    """(2*L^2 + 2*L*cw) * elem_bytes (flash.py:91-95)."""
    if L < 1 or C < 1:
        raise ShapeError(f"L and C must be >= 1, got L={L}, C={C}")
    return (2 * L * L + 2 * L * cfg.chunk_width(C)) * cfg.elem_bytes


class ScratchpadArena:
    """Caller-owned on-chip budget (memory.py:29-67).

    The B200 kernels own their real SMEM/TMEM; this object keeps the
    reference's contract: a pass whose paper footprint exceeds
    ``capacity_bytes`` is refused with ``CapacityError`` before any work, and
    ``peak_bytes`` records the high-water mark while ``live_bytes`` returns
    to 0 after every call.
    """

    def __init__(self, capacity_bytes: int = DEFAULT_CAPACITY_BYTES):
        if capacity_bytes < 0:
            raise CapacityError(f"capacity must be >= 0, got {capacity_bytes}")
        self.capacity_bytes = int(capacity_bytes)
        self.live_bytes = 0
        self.peak_bytes = 0

    def check(self, kind: str, need: int) -> None:
        """_check_budget (flash.py:98-103)."""
        if need > self.capacity_bytes:
            raise CapacityError(
                f"{kind} pass needs {need} bytes of scratchpad, "
                f"arena provides {self.capacity_bytes}"
            )

    def record(self, need: int) -> None:
        self.peak_bytes = max(self.peak_bytes, self.live_bytes + int(need))


@dataclass(frozen=True)
class TrafficReport:
    """Per-operand global-memory element counts plus the scratchpad peak (memory.py:70-84).

    ``loads``/``stores`` follow the paper's schedule exactly as the reference
    counts it (Alg. 2 reloads Q and K). ``kernel_loads`` holds what the B200
    kernel actually reads (Q and K once in the backward: P is recomputed from
    tiles that stay on chip), so algorithmic bytes = 7*L*d per unit, not 9.
    """

    loads: dict = field(default_factory=dict)
    stores: dict = field(default_factory=dict)
    peak_sram_bytes: int = 0
    kernel_loads: dict = field(default_factory=dict)

    def total_elements(self) -> int:
        return sum(self.loads.values()) + sum(self.stores.values())


def merge_reports(reports: Iterable[TrafficReport]) -> TrafficReport:
    """Sum counts; peak is per-worker, not summed (memory.py:87-98)."""
    loads: dict[str, int] = {}
    stores: dict[str, int] = {}
    kl: dict[str, int] = {}
    peak = 0
    for rep in reports:
        for name, n in rep.loads.items():
            loads[name] = loads.get(name, 0) + n
        for name, n in rep.stores.items():
            stores[name] = stores.get(name, 0) + n
        for name, n in rep.kernel_loads.items():
            kl[name] = kl.get(name, 0) + n
        peak = max(peak, rep.peak_sram_bytes)
    return TrafficReport(loads=loads, stores=stores, peak_sram_bytes=peak, kernel_loads=kl)


def forward_report(units: int, L: int, C: int, peak: int) -> TrafficReport:
    n = units * L * C
    return TrafficReport(
        loads={"Q": n, "K": n, "V": n}, stores={"O": n}, peak_sram_bytes=peak,
        kernel_loads={"Q": n, "K": n, "V": n},
    )


def backward_report(units: int, L: int, C: int, peak: int) -> TrafficReport:
    n = units * L * C
    return TrafficReport(
        loads={"Q": 2 * n, "K": 2 * n, "V": n, "dO": n},
        stores={"dQ": n, "dK": n, "dV": n},
        peak_sram_bytes=peak,
        kernel_loads={"Q": n, "K": n, "V": n, "dO": n},
    )


@dataclass(frozen=True)
class FlashContext:
    """Q/K/V references retained by the forward for recomputation (flash.py:74-81).

    ``bias``/``mask``/``mask_windows`` are the Swin extension (None = reference
    behaviour). No P, O or log-sum-exp is stored: the backward recomputes P.
    """

    q: Any
    k: Any
    v: Any
    cfg: TileConfig
    bias: Optional[Any] = None
    mask: Optional[Any] = None
    mask_windows: int = 0


def is_context(ctx) -> bool:
    return isinstance(ctx, FlashContext) and all(t is not None for t in (ctx.q, ctx.k, ctx.v))


__all__ = [
    "DEFAULT_CAPACITY_BYTES",
    "FlashContext",
    "FlashwinError",
    "ScratchpadArena",
    "TileConfig",
    "TrafficReport",
    "backward_report",
    "forward_report",
    "merge_reports",
    "peak_sram_backward",
    "peak_sram_forward",
    "resolve_r",
]
