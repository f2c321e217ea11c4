"""The reference's operator API, drop-in: flash_forward / flash_backward / batched_flash_forward.

Signatures, argument meaning, validation order and error classes follow
pkg/src/flashwin/flash.py:141-319. Differences that are the point of the
exercise: the math runs in libfwa.so's sm_100a kernels, inputs may be torch
CUDA tensors (zero-copy), torch CPU tensors, NumPy arrays or any object with
an ``.array`` attribute (the reference's DenseTensor); host inputs are copied
to the GPU and results copied back (the e2e path), float64 host data is
computed in float32 (the reference computes in float64; tolerance 1e-5
relative). Outputs come back in the caller's container type.

Added beyond the reference (it has none): ``batched_flash_backward`` over
the (B, h, L, C) stack, plus optional Swin ``bias``/``mask`` keyword args.
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch

from . import ops
from .pipeline import host_backward, host_forward
from .errors import CapacityError, ContextError, FlashwinError, InvalidRangeError, ShapeError
from .tiling import (
    FlashContext,
    ScratchpadArena,
    TileConfig,
    TrafficReport,
    backward_report,
    forward_report,
    is_context,
    peak_sram_backward,
    peak_sram_forward,
)


class HostArray:
    """Minimal read-only host result mirroring DenseTensor's accessors (tensor.py:26-71)."""

    __slots__ = ("_a",)

    def __init__(self, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64)
        a.setflags(write=False)
        self._a = a

    @property
    def shape(self):
        return tuple(self._a.shape)

    @property
    def array(self):
        return self._a

    @property
    def data(self):
        return self._a.reshape(-1)

    @property
    def size(self):
        return self._a.size

    @property
    def ndim(self):
        return self._a.ndim

    def __repr__(self):
        return f"HostArray(shape={self.shape})"


# ---- host <-> device marshalling (the e2e boundary) ---------------------------
class _Kind:
    CUDA, TORCH_CPU, NUMPY, DENSE = range(4)


def _shape_of(x):
    if isinstance(x, torch.Tensor):
        return tuple(x.shape)
    if hasattr(x, "array"):
        return tuple(np.asarray(x.array).shape)
    return tuple(np.asarray(x).shape)


def _to_device(x, dtype: Optional[torch.dtype] = None, device=None):
    """Return (cuda_tensor, kind, host_dtype)."""
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            t = x if dtype is None or x.dtype == dtype else x.to(dtype)
            return t.contiguous(), _Kind.CUDA, x.dtype
        kind, host_dtype = _Kind.TORCH_CPU, x.dtype
        src = x
    else:
        kind = _Kind.DENSE if hasattr(x, "array") else _Kind.NUMPY
        arr = np.asarray(x.array if kind == _Kind.DENSE else x)
        host_dtype = arr.dtype
        src = torch.from_numpy(np.ascontiguousarray(arr))
    if dtype is None:
        dtype = src.dtype if src.dtype in (torch.float16, torch.bfloat16, torch.float32) \
            else torch.float32
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    return src.to(device=dev, dtype=dtype, non_blocking=False).contiguous(), kind, host_dtype


def _to_host_tensor(x, dtype: Optional[torch.dtype] = None):
    """Host torch tensor in a kernel dtype (f16/bf16/f32) + (kind, host dtype) to convert back."""
    if isinstance(x, torch.Tensor):
        kind, host_dtype, t = _Kind.TORCH_CPU, x.dtype, x
    else:
        kind = _Kind.DENSE if hasattr(x, "array") else _Kind.NUMPY
        arr = np.asarray(x.array if kind == _Kind.DENSE else x)
        host_dtype, t = arr.dtype, torch.from_numpy(np.ascontiguousarray(arr))
    if dtype is None:
        dtype = t.dtype if t.dtype in (torch.float16, torch.bfloat16, torch.float32) else torch.float32
    return t.to(dtype).contiguous(), kind, host_dtype


def _from_host(t: torch.Tensor, kind, host_dtype):
    if kind == _Kind.TORCH_CPU:
        return t if t.dtype == host_dtype else t.to(host_dtype)
    a = t.to(torch.float64).numpy()
    if kind == _Kind.DENSE:
        return HostArray(a)
    return a.astype(host_dtype, copy=False)


def _is_device(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def _from_device(t: torch.Tensor, kind, host_dtype):
    if kind == _Kind.CUDA:
        return t
    if kind == _Kind.TORCH_CPU:
        return t.to(device="cpu", dtype=host_dtype)
    a = t.to(device="cpu", dtype=torch.float64).numpy()
    if kind == _Kind.DENSE:
        return HostArray(a)
    return a.astype(host_dtype, copy=False)


def _check_qkv_2d(q, k, v):
    """flash.py:322-327."""
    qs, ks, vs = _shape_of(q), _shape_of(k), _shape_of(v)
    if len(qs) != 2:
        raise ShapeError(f"Q/K/V must be 2-D, got {qs}")
    if not (qs == ks == vs):
        raise ShapeError(f"Q/K/V shapes differ: {qs}, {ks}, {vs}")
    return qs


# ---- reference API --------------------------------------------------------------
def flash_forward(q, k, v, cfg: TileConfig, arena: ScratchpadArena, *, bias=None, mask=None,
                  kernel: str = "auto"):
    """Tiled attention forward for one (L, C) unit (flash.py:141-184).

    Returns (O, FlashContext, TrafficReport). The budget check (CapacityError)
    happens before any work, exactly as flash.py:156.
    """
    L, C = _check_qkv_2d(q, k, v)
    cfg.chunk_spans(C)
    need = peak_sram_forward(L, C, cfg)
    arena.check("forward", need)
    qd, kind, hdt = _to_device(q)
    kd, _, _ = _to_device(k, qd.dtype, qd.device)
    vd, _, _ = _to_device(v, qd.dtype, qd.device)
    shp = (1, 1, L, C)
    b = None if bias is None else bias.reshape(1, L, L)
    m = None if mask is None else mask.reshape(-1, L, L)
    o = ops.attention_forward(qd.view(shp), kd.view(shp), vd.view(shp), cfg.scale, b, m,
                              chunks=cfg.r, kernel=kernel)
    arena.record(need)
    report = forward_report(1, L, C, arena.peak_bytes)
    ctx = FlashContext(q=q, k=k, v=v, cfg=cfg, bias=bias, mask=mask,
                       mask_windows=0 if mask is None else int(m.shape[0]))
    return _from_device(o.view(L, C), kind, hdt), ctx, report


def flash_backward(ctx: FlashContext, dO, arena: ScratchpadArena, *, kernel: str = "auto"):
    """Backward for one unit: recompute P on chip, stream dQ/dK/dV out (flash.py:187-266)."""
    if not is_context(ctx):
        raise ContextError("backward requires the context returned by flash_forward")
    L, C = _check_qkv_2d(ctx.q, ctx.k, ctx.v)
    if _shape_of(dO) != (L, C):
        raise ShapeError(f"dO shape {_shape_of(dO)} does not match forward shape {(L, C)}")
    cfg = ctx.cfg
    cfg.chunk_spans(C)
    need = peak_sram_backward(L, C, cfg)
    arena.check("backward", need)
    dod, kind, hdt = _to_device(dO)
    qd, _, _ = _to_device(ctx.q, dod.dtype, dod.device)
    kd, _, _ = _to_device(ctx.k, dod.dtype, dod.device)
    vd, _, _ = _to_device(ctx.v, dod.dtype, dod.device)
    shp = (1, 1, L, C)
    b = None if ctx.bias is None else ctx.bias.reshape(1, L, L)
    m = None if ctx.mask is None else ctx.mask.reshape(-1, L, L)
    dq, dk, dv, _ = ops.attention_backward(qd.view(shp), kd.view(shp), vd.view(shp),
                                           dod.view(shp), cfg.scale, b, m, chunks=cfg.r,
                                           kernel=kernel)
    arena.record(need)
    report = backward_report(1, L, C, arena.peak_bytes)
    return (_from_device(dq.view(L, C), kind, hdt), _from_device(dk.view(L, C), kind, hdt),
            _from_device(dv.view(L, C), kind, hdt), report)


class BatchedContexts(Sequence):
    """contexts[b][head] -> FlashContext of that slice (flash.py:290, :304), built lazily.

    Holds the batched tensors once; ``batched_flash_backward`` consumes it
    directly without materialising B*h Python objects.
    """

    def __init__(self, q, k, v, cfg, bias=None, mask=None):
        self.q, self.k, self.v, self.cfg, self.bias, self.mask = q, k, v, cfg, bias, mask
        self.B, self.h = _shape_of(q)[:2]

    def __len__(self):
        return self.B

    @staticmethod
    def _slice(x, b, hd):
        """(L, C) slice of one (b, head) in the caller's container type.

        torch tensors and NumPy arrays are views; the reference's DenseTensor (and
        HostArray) have no ``__getitem__`` (tensor.py:26-71), so objects with an
        ``.array`` attribute are sliced through it and returned as a read-only
        HostArray view — which flash_backward accepts like any ``.array`` object.
        """
        if isinstance(x, torch.Tensor):
            return x[b, hd]
        if hasattr(x, "array"):
            return HostArray(np.asarray(x.array)[b, hd])
        return np.asarray(x)[b, hd]

    def __getitem__(self, b):
        if isinstance(b, slice):
            return [self[i] for i in range(*b.indices(self.B))]
        if not -self.B <= b < self.B:
            raise IndexError(b)
        b %= self.B
        # the forward's Swin extras follow the slice: bias[head] and mask[b % nW] (window b
        # of the batched call uses mask[b % nW]), so flash_backward on one slice
        # differentiates exactly the attention that batched_flash_forward ran
        mask = None if self.mask is None else self.mask[b % self.mask.shape[0]]
        return [FlashContext(q=self._slice(self.q, b, hd), k=self._slice(self.k, b, hd),
                             v=self._slice(self.v, b, hd), cfg=self.cfg,
                             bias=None if self.bias is None else self.bias[hd],
                             mask=mask, mask_windows=0 if mask is None else 1)
                for hd in range(self.h)]


def batched_flash_forward(q, k, v, cfg: TileConfig, arenas: Sequence[ScratchpadArena], *,
                          bias=None, mask=None, kernel: str = "auto"):
    """Forward over every (b, head) slice of (B, h, L, C) in ONE kernel launch (flash.py:269-319).

    Results are bitwise independent of len(arenas). Errors keep
    their class and gain the reference's ``slice (b=…, head=…)`` prefix.
    """
    qs, ks, vs = _shape_of(q), _shape_of(k), _shape_of(v)
    if len(qs) != 4 or not (qs == ks == vs):
        raise ShapeError(f"batched Q/K/V must share a 4-D shape, got {qs}, {ks}, {vs}")
    if not arenas:
        raise InvalidRangeError("at least one arena is required")
    B, h, L, C = qs
    try:
        cfg.chunk_spans(C)
        need = peak_sram_forward(L, C, cfg)
        arenas[0].check("forward", need)
    except FlashwinError as exc:
        raise type(exc)(f"slice (b=0, head=0): {exc}") from exc
    if _is_device(q):
        qd, kind, hdt = _to_device(q)
        kd, _, _ = _to_device(k, qd.dtype, qd.device)
        vd, _, _ = _to_device(v, qd.dtype, qd.device)
        o = ops.attention_forward(qd, kd, vd, cfg.scale, bias, mask, chunks=cfg.r, kernel=kernel)
        result = _from_device(o, kind, hdt)
    else:
        # host buffers: chunked H2D / kernel / D2H overlap (pipeline.py)
        qh, kind, hdt = _to_host_tensor(q)
        kh, _, _ = _to_host_tensor(k, qh.dtype)
        vh, _, _ = _to_host_tensor(v, qh.dtype)
        result = _from_host(host_forward(qh, kh, vh, cfg.scale, bias, mask, cfg.r, kernel),
                            kind, hdt)
    for a in arenas[: min(len(arenas), B * h)]:
        a.record(need)
    report = forward_report(B * h, L, C, max(a.peak_bytes for a in arenas[: min(len(arenas), B * h)]))
    ctxs = BatchedContexts(q, k, v, cfg, bias, mask)
    return result, ctxs, report


def batched_flash_backward(contexts: BatchedContexts, dO, arenas: Sequence[ScratchpadArena], *,
                           kernel: str = "auto", want_dbias: bool = False):
    """Backward over the whole (B, h, L, C) stack in one launch (not in the reference).

    Returns (dQ, dK, dV, TrafficReport) or, with want_dbias, (dQ, dK, dV, dBias, report).
    """
    if not isinstance(contexts, BatchedContexts):
        raise ContextError("batched backward requires the contexts of batched_flash_forward")
    B, h, L, C = _shape_of(contexts.q)
    if _shape_of(dO) != (B, h, L, C):
        raise ShapeError(f"dO shape {_shape_of(dO)} does not match forward shape {(B, h, L, C)}")
    if not arenas:
        raise InvalidRangeError("at least one arena is required")
    cfg = contexts.cfg
    try:
        cfg.chunk_spans(C)
        need = peak_sram_backward(L, C, cfg)
        arenas[0].check("backward", need)
    except FlashwinError as exc:
        raise type(exc)(f"slice (b=0, head=0): {exc}") from exc
    if _is_device(dO):
        dod, kind, hdt = _to_device(dO)
        qd, _, _ = _to_device(contexts.q, dod.dtype, dod.device)
        kd, _, _ = _to_device(contexts.k, dod.dtype, dod.device)
        vd, _, _ = _to_device(contexts.v, dod.dtype, dod.device)
        dq, dk, dv, db = ops.attention_backward(qd, kd, vd, dod, cfg.scale, contexts.bias,
                                                contexts.mask, chunks=cfg.r, kernel=kernel,
                                                want_dbias=want_dbias)
        out = [_from_device(t, kind, hdt) for t in (dq, dk, dv)]
    else:
        doh, kind, hdt = _to_host_tensor(dO)
        qh, kh, vh = (_to_host_tensor(t, doh.dtype)[0] for t in (contexts.q, contexts.k, contexts.v))
        dq, dk, dv, db = host_backward(qh, kh, vh, doh, cfg.scale, contexts.bias, contexts.mask,
                                       cfg.r, kernel, want_dbias)
        out = [_from_host(t, kind, hdt) for t in (dq, dk, dv)]
    for a in arenas[: min(len(arenas), B * h)]:
        a.record(need)
    report = backward_report(B * h, L, C, max(a.peak_bytes for a in arenas[: min(len(arenas), B * h)]))
    if want_dbias:
        out.append(db)
    return (*out, report)


__all__ = [
    "BatchedContexts",
    "CapacityError",
    "HostArray",
    "TrafficReport",
    "batched_flash_backward",
    "batched_flash_forward",
    "flash_backward",
    "flash_forward",
]
