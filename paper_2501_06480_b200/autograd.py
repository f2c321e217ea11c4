"""torch.autograd binding: the FlashContext analogue is ctx.save_for_backward(q, k, v[, bias, mask]).

Nothing else is saved (no P, O or log-sum-exp; flash.py:74-81):
the backward kernel recomputes P on chip.
"""

from __future__ import annotations

import math
from typing import Optional

import torch

from . import ops


class WindowAttentionFunction(torch.autograd.Function):
    """O = softmax(scale*QK^T + bias[h] + mask[n % nW]) V over (N, h, L, d)."""

    @staticmethod
    def forward(ctx, q, k, v, bias, mask, scale, kernel):
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        # large windows: the (bias + mask) score table is built once per layer call and
        # shared by this forward and its backward (None for L <= 64 / no bias or mask)
        table = ops.build_add_table(*q.shape, q.dtype, bias, mask, kernel=kernel)
        o = ops.attention_forward(q, k, v, scale, bias, mask, kernel=kernel, add_table=table)
        ctx.save_for_backward(q, k, v, bias, mask, table)
        ctx.scale = scale
        ctx.kernel = kernel
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, bias, mask, table = ctx.saved_tensors
        want_db = bias is not None and ctx.needs_input_grad[3]
        dq, dk, dv, db = ops.attention_backward(q, k, v, do.contiguous(), ctx.scale, bias, mask,
                                                kernel=ctx.kernel, want_dbias=want_db,
                                                add_table=table)
        return dq, dk, dv, db, None, None, None


class WindowAttentionQKVFunction(torch.autograd.Function):
    """Fused-layout variant: (N, L, 3*h*d) qkv-Linear output -> (N, L, h*d) proj input."""

    @staticmethod
    def forward(ctx, qkv, bias, mask, heads, scale, kernel):
        qkv = qkv.contiguous()
        N, L = qkv.shape[0], qkv.shape[1]
        d = qkv.shape[-1] // (3 * heads) if qkv.dim() == 3 else qkv.shape[-1]
        table = ops.build_add_table(N, heads, L, d, qkv.dtype, bias, mask, kernel=kernel)
        o = ops.attention_forward_qkv(qkv, heads, scale, bias, mask, kernel=kernel, add_table=table)
        ctx.save_for_backward(qkv, bias, mask, table)
        ctx.heads, ctx.scale, ctx.kernel = heads, scale, kernel
        return o

    @staticmethod
    def backward(ctx, do):
        qkv, bias, mask, table = ctx.saved_tensors
        want_db = bias is not None and ctx.needs_input_grad[1]
        dqkv, db = ops.attention_backward_qkv(qkv, do.contiguous(), ctx.heads, ctx.scale, bias,
                                              mask, kernel=ctx.kernel, want_dbias=want_db,
                                              add_table=table)
        return dqkv, db, None, None, None, None


class WindowPartitionFunction(torch.autograd.Function):
    """(B,H,W,C) -> (B*nW, k*k, C) with Swin's cyclic shift; the adjoint of a permutation
    is its inverse, so the backward is the device window_reverse (and vice versa)."""

    @staticmethod
    def forward(ctx, x, k, shift):
        ctx.k, ctx.shift, ctx.hw = k, shift, (x.shape[1], x.shape[2])
        return ops.window_partition(x.contiguous(), k, shift)

    @staticmethod
    def backward(ctx, gy):
        return ops.window_reverse(gy.contiguous(), ctx.k, *ctx.hw, ctx.shift), None, None


class WindowReverseFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, y, k, H, W, shift):
        ctx.k, ctx.shift = k, shift
        return ops.window_reverse(y.contiguous(), k, H, W, shift)

    @staticmethod
    def backward(ctx, gx):
        return ops.window_partition(gx.contiguous(), ctx.k, ctx.shift), None, None, None, None


def partition_windows(x: torch.Tensor, k: int, shift: int = 0) -> torch.Tensor:
    """Differentiable device window partition (+ cyclic shift)."""
    return WindowPartitionFunction.apply(x, k, shift)


def reverse_windows(y: torch.Tensor, k: int, H: int, W: int, shift: int = 0) -> torch.Tensor:
    """Differentiable device window reverse (+ inverse cyclic shift)."""
    return WindowReverseFunction.apply(y, k, H, W, shift)


class RelativePositionBias(torch.autograd.Function):
    """Swin table ((2k-1)^2, h) -> bias (h, L, L); backward is a deterministic scatter-add."""

    @staticmethod
    def forward(ctx, table, k):
        ctx.k = k
        return ops.bias_gather(table, k)

    @staticmethod
    def backward(ctx, dbias):
        return ops.bias_scatter(dbias, ctx.k), None


def window_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                     scale: Optional[float] = None, bias: Optional[torch.Tensor] = None,
                     mask: Optional[torch.Tensor] = None, kernel: str = "auto") -> torch.Tensor:
    """Differentiable window attention on (N, h, L, d) CUDA tensors (scale defaults to d^-1/2)."""
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[-1])
    return WindowAttentionFunction.apply(q, k, v, bias, mask, float(scale), kernel)


def window_attention_qkv(qkv: torch.Tensor, heads: int, scale: Optional[float] = None,
                         bias: Optional[torch.Tensor] = None, mask: Optional[torch.Tensor] = None,
                         kernel: str = "auto") -> torch.Tensor:
    """Swin window attention straight from the qkv-Linear output (N, L, 3*h*d) to the
    proj-Linear input (N, L, h*d), differentiable (dqkv, dBias)."""
    d = qkv.shape[-1] // (3 * heads) if qkv.dim() == 3 else qkv.shape[-1]
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    return WindowAttentionQKVFunction.apply(qkv, bias, mask, heads, float(scale), kernel)


def relative_position_bias(table: torch.Tensor, k: int) -> torch.Tensor:
    return RelativePositionBias.apply(table, k)
