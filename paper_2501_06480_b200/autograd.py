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
        o = ops.attention_forward(q, k, v, scale, bias, mask, kernel=kernel)
        ctx.save_for_backward(q, k, v, bias, mask)
        ctx.scale = scale
        ctx.kernel = kernel
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, bias, mask = ctx.saved_tensors
        want_db = bias is not None and ctx.needs_input_grad[3]
        dq, dk, dv, db = ops.attention_backward(q, k, v, do.contiguous(), ctx.scale, bias, mask,
                                                kernel=ctx.kernel, want_dbias=want_db)
        return dq, dk, dv, db, None, None, None


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


def relative_position_bias(table: torch.Tensor, k: int) -> torch.Tensor:
    return RelativePositionBias.apply(table, k)
