"""Swin (S)W-MSA block on this package's kernels.

The reference package stops at the attention call (pkg/src/flashwin/flash.py:269-319) and
its window partition (windowing.py:44-70); the paper's end-to-end claim ("at least 10 %
... end-to-end speedup") is about the Swin block around it. This module
is that block, with every glue step on the device kernels:

  x (B, H, W, C) --roll(-s) + partition (one kernel)--> (B*nW, L, C)
    --qkv Linear (cuBLAS)--> (N, L, 3C), read in place by the attention kernel
    --window attention + relative-position bias + shifted-window mask--> (N, L, C) written
      straight in the proj-Linear layout (no permute copies either side)
    --proj Linear (cuBLAS)--> --reverse + roll(+s) (one kernel)--> (B, H, W, C)

``TorchSwinWindowAttention`` is the same block written the usual way in PyTorch (roll,
view/permute partition, q @ k^T + bias + mask, softmax, @ v, permutes, reverse); it shares
weights with the fused block and is the baseline bench.py times it against.
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import ops
from .autograd import partition_windows, relative_position_bias, reverse_windows, window_attention_qkv


def relative_position_index(k: int) -> torch.Tensor:
    """(L, L) index into the ((2k-1)^2, h) table (Swin's definition)."""
    c = np.stack(np.meshgrid(np.arange(k), np.arange(k), indexing="ij")).reshape(2, -1)
    rel = (c[:, :, None] - c[:, None, :]).transpose(1, 2, 0) + (k - 1)
    return torch.from_numpy((rel[..., 0] * (2 * k - 1) + rel[..., 1]).astype(np.int64))


class SwinWindowAttention(torch.nn.Module):
    """(S)W-MSA: window attention over (B, H, W, C) with Swin's relative-position bias and,
    for shift > 0, the cyclic shift and its mask. Runs in the parameters' dtype (f16/bf16)."""

    def __init__(self, dim: int, heads: int, window: int, shift: int = 0,
                 dtype: torch.dtype = torch.bfloat16, device="cuda"):
        super().__init__()
        if dim % heads:
            raise ValueError(f"dim {dim} is not a multiple of heads {heads}")
        self.dim, self.heads, self.window, self.shift = dim, heads, window, shift
        self.qkv = torch.nn.Linear(dim, 3 * dim, device=device, dtype=dtype)
        self.proj = torch.nn.Linear(dim, dim, device=device, dtype=dtype)
        self.table = torch.nn.Parameter(
            torch.nn.init.trunc_normal_(torch.empty((2 * window - 1) ** 2, heads, device=device),
                                        std=0.02))
        self._masks = {}

    def mask(self, H: int, W: int) -> Optional[torch.Tensor]:
        if not self.shift:
            return None
        key = (H, W)
        if key not in self._masks:
            self._masks[key] = ops.shift_mask(H, W, self.window, self.shift,
                                              device=self.table.device)
        return self._masks[key]

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        B, H, W, C = x.shape
        k = self.window
        xw = partition_windows(x, k, self.shift)
        qkv = self.qkv(xw)
        bias = relative_position_bias(self.table, k)
        o = window_attention_qkv(qkv, self.heads, None, bias, self.mask(H, W))
        return reverse_windows(self.proj(o), k, H, W, self.shift)


class TorchSwinWindowAttention(torch.nn.Module):
    """The same block in plain PyTorch ops (the usual Swin implementation), sharing weights
    with a SwinWindowAttention: the end-to-end baseline."""

    def __init__(self, fused: SwinWindowAttention):
        super().__init__()
        self.f = fused
        self.register_buffer("rpi", relative_position_index(fused.window).to(fused.table.device),
                             persistent=False)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        f = self.f
        B, H, W, C = x.shape
        k, s, h = f.window, f.shift, f.heads
        if s:
            x = torch.roll(x, (-s, -s), (1, 2))
        xw = x.view(B, H // k, k, W // k, k, C).permute(0, 1, 3, 2, 4, 5).reshape(-1, k * k, C)
        N, L, _ = xw.shape
        qkv = f.qkv(xw).view(N, L, 3, h, C // h).permute(2, 0, 3, 1, 4)
        q, kk, v = qkv[0], qkv[1], qkv[2]
        bias = f.table[self.rpi.view(-1)].view(L, L, h).permute(2, 0, 1)
        a = (q @ kk.transpose(-1, -2)) * (C // h) ** -0.5 + bias[None].to(q.dtype)
        m = f.mask(H, W)
        if m is not None:
            nW = m.shape[0]
            a = (a.view(N // nW, nW, h, L, L) + m[None, :, None].to(a.dtype)).view(N, h, L, L)
        o = (torch.softmax(a, -1) @ v).transpose(1, 2).reshape(N, L, C)
        y = f.proj(o).view(B, H // k, W // k, k, k, C).permute(0, 1, 3, 2, 4, 5).reshape(B, H, W, C)
        if s:
            y = torch.roll(y, (s, s), (1, 2))
        return y


def time_block_fwd_bwd(block: torch.nn.Module, x: torch.Tensor, reps: int = 20,
                       warmup: int = 3) -> float:
    """Average device ms of forward + backward (loss = sum(y * g)) over `reps` eager steps."""
    g = torch.randn_like(x)
    xr = x.detach().requires_grad_(True)

    def step():
        y = block(xr)
        y.backward(g)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def block_speedup(B: int, H: int, C: int, heads: int, window: int, shift: int,
                  dtype=torch.bfloat16, reps: int = 20) -> dict:
    """Fused vs plain-PyTorch block, fwd + bwd, same weights and input (B, H, H, C)."""
    torch.manual_seed(0)
    fused = SwinWindowAttention(C, heads, window, shift, dtype=dtype)
    base = TorchSwinWindowAttention(fused)
    x = torch.randn(B, H, H, C, device="cuda", dtype=dtype)
    t_fused = time_block_fwd_bwd(fused, x, reps)
    t_base = time_block_fwd_bwd(base, x, reps)
    return {"B": B, "H": H, "C": C, "heads": heads, "window": window, "shift": shift,
            "dtype": str(dtype).replace("torch.", ""), "torch_ms": t_base, "fwa_ms": t_fused,
            "speedup": t_base / t_fused, "L": window * window,
            "windows": B * (H // window) ** 2}


__all__ = ["SwinWindowAttention", "TorchSwinWindowAttention", "block_speedup",
           "relative_position_index", "time_block_fwd_bwd"]
