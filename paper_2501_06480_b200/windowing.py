"""Window partition / reverse (pkg/src/flashwin/windowing.py:17-70) on device.

``WindowConfig`` validates exactly like the reference. ``window_partition`` /
``window_reverse`` accept the reference's single image (H, W, C) or a batch
(B, H, W, C), torch CUDA tensors (zero-copy) or host arrays (copied), and an
optional Swin cyclic ``shift`` (extension). The device kernel moves bytes, so
the round trip is bitwise.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import PartitionError, ShapeError


@dataclass(frozen=True)
class WindowConfig:
    """Image/window geometry: H x W pixels, C channels, k x k windows (windowing.py:17-41)."""

    H: int
    W: int
    C: int
    k: int

    def __post_init__(self):
        for name in ("H", "W", "C", "k"):
            if getattr(self, name) < 1:
                raise ShapeError(f"{name} must be >= 1, got {getattr(self, name)}")
        if self.H % self.k or self.W % self.k:
            raise PartitionError(f"window size {self.k} must divide image {self.H}x{self.W}")

    @property
    def num_windows(self) -> int:
        return (self.H * self.W) // (self.k * self.k)

    @property
    def seq_len(self) -> int:
        return self.k * self.k


def _dev(x):
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            return x.contiguous(), None
        return x.cuda().contiguous(), ("torch", x.dtype)
    arr = np.asarray(x.array if hasattr(x, "array") else x)
    kind = "dense" if hasattr(x, "array") else "numpy"
    return torch.from_numpy(np.ascontiguousarray(arr)).cuda(), (kind, arr.dtype)


def _back(t, how):
    if how is None:
        return t
    kind, dt = how
    if kind == "torch":
        return t.cpu()
    a = t.cpu().numpy()
    if kind == "dense":
        from .api import HostArray
        return HostArray(a)
    return a


def window_partition(x, cfg: WindowConfig, shift: int = 0):
    """(H,W,C) -> (N,L,C) or (B,H,W,C) -> (B*N,L,C) (windowing.py:44-54)."""
    t, how = _dev(x)
    if tuple(t.shape[-3:]) != (cfg.H, cfg.W, cfg.C) or t.dim() not in (3, 4):
        raise ShapeError(f"expected image shape {(cfg.H, cfg.W, cfg.C)}, got {tuple(t.shape)}")
    single = t.dim() == 3
    y = ops.window_partition(t.unsqueeze(0) if single else t, cfg.k, shift)
    return _back(y, how)


def window_reverse(y, cfg: WindowConfig, shift: int = 0):
    """Inverse of window_partition (windowing.py:57-70); a stack of N*B windows gives (B,H,W,C)."""
    t, how = _dev(y)
    if t.dim() != 3 or t.shape[1:] != (cfg.seq_len, cfg.C) or t.shape[0] % cfg.num_windows:
        raise ShapeError(
            f"expected window stack shape {(cfg.num_windows, cfg.seq_len, cfg.C)}, got {tuple(t.shape)}")
    single = t.shape[0] == cfg.num_windows
    x = ops.window_reverse(t, cfg.k, cfg.H, cfg.W, shift)
    return _back(x[0] if single else x, how)
