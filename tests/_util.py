"""Shared helpers for the GPU parity tests: identical inputs on device and in the oracle."""

from __future__ import annotations

import numpy as np
import torch

from oracle import flashwin_oracle as orc

TOL_F32_REL = 1e-5   # north star: fp32 within 1e-5 relative (max|err| / max|oracle|)
TOL_LOWP_ABS = 2e-2  # north star: fp16/bf16 within 2e-2 of the fp64 oracle on the same inputs

DTYPES = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}


def quantize(a: np.ndarray, dtype: torch.dtype) -> np.ndarray:
    """f64 -> f32 -> dtype -> f64: the device fill's rounding chain (include/fwa.h)."""
    return torch.from_numpy(np.asarray(a)).to(torch.float32).to(dtype).to(torch.float64).numpy()


def draw(seed: int, shape, n: int, dtype: torch.dtype, device="cuda"):
    """n successive fill_uniform draws of Rng(seed): device tensors + quantised f64 copies."""
    from paper_2501_06480_b200 import Rng, fill_uniform

    rng = Rng(seed)
    dev = [fill_uniform(rng, shape, -1.0, 1.0, dtype=dtype, device=device) for _ in range(n)]
    host = [quantize(a, dtype) for a in orc.draw_qkvdo(seed, shape, n)]
    return dev, host


def err_ok(got: torch.Tensor, ref: np.ndarray, dtype: torch.dtype):
    g = got.detach().to(torch.float64).cpu().numpy()
    err = float(np.abs(g - ref).max()) if ref.size else 0.0
    if dtype == torch.float32:
        scale = max(float(np.abs(ref).max()), 1e-30)
        return err / scale <= TOL_F32_REL, err / scale
    return err <= TOL_LOWP_ABS, err
