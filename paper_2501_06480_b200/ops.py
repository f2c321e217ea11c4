"""Device-level window-attention ops on torch CUDA tensors, through the C-ABI.

Layouts (include/fwa.h): q, k, v, o, dO, dq, dk, dv are contiguous
[N_windows][heads][L][d] in float32 / float16 / bfloat16 on one CUDA device;
bias is float32 [heads][L][L]; mask is float32 [nW][L][L] and window n uses
mask[n % nW]. All launches go on torch's current stream. PyTorch is only the
allocator and stream provider here; the math runs in libfwa.so.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import torch

from . import _native as nat
from .errors import InvalidRangeError, ShapeError

_DTYPES = {torch.float32: nat.FWA_F32, torch.float16: nat.FWA_F16, torch.bfloat16: nat.FWA_BF16}
_KERNELS = {"auto": nat.KERNEL_AUTO, "generic": nat.KERNEL_GENERIC, "tc": nat.KERNEL_TC}


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def dtype_id(dtype: torch.dtype) -> int:
    try:
        return _DTYPES[dtype]
    except KeyError:
        raise InvalidRangeError(f"dtype {dtype} not supported (float32, float16, bfloat16)") from None


def make_desc(N, h, L, d, dtype, scale=1.0, chunks=1, mask_windows=0, kernel="auto",
              add_table: Optional[torch.Tensor] = None) -> nat.FwaDesc:
    if kernel not in _KERNELS:
        raise InvalidRangeError(f"kernel must be one of {sorted(_KERNELS)}, got {kernel!r}")
    return nat.FwaDesc(
        num_windows=int(N), heads=int(h), seq_len=int(L), head_dim=int(d),
        dtype=dtype_id(dtype) if isinstance(dtype, torch.dtype) else int(dtype),
        scale=float(scale), chunks=int(chunks), mask_windows=int(mask_windows),
        kernel=_KERNELS[kernel], reserved=0,
        add_table=None if add_table is None else add_table.data_ptr(),
    )


def _workspace(nbytes: int, device) -> Optional[torch.Tensor]:
    """Caller-owned scratch for the C-ABI (the library never allocates device memory)."""
    return torch.empty(nbytes, dtype=torch.uint8, device=device) if nbytes else None


def build_add_table(N, h, L, d, dtype, bias=None, mask=None, kernel: str = "auto",
                    device=None) -> Optional[torch.Tensor]:
    """The large-window kernels' (bias + mask) * log2e f16 table, built once so a layer's
    forward and backward share it (``add_table=`` of attention_forward/backward).
    None when no kernel of this shape reads a table (L <= 64, no bias/mask)."""
    if bias is None and mask is None:
        return None
    ref = bias if bias is not None else mask
    device = ref.device if device is None else device
    mw = _check_bias_mask((N, h, L, d), device, bias, mask)
    desc = make_desc(N, h, L, d, dtype, 1.0, 1, mw, kernel)
    lib = nat.load()
    nbytes = int(lib.fwa_add_table_bytes(ctypes.byref(desc), int(bias is not None),
                                         int(mask is not None)))
    if not nbytes:
        return None
    table = torch.empty(nbytes, dtype=torch.uint8, device=device)
    with torch.cuda.device(device):
        st = lib.fwa_build_add_table(ctypes.byref(desc), _ptr(bias), _ptr(mask), _ptr(table),
                                     ctypes.c_size_t(nbytes), _stream(device))
    nat.check(st)
    return table


def _check_qkv(q, k, v, *more):
    for t in (q, k, v) + more:
        if not isinstance(t, torch.Tensor):
            raise ShapeError(f"expected torch.Tensor, got {type(t).__name__}")
        if not t.is_cuda:
            raise ShapeError("device op needs CUDA tensors (use the api module for host arrays)")
    if q.dim() != 4:
        raise ShapeError(f"Q/K/V must be 4-D (N, h, L, d), got {tuple(q.shape)}")
    for t in (k, v) + more:
        if t.shape != q.shape:
            raise ShapeError(f"Q/K/V shapes differ: {tuple(q.shape)}, {tuple(t.shape)}")
        if t.dtype != q.dtype:
            raise ShapeError(f"Q/K/V dtypes differ: {q.dtype}, {t.dtype}")
        if t.device != q.device:
            raise ShapeError("Q/K/V live on different devices")
    for t in (q, k, v) + more:
        if not t.is_contiguous():
            raise ShapeError("Q/K/V must be contiguous (N, h, L, d)")
    dtype_id(q.dtype)
    return q.shape


def _check_bias_mask(shape, device, bias, mask):
    N, h, L, _ = shape
    mw = 0
    if bias is not None:
        if bias.dtype != torch.float32 or tuple(bias.shape) != (h, L, L) or not bias.is_contiguous():
            raise ShapeError(f"bias must be contiguous float32 (h, L, L) = {(h, L, L)}, "
                             f"got {bias.dtype} {tuple(bias.shape)}")
        if bias.device != device:
            raise ShapeError("bias lives on another device")
    if mask is not None:
        if mask.dtype != torch.float32 or mask.dim() != 3 or tuple(mask.shape[1:]) != (L, L) \
                or not mask.is_contiguous():
            raise ShapeError(f"mask must be contiguous float32 (nW, L, L), got {mask.dtype} "
                             f"{tuple(mask.shape)}")
        if mask.device != device:
            raise ShapeError("mask lives on another device")
        mw = mask.shape[0]
    return mw


def attention_forward(q, k, v, scale: float = 1.0, bias=None, mask=None, chunks: int = 1,
                      kernel: str = "auto", out: Optional[torch.Tensor] = None,
                      add_table: Optional[torch.Tensor] = None) -> torch.Tensor:
    """O = softmax(scale*QK^T + bias[h] + mask[n % nW]) V for every (window, head) unit.

    ``add_table``: a build_add_table() result for this bias/mask (skips the per-call build).
    """
    N, h, L, d = _check_qkv(q, k, v)
    mw = _check_bias_mask(q.shape, q.device, bias, mask)
    desc = make_desc(N, h, L, d, q.dtype, scale, chunks, mw, kernel, add_table)
    if out is None:
        out = torch.empty_like(q)
    elif out.shape != q.shape or out.dtype != q.dtype or not out.is_contiguous():
        raise ShapeError("out must match q's shape/dtype and be contiguous")
    lib = nat.load()
    ws_bytes = int(lib.fwa_fwd_workspace_bytes(ctypes.byref(desc), int(bias is not None),
                                               int(mask is not None)))
    ws = _workspace(ws_bytes, q.device)
    with torch.cuda.device(q.device):
        st = lib.fwa_fwd(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(bias), _ptr(mask),
                         _ptr(out), _ptr(ws), ctypes.c_size_t(ws_bytes), _stream(q.device))
    nat.check(st)
    return out


def attention_backward(q, k, v, do, scale: float = 1.0, bias=None, mask=None, chunks: int = 1,
                       kernel: str = "auto", want_dbias: bool = False,
                       add_table: Optional[torch.Tensor] = None):
    """(dQ, dK, dV, dBias-or-None); P is recomputed on chip, nothing else is saved."""
    N, h, L, d = _check_qkv(q, k, v, do)
    mw = _check_bias_mask(q.shape, q.device, bias, mask)
    if want_dbias and bias is None:
        raise ShapeError("dBias needs the bias the forward used")
    desc = make_desc(N, h, L, d, q.dtype, scale, chunks, mw, kernel, add_table)
    lib = nat.load()
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    dbias = torch.empty((h, L, L), dtype=torch.float32, device=q.device) if want_dbias else None
    ws_bytes = int(lib.fwa_bwd_workspace_bytes(ctypes.byref(desc), int(bias is not None),
                                               int(mask is not None), int(want_dbias)))
    ws = _workspace(ws_bytes, q.device)
    with torch.cuda.device(q.device):
        st = lib.fwa_bwd(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(do), _ptr(bias),
                         _ptr(mask), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dbias), _ptr(ws),
                         ctypes.c_size_t(ws_bytes), _stream(q.device))
    nat.check(st)
    return dq, dk, dv, dbias


def footprint(N, h, L, d, dtype=torch.float16, chunks=1, kernel="auto") -> dict:
    """Which kernel runs and its real SMEM/TMEM, next to the paper's closed forms."""
    desc = make_desc(N, h, L, d, dtype, 1.0, chunks, 0, kernel)
    fp = nat.FwaFootprint()
    nat.check(nat.load().fwa_footprint(ctypes.byref(desc), ctypes.byref(fp)))
    names = {nat.KERNEL_GENERIC: "generic", nat.KERNEL_TC: "tc"}
    return {
        "kernel_fwd": names.get(fp.kernel_fwd, "?"), "kernel_bwd": names.get(fp.kernel_bwd, "?"),
        "smem_bytes_fwd": fp.smem_bytes_fwd, "smem_bytes_bwd": fp.smem_bytes_bwd,
        "tmem_cols_fwd": fp.tmem_cols_fwd, "tmem_cols_bwd": fp.tmem_cols_bwd,
        "paper_peak_fwd": fp.paper_peak_fwd, "paper_peak_bwd": fp.paper_peak_bwd,
        "hbm_bytes_fwd": fp.hbm_bytes_fwd, "hbm_bytes_bwd": fp.hbm_bytes_bwd,
    }


# ---- windowing / Swin helpers ------------------------------------------------
def window_partition(x: torch.Tensor, k: int, shift: int = 0) -> torch.Tensor:
    """(B,H,W,C) -> (B*nW, k*k, C) on device; bitwise copy (+ Swin roll by -shift)."""
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dim() == 4 and x.is_contiguous()):
        raise ShapeError("window_partition needs a contiguous CUDA (B, H, W, C) tensor")
    B, H, W, C = x.shape
    desc = nat.FwaWinDesc(batch=B, height=H, width=W, channels=C, window=int(k), shift=int(shift),
                          elem_bytes=x.element_size())
    if H % max(k, 1) or W % max(k, 1):
        out = x.new_empty(1)  # C-ABI raises PartitionError below
    else:
        out = x.new_empty((B * (H // k) * (W // k), k * k, C))
    with torch.cuda.device(x.device):
        st = nat.load().fwa_window_partition(ctypes.byref(desc), _ptr(x), _ptr(out),
                                             _stream(x.device))
    nat.check(st)
    return out


def window_reverse(y: torch.Tensor, k: int, H: int, W: int, shift: int = 0) -> torch.Tensor:
    """(B*nW, k*k, C) -> (B,H,W,C) on device (then roll by +shift)."""
    if not (isinstance(y, torch.Tensor) and y.is_cuda and y.dim() == 3 and y.is_contiguous()):
        raise ShapeError("window_reverse needs a contiguous CUDA (N, L, C) tensor")
    if H % k or W % k:
        from .errors import PartitionError
        raise PartitionError(f"window size {k} must divide image {H}x{W}")
    nW = (H // k) * (W // k)
    N, L, C = y.shape
    if L != k * k or N % nW:
        raise ShapeError(f"window stack {tuple(y.shape)} does not match k={k}, image {H}x{W}")
    B = N // nW
    desc = nat.FwaWinDesc(batch=B, height=H, width=W, channels=C, window=int(k), shift=int(shift),
                          elem_bytes=y.element_size())
    out = y.new_empty((B, H, W, C))
    with torch.cuda.device(y.device):
        st = nat.load().fwa_window_reverse(ctypes.byref(desc), _ptr(y), _ptr(out), _stream(y.device))
    nat.check(st)
    return out


def bias_gather(table: torch.Tensor, k: int) -> torch.Tensor:
    """Swin relative-position table ((2k-1)^2, h) float32 -> bias (h, L, L)."""
    T = (2 * k - 1) ** 2
    if table.dtype != torch.float32 or table.dim() != 2 or table.shape[0] != T or not table.is_cuda:
        raise ShapeError(f"table must be CUDA float32 ({T}, heads)")
    table = table.contiguous()
    h = table.shape[1]
    out = torch.empty((h, k * k, k * k), dtype=torch.float32, device=table.device)
    with torch.cuda.device(table.device):
        st = nat.load().fwa_bias_gather(_ptr(table), k, h, _ptr(out), _stream(table.device))
    nat.check(st)
    return out


def bias_scatter(dbias: torch.Tensor, k: int) -> torch.Tensor:
    """dBias (h, L, L) -> dTable ((2k-1)^2, h), deterministic fixed-order sums."""
    dbias = dbias.contiguous()
    h = dbias.shape[0]
    out = torch.empty(((2 * k - 1) ** 2, h), dtype=torch.float32, device=dbias.device)
    with torch.cuda.device(dbias.device):
        st = nat.load().fwa_bias_scatter(_ptr(dbias), k, h, _ptr(out), _stream(dbias.device))
    nat.check(st)
    return out


def shift_mask(H: int, W: int, k: int, shift: int, neg: float = -100.0, device="cuda") -> torch.Tensor:
    """Swin shifted-window mask (nW, L, L) float32 built on device."""
    nW = (H // k) * (W // k) if (k and H % k == 0 and W % k == 0) else 1
    out = torch.empty((nW, k * k, k * k), dtype=torch.float32, device=device)
    with torch.cuda.device(out.device):
        st = nat.load().fwa_shift_mask(H, W, k, shift, neg, _ptr(out), _stream(out.device))
    nat.check(st)
    return out


def fill_uniform_(out: torch.Tensor, state: int, lo: float = -1.0, hi: float = 1.0) -> torch.Tensor:
    """In-place SplitMix64 fill (tensor.py:118-138): f64 draw -> f32 -> out.dtype."""
    if not (out.is_cuda and out.is_contiguous()):
        raise ShapeError("fill_uniform_ needs a contiguous CUDA tensor")
    with torch.cuda.device(out.device):
        st = nat.load().fwa_fill_uniform(ctypes.c_uint64(state & ((1 << 64) - 1)), out.numel(),
                                         float(lo), float(hi), dtype_id(out.dtype), _ptr(out),
                                         _stream(out.device))
    nat.check(st)
    return out


# ---- fused Swin layouts (qkv-Linear output in, proj-Linear input out) -------------
def _qkv_view(qkv: torch.Tensor, heads: int):
    if qkv.dim() == 3:
        N, L, C3 = qkv.shape
        if C3 % (3 * heads):
            raise ShapeError(f"qkv last dim {C3} is not 3*heads*d for heads={heads}")
        qkv = qkv.view(N, L, 3, heads, C3 // (3 * heads))
    if qkv.dim() != 5 or qkv.shape[2] != 3 or qkv.shape[3] != heads:
        raise ShapeError(f"qkv must be (N, L, 3, heads, d) or (N, L, 3*heads*d), got {tuple(qkv.shape)}")
    if not (qkv.is_cuda and qkv.is_contiguous()):
        raise ShapeError("qkv must be a contiguous CUDA tensor")
    return qkv


def _split_qkv(qkv5):
    """Device-side permute (fallback for shapes without the fused kernel)."""
    q, k, v = (qkv5[:, :, i].permute(0, 2, 1, 3).contiguous() for i in range(3))
    return q, k, v


def attention_forward_qkv(qkv: torch.Tensor, heads: int, scale: float = 1.0, bias=None, mask=None,
                          kernel: str = "auto", add_table: Optional[torch.Tensor] = None
                          ) -> torch.Tensor:
    """O (N, L, heads*d) from the packed qkv (N, L, 3*heads*d): Swin's qkv -> attn -> proj glue.

    The tcgen05 kernels read Q/K/V in place and write O in the proj layout (no permutes):
    the tile kernel for L <= 64, the flat-row kernel in pieces mode for Swin-B's L = 144
    (and 128/192/256) at d = 32. Other shapes go through device permutes + attention_forward.
    """
    qkv5 = _qkv_view(qkv, heads)
    N, L, _, h, d = qkv5.shape
    mw = _check_bias_mask((N, h, L, d), qkv.device, bias, mask)
    o = torch.empty((N, L, h * d), dtype=qkv.dtype, device=qkv.device)
    if kernel != "generic" and qkv.dtype in (torch.float16, torch.bfloat16):
        desc = make_desc(N, h, L, d, qkv.dtype, scale, 1, mw, kernel, add_table)
        lib = nat.load()
        ws_bytes = int(lib.fwa_fwd_workspace_bytes(ctypes.byref(desc), int(bias is not None),
                                                   int(mask is not None)))
        ws = _workspace(ws_bytes, qkv.device)
        with torch.cuda.device(qkv.device):
            st = lib.fwa_fwd_qkv(ctypes.byref(desc), _ptr(qkv5), _ptr(bias), _ptr(mask),
                                 _ptr(o), _ptr(ws), ctypes.c_size_t(ws_bytes), _stream(qkv.device))
        if st == 0:
            return o
        if st != 2 or kernel == "tc":
            nat.check(st)
    q, k, v = _split_qkv(qkv5)
    out = attention_forward(q, k, v, scale, bias, mask, kernel="generic" if kernel == "generic" else "auto")
    o.copy_(out.permute(0, 2, 1, 3).reshape(N, L, h * d))
    return o


def attention_backward_qkv(qkv: torch.Tensor, do: torch.Tensor, heads: int, scale: float = 1.0,
                           bias=None, mask=None, kernel: str = "auto", want_dbias: bool = False,
                           add_table: Optional[torch.Tensor] = None):
    """(dqkv (N, L, 3*heads*d), dBias-or-None) for dO in the proj layout (N, L, heads*d)."""
    qkv5 = _qkv_view(qkv, heads)
    N, L, _, h, d = qkv5.shape
    if tuple(do.shape) != (N, L, h * d) or not do.is_contiguous() or do.dtype != qkv.dtype:
        raise ShapeError(f"dO must be contiguous {qkv.dtype} (N, L, heads*d) = {(N, L, h * d)}")
    mw = _check_bias_mask((N, h, L, d), qkv.device, bias, mask)
    dqkv = torch.empty((N, L, 3 * h * d), dtype=qkv.dtype, device=qkv.device)
    dbias = torch.empty((h, L, L), dtype=torch.float32, device=qkv.device) if want_dbias else None
    if kernel != "generic" and qkv.dtype in (torch.float16, torch.bfloat16):
        desc = make_desc(N, h, L, d, qkv.dtype, scale, 1, mw, kernel, add_table)
        lib = nat.load()
        ws_bytes = int(lib.fwa_bwd_workspace_bytes(ctypes.byref(desc), int(bias is not None),
                                                   int(mask is not None), int(want_dbias)))
        ws = _workspace(ws_bytes, qkv.device)
        with torch.cuda.device(qkv.device):
            st = lib.fwa_bwd_qkv(ctypes.byref(desc), _ptr(qkv5), _ptr(do), _ptr(bias), _ptr(mask),
                                 _ptr(dqkv), _ptr(dbias), _ptr(ws), ctypes.c_size_t(ws_bytes),
                                 _stream(qkv.device))
        if st == 0:
            return dqkv, dbias
        if st != 2 or kernel == "tc":
            nat.check(st)
    q, k, v = _split_qkv(qkv5)
    do4 = do.view(N, L, h, d).permute(0, 2, 1, 3).contiguous()
    dq, dk, dv, db = attention_backward(q, k, v, do4, scale, bias, mask,
                                        kernel="generic" if kernel == "generic" else "auto",
                                        want_dbias=want_dbias)
    dqkv.view(N, L, 3, h, d).copy_(torch.stack([t.permute(0, 2, 1, 3) for t in (dq, dk, dv)], dim=2))
    return dqkv, db
