"""CPU oracle for the Flash Window Attention hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` leg /
``--impl reference`` arm may import it. The product path
(``paper_2501_06480_b200``) never imports anything under ``oracle/`` and fails
loudly when its CUDA library is missing.

It is a float64 NumPy restatement of the reference package ``flashwin``
(``/root/reference/pkg/src/flashwin``), vectorised over (window, head) units:

* SplitMix64 ``Rng`` / ``fill_uniform``      — tensor.py:74-138
* ``naive_forward`` / ``naive_backward``     — reference.py:49-124
* tiled forward (Alg. 1, chunked S)          — flash.py:141-184
* tiled backward (Alg. 2, three phases)      — flash.py:187-266
* ``TileConfig`` chunk arithmetic            — flash.py:41-71
* ``peak_sram_forward/backward``             — flash.py:84-95
* ``window_partition`` / ``window_reverse``  — windowing.py:44-70

plus an EXTENSION the reference does not have (SPEC.md:14 puts it out of
scope there): the Swin additive relative-position bias and shifted-window
mask, S = scale*QK^T + bias[h] + mask[n mod nW], and the matching dBias.
With bias = mask = None every function reduces exactly to the reference.

Parity pinning: the non-extension functions are checked against golden
vectors produced by importing the real reference (``tests/golden/make_golden.py``
→ ``tests/golden/*.npz|json``; see ``tests/test_oracle.py``). The bias/mask
extension is pinned only by its reduction to the reference at bias=mask=0
and by finite differences ("parity unpinned" for the extension itself).
"""

from __future__ import annotations

import math

import numpy as np

# SplitMix64 constants (tensor.py:19-22)
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1


# ---------------------------------------------------------------------------
# SplitMix64 (tensor.py:74-138)
# ---------------------------------------------------------------------------
class Rng:
    """SplitMix64 stream; same state update and mixing as tensor.py:74-101."""

    __slots__ = ("state",)

    def __init__(self, seed: int):
        self.state = int(seed) & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + GOLDEN) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * MIX1) & MASK64
        z = ((z ^ (z >> 27)) * MIX2) & MASK64
        return z ^ (z >> 31)

    def next_float(self) -> float:
        return (self.next_u64() >> 11) * 2.0**-53

    def split(self) -> "Rng":
        return Rng(self.next_u64())


def splitmix_u64(state: int, n: int) -> np.ndarray:
    """Draws 1..n of the stream whose current state is ``state`` (tensor.py:129-135)."""
    idx = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(state) + np.uint64(GOLDEN) * idx
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
    return z ^ (z >> np.uint64(31))


def fill_uniform(rng: Rng, shape, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Row-major i.i.d. U[lo, hi) draws, one SplitMix64 draw per element (tensor.py:118-138)."""
    shape = tuple(int(e) for e in shape)
    n = math.prod(shape)
    z = splitmix_u64(rng.state, n)
    rng.state = (rng.state + n * GOLDEN) & MASK64
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0**-53
    return (lo + (hi - lo) * u).reshape(shape)


def draw_qkvdo(seed: int, shape, n: int = 4, lo: float = -1.0, hi: float = 1.0):
    """q, k, v[, dO] as successive fill_uniform draws of one Rng(seed) (harness.py:202, :498)."""
    rng = Rng(seed)
    return [fill_uniform(rng, shape, lo, hi) for _ in range(n)]


# ---------------------------------------------------------------------------
# TileConfig arithmetic (flash.py:41-71) and peaks (flash.py:84-95)
# ---------------------------------------------------------------------------
def chunk_width(C: int, r: int) -> int:
    if r > C:
        raise ValueError(f"chunk count {r} exceeds feature count {C}")
    cw = -(-C // r)
    if cw * (r - 1) >= C:
        raise ValueError(f"chunk count {r} leaves an empty chunk for {C} features")
    return cw


def chunk_spans(C: int, r: int):
    cw = chunk_width(C, r)
    return [(i * cw, min((i + 1) * cw, C)) for i in range(r)]


def peak_sram_forward(L: int, C: int, r: int, elem_bytes: int = 4) -> int:
    return (L * L + 2 * L * chunk_width(C, r)) * elem_bytes


def peak_sram_backward(L: int, C: int, r: int, elem_bytes: int = 4) -> int:
    return (2 * L * L + 2 * L * chunk_width(C, r)) * elem_bytes


# ---------------------------------------------------------------------------
# Attention (reference.py:49-124) batched over leading axes, plus bias/mask
# ---------------------------------------------------------------------------
def _additive(S_shape, heads_axis_len, bias, mask, mask_windows):
    """Broadcast bias (h,L,L) and mask (nW,L,L) onto S of shape (N,h,L,L)."""
    add = 0.0
    if bias is not None:
        add = add + np.asarray(bias, dtype=np.float64)[None, :, :, :]
    if mask is not None:
        m = np.asarray(mask, dtype=np.float64)
        N = S_shape[0]
        nW = m.shape[0] if mask_windows is None else mask_windows
        idx = np.arange(N) % nW
        add = add + m[idx][:, None, :, :]
    return add


def softmax_rows(s: np.ndarray) -> np.ndarray:
    """Max-subtracted row softmax over the last axis (reference.py:49-58)."""
    if not np.isfinite(s).all():
        raise FloatingPointError("softmax input contains non-finite entries")
    e = np.exp(s - s.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def attention_forward(q, k, v, scale=1.0, bias=None, mask=None, mask_windows=None):
    """O, P for q,k,v of shape (..., L, d); 4-D (N,h,L,d) when bias/mask given.

    reference.py:69-78 (S = scale*QK^T, P = softmax_rows(S), O = PV) + extension.
    """
    q, k, v = (np.asarray(t, dtype=np.float64) for t in (q, k, v))
    s = scale * (q @ np.swapaxes(k, -1, -2))
    if bias is not None or mask is not None:
        s = s + _additive(s.shape, s.shape[1], bias, mask, mask_windows)
    p = softmax_rows(s)
    return p @ v, p


def attention_backward(q, k, v, p, do, scale=1.0, want_dbias=False):
    """dQ, dK, dV (and dBias summed over windows) — reference.py:81-124.

    dV = P^T dO; dP = dO V^T; dS = P*(dP - rowdot(P,dP)); dQ = scale*dS K;
    dK = scale*dS^T Q. dBias[h] = sum_n dS[n,h] (extension; dS before the scale).
    """
    q, k, v, p, do = (np.asarray(t, dtype=np.float64) for t in (q, k, v, p, do))
    dv = np.swapaxes(p, -1, -2) @ do
    dp = do @ np.swapaxes(v, -1, -2)
    ds = p * (dp - (p * dp).sum(axis=-1, keepdims=True))
    dq = scale * (ds @ k)
    dk = scale * (np.swapaxes(ds, -1, -2) @ q)
    if want_dbias:
        return dq, dk, dv, ds.sum(axis=0)
    return dq, dk, dv


def mask_grad(ds: np.ndarray, nW: int) -> np.ndarray:
    """dMask[w] = sum over windows n with n mod nW == w (extension)."""
    N = ds.shape[0]
    out = np.zeros((nW,) + ds.shape[2:])
    np.add.at(out, np.arange(N) % nW, ds.sum(axis=1))
    return out


# ---------------------------------------------------------------------------
# Tiled Alg. 1 / Alg. 2 (flash.py:141-266), vectorised over units
# ---------------------------------------------------------------------------
def tiled_forward(q, k, v, r: int, scale: float = 1.0):
    """Feature-chunked forward: S = sum_i Q_i K_i^T; softmax; O_i = P V_i (flash.py:162-180).

    Returns (O, traffic) where traffic counts elements per operand like
    flash.py:106-124 (loads Q,K,V = L*C per unit; stores O = L*C per unit).
    """
    q, k, v = (np.asarray(t, dtype=np.float64) for t in (q, k, v))
    *lead, L, C = q.shape
    units = math.prod(lead) if lead else 1
    spans = chunk_spans(C, r)
    s = np.zeros(tuple(lead) + (L, L))
    for lo, hi in spans:
        s += q[..., lo:hi] @ np.swapaxes(k[..., lo:hi], -1, -2)
    s *= scale
    s -= s.max(axis=-1, keepdims=True)
    np.exp(s, out=s)
    s /= s.sum(axis=-1, keepdims=True)
    o = np.empty_like(q)
    for lo, hi in spans:
        o[..., lo:hi] = s @ v[..., lo:hi]
    n = units * L * C
    return o, {"loads": {"Q": n, "K": n, "V": n}, "stores": {"O": n}}


def tiled_backward(q, k, v, do, r: int, scale: float = 1.0):
    """Three-phase backward of flash.py:187-266 (P recomputed, Q/K reloaded)."""
    q, k, v, do = (np.asarray(t, dtype=np.float64) for t in (q, k, v, do))
    *lead, L, C = q.shape
    units = math.prod(lead) if lead else 1
    spans = chunk_spans(C, r)
    p = np.zeros(tuple(lead) + (L, L))
    for lo, hi in spans:  # phase 1 (flash.py:215-225)
        p += q[..., lo:hi] @ np.swapaxes(k[..., lo:hi], -1, -2)
    p *= scale
    p -= p.max(axis=-1, keepdims=True)
    np.exp(p, out=p)
    p /= p.sum(axis=-1, keepdims=True)
    dp = np.zeros_like(p)
    dv = np.empty_like(q)
    for lo, hi in spans:  # phase 2 (flash.py:227-238)
        dp += do[..., lo:hi] @ np.swapaxes(v[..., lo:hi], -1, -2)
        dv[..., lo:hi] = np.swapaxes(p, -1, -2) @ do[..., lo:hi]
    ds = p * (dp - (p * dp).sum(axis=-1, keepdims=True))  # flash.py:133-138
    ds *= scale
    dq = np.empty_like(q)
    dk = np.empty_like(q)
    for lo, hi in spans:  # phase 3 (flash.py:245-257)
        dq[..., lo:hi] = ds @ k[..., lo:hi]
        dk[..., lo:hi] = np.swapaxes(ds, -1, -2) @ q[..., lo:hi]
    n = units * L * C
    traffic = {
        "loads": {"Q": 2 * n, "K": 2 * n, "V": n, "dO": n},
        "stores": {"dQ": n, "dK": n, "dV": n},
    }
    return dq, dk, dv, traffic


# ---------------------------------------------------------------------------
# Windowing (windowing.py:44-70) + batch axis and Swin cyclic shift (extension)
# ---------------------------------------------------------------------------
def window_partition(x: np.ndarray, k: int, shift: int = 0) -> np.ndarray:
    """(H,W,C) -> (nW,L,C) or (B,H,W,C) -> (B*nW,L,C); windowing.py:44-54.

    shift > 0 applies Swin's cyclic shift first: x = roll(x, (-shift,-shift), (H,W)).
    """
    x = np.asarray(x)
    single = x.ndim == 3
    if single:
        x = x[None]
    B, H, W, C = x.shape
    if H % k or W % k:
        raise ValueError(f"window size {k} must divide image {H}x{W}")
    if shift:
        x = np.roll(x, (-shift, -shift), axis=(1, 2))
    y = x.reshape(B, H // k, k, W // k, k, C).transpose(0, 1, 3, 2, 4, 5)
    return y.reshape(B * (H // k) * (W // k), k * k, C)


def window_reverse(y: np.ndarray, k: int, H: int, W: int, shift: int = 0, batched: bool = True):
    """Inverse of window_partition (windowing.py:57-70), then roll(+shift)."""
    y = np.asarray(y)
    nW = (H // k) * (W // k)
    B = y.shape[0] // nW
    C = y.shape[-1]
    x = y.reshape(B, H // k, W // k, k, k, C).transpose(0, 1, 3, 2, 4, 5).reshape(B, H, W, C)
    if shift:
        x = np.roll(x, (shift, shift), axis=(1, 2))
    return x if batched else x[0]


# ---------------------------------------------------------------------------
# Swin relative-position bias and shifted-window mask (extension, not in reference)
# ---------------------------------------------------------------------------
def relative_position_index(k: int) -> np.ndarray:
    """(L, L) int index into the ((2k-1)^2, h) table, Swin's definition."""
    coords = np.stack(np.meshgrid(np.arange(k), np.arange(k), indexing="ij")).reshape(2, -1)
    rel = coords[:, :, None] - coords[:, None, :]
    rel = rel.transpose(1, 2, 0) + (k - 1)
    return (rel[..., 0] * (2 * k - 1) + rel[..., 1]).astype(np.int64)


def gather_bias(table: np.ndarray, k: int) -> np.ndarray:
    """table ((2k-1)^2, h) -> bias (h, L, L)."""
    idx = relative_position_index(k)
    return np.asarray(table)[idx.reshape(-1)].reshape(k * k, k * k, -1).transpose(2, 0, 1)


def shifted_window_mask(H: int, W: int, k: int, shift: int, neg: float = -100.0) -> np.ndarray:
    """(nW, L, L) additive mask of Swin's shifted-window attention (0 or ``neg``)."""
    img = np.zeros((1, H, W, 1))
    cnt = 0
    for hs in (slice(0, -k), slice(-k, -shift), slice(-shift, None)):
        for ws in (slice(0, -k), slice(-k, -shift), slice(-shift, None)):
            img[:, hs, ws, :] = cnt
            cnt += 1
    mw = window_partition(img[0], k)[..., 0]  # (nW, L)
    diff = mw[:, None, :] - mw[:, :, None]
    return np.where(diff != 0, neg, 0.0)
