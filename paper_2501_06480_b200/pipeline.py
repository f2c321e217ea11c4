"""Host-buffer execution of the batched ops: H2D, kernel and D2H overlapped on three streams.

Used by ``api.batched_flash_forward`` / ``batched_flash_backward`` when the
caller passes host tensors (the reference's calling convention: everything in
host memory). The window batch is split into chunks whose starts are multiples
of the mask period nW (window n keeps mask[n % nW]); chunk i+1 is copied in
while chunk i computes and chunk i-1 is copied out, so the PCIe transfers,
not the sum of transfer + compute, bound the wall time.
"""

from __future__ import annotations

from typing import Optional

import torch

from . import ops


def _chunk_bounds(n: int, period: int, chunks: int):
    period = max(1, period)
    blocks = -(-n // period)
    per = max(1, -(-blocks // max(1, chunks))) * period
    return [(a, min(n, a + per)) for a in range(0, n, per)]


def _n_chunks(t: torch.Tensor, requested) -> int:
    """Chunks of ~CHUNK_BYTES per input tensor (the pipeline's fill + drain is one chunk of
    H2D and one of D2H, so more chunks overlap more; each costs a few launches).
    FWA_HOST_CHUNK_MB overrides the chunk size."""
    if requested:
        return requested
    import os

    mb = float(os.environ.get("FWA_HOST_CHUNK_MB", "8"))
    return int(min(128, max(2, -(-t.numel() * t.element_size() // int(mb * (1 << 20))))))


def _pinned(t: torch.Tensor) -> torch.Tensor:
    t = t.contiguous()
    return t if t.is_pinned() else t.pin_memory()


def host_forward(qh: torch.Tensor, kh: torch.Tensor, vh: torch.Tensor, scale: float,
                 bias: Optional[torch.Tensor] = None, mask: Optional[torch.Tensor] = None,
                 chunks_r: int = 1, kernel: str = "auto", n_chunks: int = 0) -> torch.Tensor:
    """O for host (N, h, L, d) tensors; returns a pinned host tensor."""
    dev = torch.device("cuda", torch.cuda.current_device())
    qh, kh, vh = _pinned(qh), _pinned(kh), _pinned(vh)
    N = qh.shape[0]
    out_h = torch.empty(qh.shape, dtype=qh.dtype, pin_memory=True)
    comp = torch.cuda.current_stream(dev)
    qd = torch.empty(qh.shape, dtype=qh.dtype, device=dev)
    kd, vd, od = torch.empty_like(qd), torch.empty_like(qd), torch.empty_like(qd)
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    h2d.wait_stream(comp)
    d2h.wait_stream(comp)
    for t in (qd, kd, vd):
        t.record_stream(h2d)
    od.record_stream(d2h)
    nW = mask.shape[0] if mask is not None else 1
    for a, b in _chunk_bounds(N, nW, _n_chunks(qh, n_chunks)):
        with torch.cuda.stream(h2d):
            for dst, src in ((qd, qh), (kd, kh), (vd, vh)):
                dst[a:b].copy_(src[a:b], non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(h2d)
        comp.wait_event(ev_in)
        ops.attention_forward(qd[a:b], kd[a:b], vd[a:b], scale, bias, mask, chunks=chunks_r,
                              kernel=kernel, out=od[a:b])
        ev_c = torch.cuda.Event()
        ev_c.record(comp)
        d2h.wait_event(ev_c)
        with torch.cuda.stream(d2h):
            out_h[a:b].copy_(od[a:b], non_blocking=True)
    d2h.synchronize()
    return out_h


def host_backward(qh, kh, vh, doh, scale: float, bias=None, mask=None, chunks_r: int = 1,
                  kernel: str = "auto", want_dbias: bool = False, n_chunks: int = 0):
    """(dQ, dK, dV) pinned host tensors (+ dBias on the device, summed over chunks in order)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    qh, kh, vh, doh = _pinned(qh), _pinned(kh), _pinned(vh), _pinned(doh)
    N = qh.shape[0]
    outs_h = [torch.empty(qh.shape, dtype=qh.dtype, pin_memory=True) for _ in range(3)]
    comp = torch.cuda.current_stream(dev)
    ins_d = [torch.empty(qh.shape, dtype=qh.dtype, device=dev) for _ in range(4)]
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    h2d.wait_stream(comp)
    d2h.wait_stream(comp)
    for t in ins_d:
        t.record_stream(h2d)
    nW = mask.shape[0] if mask is not None else 1
    dbias = None
    for a, b in _chunk_bounds(N, nW, _n_chunks(qh, n_chunks)):
        with torch.cuda.stream(h2d):
            for dst, src in zip(ins_d, (qh, kh, vh, doh)):
                dst[a:b].copy_(src[a:b], non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(h2d)
        comp.wait_event(ev_in)
        dq, dk, dv, db = ops.attention_backward(*(t[a:b] for t in ins_d), scale, bias, mask,
                                                chunks=chunks_r, kernel=kernel,
                                                want_dbias=want_dbias)
        if want_dbias:
            dbias = db if dbias is None else dbias + db
        ev_c = torch.cuda.Event()
        ev_c.record(comp)
        d2h.wait_event(ev_c)
        with torch.cuda.stream(d2h):
            for dst, src in zip(outs_h, (dq, dk, dv)):
                src.record_stream(d2h)
                dst[a:b].copy_(src, non_blocking=True)
    d2h.synchronize()
    return (*outs_h, dbias)
