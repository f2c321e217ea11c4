"""Multi-GPU sharding of the window-attention hot path.

Units are independent in forward and backward, so G ranks (one process per
GPU, torchrun) take contiguous ranges of whole images: rank r owns images
[B*r/G, B*(r+1)/G) -> windows [b0*nW, b1*nW). Window n keeps mask index
n mod nW with no remapping (image boundaries are multiples of nW) and there
is no halo. No collective runs on the hot path; ``gather_checksums`` is the
optional validation gather (NCCL all_gather over NVLink on GPUs, gloo on CPU).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    image_begin: int
    image_end: int
    window_begin: int
    window_end: int

    @property
    def images(self) -> int:
        return self.image_end - self.image_begin

    @property
    def windows(self) -> int:
        return self.window_end - self.window_begin


def shard_images(batch: int, windows_per_image: int, rank: int, world: int) -> Shard:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    b0 = batch * rank // world
    b1 = batch * (rank + 1) // world
    return Shard(rank, world, b0, b1, b0 * windows_per_image, b1 * windows_per_image)


def unit_checksum(t: torch.Tensor) -> torch.Tensor:
    """Per-window float64 checksum (sum over heads, rows, features) — order-fixed."""
    return t.double().flatten(1).sum(dim=1)


def window_hash(t: torch.Tensor) -> torch.Tensor:
    """Per-window int64 hash of the raw bits of a (N, ...) tensor: sum of bits x (position + 1)
    with wrapping integer arithmetic, so any single-bit difference shows and the value does not
    depend on summation order (bitwise comparisons across world sizes)."""
    n = t.shape[0]
    bits = t.contiguous().view(n, -1)
    ib = {2: torch.int16, 4: torch.int32, 8: torch.int64}[t.element_size()]
    b = bits.view(ib).to(torch.int64)
    w = torch.arange(1, b.shape[1] + 1, device=t.device, dtype=torch.int64) * 0x9E3779B1
    return (b * w).sum(dim=1)


def gather_checksums(local: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """all_gather of per-window checksums (n_local, ...) of unequal shard sizes -> full
    (sum(counts), ...) on every rank (validation only; NCCL over NVLink on GPUs, gloo on CPU)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    width = max(counts)
    on_dev = dist.get_backend(group) == "nccl"
    src = local if on_dev else local.cpu()
    buf = torch.zeros((width,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    buf[: src.shape[0]] = src
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return torch.cat([o[:c] for o, c in zip(outs, counts)])


def validate_sharding(rank: int, world: int, device, layer=(8192, 3, 49, 32), batch: int = 128,
                      dtype=torch.float16, seed: int = 42, group=None) -> dict:
    """1-GPU vs G-GPU bitwise check of the sharded hot path (analogue of the reference's
    worker-count invariance test, pkg/tests/test_flash.py:308-319).

    Every rank draws only its shard of one global (N, h, L, d) layer (counter-based fill),
    runs the forward and backward kernels on it, hashes each window's O / dQ / dK / dV bits
    and all-gathers the hashes; rank 0 then recomputes the whole layer alone and compares.
    Returns {"ok": bool-on-rank-0, ...} (ok is None on other ranks).
    """
    from . import ops
    from .rng import fill_uniform_at

    N, h, L, d = layer
    nW = N // batch
    sh = shard_images(batch, nW, rank, world)
    unit = h * L * d
    scale = d ** -0.5

    def run(w0, w1):
        shape = (w1 - w0, h, L, d)
        q, k, v, do = (fill_uniform_at(seed + i * N * unit * 0x9E3779B97F4A7C15, w0 * unit, shape,
                                       dtype=dtype, device=device) for i in range(4))
        o = ops.attention_forward(q, k, v, scale)
        dq, dk, dv, _ = ops.attention_backward(q, k, v, do, scale)
        return torch.stack([window_hash(t) for t in (o, dq, dk, dv)], dim=1)

    local = run(sh.window_begin, sh.window_end) if sh.windows else \
        torch.zeros((0, 4), dtype=torch.int64, device=device)
    counts = [shard_images(batch, nW, r, world).windows for r in range(world)]
    full = gather_checksums(local, counts, group)
    out = {"ok": None, "layer": list(layer), "images": batch, "world": world,
           "checked": "per-window bit hashes of O, dQ, dK, dV"}
    if rank == 0:
        ref = run(0, N).to(full.device)
        out["ok"] = bool(torch.equal(full, ref))
        out["mismatched_windows"] = int((full != ref).any(dim=1).sum().item())
    return out
