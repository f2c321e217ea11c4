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


def gather_checksums(local: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """all_gather of per-window checksums of unequal shard sizes -> full vector (validation only)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    width = max(counts)
    buf = torch.zeros(width, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return torch.cat([o[:c] for o, c in zip(outs, counts)])
