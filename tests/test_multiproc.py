"""Multi-process (world_size 2, gloo, CPU) coverage of the sharded path.

Each rank owns a contiguous range of whole images (shard.shard_images), runs
window attention on its windows (here the CPU oracle stands in for the
kernel, since there is no GPU in this container), and the per-window
checksums are gathered with shard.gather_checksums. The gathered vector must
equal the single-process result bit for bit, and each rank's mask indices
(n mod nW) must be unchanged by the sharding.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import flashwin_oracle as orc
from paper_2501_06480_b200.shard import gather_checksums, shard_images, unit_checksum

B, NW, H, L, D = 5, 4, 2, 16, 8   # 5 images x 4 windows, ragged split over 2 ranks


def _inputs():
    q, k, v = orc.draw_qkvdo(321, (B * NW, H, L, D), 3)
    mask = orc.shifted_window_mask(8, 8, 4, 2)        # (4, 16, 16)
    bias = orc.fill_uniform(orc.Rng(5), (H, L, L), -0.2, 0.2)
    return q, k, v, bias, mask


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q, k, v, bias, mask = _inputs()
    sh = shard_images(B, NW, rank, world)
    sl = slice(sh.window_begin, sh.window_end)
    # local windows keep their global mask index because shards start at image boundaries
    o, _ = orc.attention_forward(q[sl], k[sl], v[sl], 0.35, bias=bias, mask=mask)
    local = unit_checksum(torch.from_numpy(o))
    counts = [shard_images(B, NW, r, world).windows for r in range(world)]
    full = gather_checksums(local, counts)
    if rank == 0:
        torch.save(full, result_path)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_matches_single_process(tmp_path):
    path = str(tmp_path / "gathered.pt")
    mp.start_processes(_worker, args=(2, _free_port(), path), nprocs=2, join=True,
                       start_method="spawn")
    gathered = torch.load(path)
    q, k, v, bias, mask = _inputs()
    o, _ = orc.attention_forward(q, k, v, 0.35, bias=bias, mask=mask)
    ref = unit_checksum(torch.from_numpy(o))
    assert gathered.shape == ref.shape
    assert torch.equal(gathered, ref)  # bitwise: same units, same order, same arithmetic


def test_shards_preserve_mask_index():
    for world in (1, 2, 3, 4):
        for r in range(world):
            sh = shard_images(B, NW, r, world)
            assert sh.window_begin % NW == 0
            assert [n % NW for n in range(sh.window_begin, sh.window_end)] == \
                [n % NW for n in range(sh.windows)]
