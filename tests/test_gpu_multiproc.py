"""Sharded hot path with the real kernels: 2 ranks (processes) on one GPU, gloo.

Each rank draws only its shard of a global layer (counter-based SplitMix64 fill), runs the
forward and backward kernels on it and all-gathers per-window bit hashes of O / dQ / dK /
dV; rank 0 recomputes the whole layer alone and the hashes must match bit for bit (the
reference's worker-count invariance, pkg/tests/test_flash.py:308-319). The
ranks' kernels never wait on one another (no collective inside a kernel), so sharing one
GPU is safe; on a multi-GPU box bench.py runs the same check over NCCL after its timing.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, layer, batch, dtype, path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2501_06480_b200.shard import validate_sharding

    res = validate_sharding(rank, world, torch.device("cuda", 0), layer, batch, dtype)
    if rank == 0:
        torch.save(res, path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("layer,batch,dtype", [
    ((1024, 3, 49, 32), 16, torch.float16),     # Swin-T stage 1 windows (tile kernels)
    ((320, 4, 144, 32), 5, torch.bfloat16),      # Swin-B window 12 (flat-row kernels), ragged
])
def test_sharded_kernels_match_one_gpu_bitwise(tmp_path, world, layer, batch, dtype):
    path = str(tmp_path / "res.pt")
    mp.start_processes(_worker, args=(world, _free_port(), layer, batch, dtype, path),
                       nprocs=world, join=True, start_method="spawn")
    res = torch.load(path)
    assert res["ok"], res
