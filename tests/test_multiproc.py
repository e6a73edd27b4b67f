"""World-size-2 CPU (gloo) coverage of the multi-GPU path's host logic: batch sharding,
per-image seeds (any partition sees identical images), result gathering to rank 0 and the
max-over-ranks timing reduction.  The per-rank "kernel" here is the fp64 oracle (CPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2401_06197_b200.sharding import shard_images


def test_shard_images_partition():
    for batch in (1, 7, 64, 512):
        for world in (1, 2, 3, 4, 8):
            parts = [shard_images(batch, world, r) for r in range(world)]
            flat = [i for p in parts for i in p]
            assert flat == list(range(batch))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
    with pytest.raises(ValueError):
        shard_images(8, 2, 2)


def test_per_image_seeds_are_partition_invariant():
    a = synth.make_case(4, 6, 6, 2, 16, 6, 6, 9, 54, "f32")
    b = synth.make_case(2, 6, 6, 2, 16, 6, 6, 9, 54, "f32", images=[2, 3])
    for ta, tb in zip(a, b):
        assert torch.equal(ta[2:], tb)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, batch, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    imgs = shard_images(batch, world, rank)
    g = oracle.Geometry(N=len(imgs), H=7, W=6, G=2, D=16)
    x, om, gy = synth.make_case(len(imgs), 7, 6, 2, 16, 7, 6, 9, 54, "f32", images=imgs)
    y = torch.from_numpy(oracle.forward(g, x, om))
    _, gom = oracle.backward(g, x, om, gy)
    gom = torch.from_numpy(gom)
    # gather to rank 0 (shards have equal size here)
    ys = [torch.empty_like(y) for _ in range(world)] if rank == 0 else None
    goms = [torch.empty_like(gom) for _ in range(world)] if rank == 0 else None
    dist.gather(y, ys, dst=0)
    dist.gather(gom, goms, dst=0)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max-over-ranks step time
    if rank == 0:
        torch.save({"y": torch.cat(ys), "gom": torch.cat(goms), "tmax": t.item()}, out)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shard_gather_matches_single_process(tmp_path):
    batch, world = 4, 2
    out = str(tmp_path / "r0.pt")
    mp.start_processes(_worker, args=(world, _free_port(), batch, out), nprocs=world,
                       join=True, start_method="spawn")
    res = torch.load(out)
    g = oracle.Geometry(N=batch, H=7, W=6, G=2, D=16)
    x, om, gy = synth.make_case(batch, 7, 6, 2, 16, 7, 6, 9, 54, "f32")
    y = oracle.forward(g, x, om)
    _, gom = oracle.backward(g, x, om, gy)
    assert np.array_equal(res["y"].numpy(), y)       # bit-identical across world sizes
    assert np.array_equal(res["gom"].numpy(), gom)
    assert res["tmax"] == 2.0
