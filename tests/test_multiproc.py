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


def _worker(rank, world, port, batch, out, corrupt):
    """One rank of bench.py's N > 1 host logic under gloo: shard, compute this rank's images
    (the fp64 oracle stands in for the kernels), then bench.cross_rank_check (gather of
    every rank's first-image outputs to rank 0 and recompute-alone comparison) and
    bench.max_over_ranks (the step-time reduction) -- the functions bench.py itself calls."""
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    imgs = bench._shard(batch, world, rank, True)
    cpu = torch.device("cpu")

    def outputs_of(images):
        g = oracle.Geometry(N=len(images), H=7, W=6, G=2, D=16)
        x, om, gy = synth.make_case(len(images), 7, 6, 2, 16, 7, 6, 9, 54, "f32", images=images)
        y = torch.from_numpy(oracle.forward(g, x, om))
        gom = torch.from_numpy(oracle.backward(g, x, om, gy)[1])
        return [y, gom]

    mine = [t[:1] for t in outputs_of(imgs)]
    if corrupt and rank == 1:
        mine[1] = mine[1].clone()
        mine[1].view(-1)[5] += 1e-12
    res = bench.cross_rank_check(imgs[0], mine, lambda n, i: outputs_of([n])[i], world, rank,
                                 dist, cpu)
    tmax = bench.max_over_ranks(float(rank + 1), world, dist, cpu)
    if rank == 0:
        torch.save({"check": res, "tmax": tmax, "firsts": imgs[0]}, out)
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("corrupt", [False, True])
def test_two_rank_gloo_bench_cross_rank_check(tmp_path, corrupt):
    batch, world = 4, 2
    out = str(tmp_path / "r0.pt")
    mp.start_processes(_worker, args=(world, _free_port(), batch, out, corrupt), nprocs=world,
                       join=True, start_method="spawn")
    res = torch.load(out)
    assert res["check"] == {"cross_rank_bitexact": not corrupt, "ranks": 2}
    assert res["tmax"] == 2.0


def test_bench_self_launches_ranks_for_gpus_n():
    """`python bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks; the
    reference arm (CPU, rank 0 prints) proves the launcher and the rank environment."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["OMP_NUM_THREADS"] = "2"
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--workload", "c1", "--steps", "1", "--warmup", "3"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, p.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
