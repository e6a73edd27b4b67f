"""Batch sharding for multi-GPU runs: one process per GPU, images are
independent (y[n] depends only on x[n], om[n]; grad_input[n] only on gy[n]), so rank r of
world size W owns a contiguous block of images and no collective touches the data path.
NCCL is used only outside the timed region (barrier, max-over-ranks timing, verification
gathers)."""
from __future__ import annotations

import os
from typing import List, Tuple


def dist_env() -> Tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 if absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_images(batch: int, world: int, rank: int) -> List[int]:
    """Global image indices owned by `rank`: a contiguous block, sizes differing by at most
    one when `world` does not divide `batch` (strong scaling of a fixed global batch)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))
