"""One-process-per-GPU plumbing over torch.distributed (the bench contract's
launch mode). torch is only the transport for the shards' IPC blobs (a few KB,
once); the data path is the library's peer-pointer edge reads.

    shard = open_ring_shard(cfg)     # rank/world/device from the environment
    shard.advance()                  # lockstep with the ring neighbours
"""
from __future__ import annotations

import os
from typing import Optional, Tuple


def ring_neighbours(rank: int, world: int) -> Tuple[int, int]:
    """(left, right) of `rank` on the periodic ring (partition.cpp:28-33)."""
    return (rank + world - 1) % world, (rank + 1) % world


def exchange_ring(blob: bytes, rank: int, world: int, group=None) -> Tuple[bytes, bytes]:
    """All-gather every rank's blob and return (left neighbour's, right neighbour's)."""
    import torch.distributed as dist
    blobs = [None] * world
    dist.all_gather_object(blobs, blob, group=group)
    left, right = ring_neighbours(rank, world)
    return blobs[left], blobs[right]


def open_ring_shard(cfg, rank: Optional[int] = None, world: Optional[int] = None, device: Optional[int] = None,
                    group=None):
    """Create this process's shard of `cfg` (cfg.ranks must equal the world
    size) and connect it to its ring neighbours."""
    import torch.distributed as dist

    from .api import InvalidConfig, Shard
    rank = dist.get_rank(group) if rank is None else rank
    world = dist.get_world_size(group) if world is None else world
    if device is None:  # one GPU per local rank (wraps when ranks outnumber GPUs, e.g. tests)
        from .api import device_count
        device = int(os.environ.get("LOCAL_RANK", rank)) % max(1, device_count())
    if cfg.ranks != world:
        raise InvalidConfig(f"cfg.ranks={cfg.ranks} must equal the process count {world}")
    shard = Shard(cfg, rank, device)
    left, right = exchange_ring(shard.export(), rank, world, group)
    shard.connect(left, right)
    return shard
