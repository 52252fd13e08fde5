"""Multi-GPU plumbing for the SPS library (host side only).

One process per GPU; torch.distributed is used for the bootstrap only: rank 0 asks
libremoe for an NCCL unique id and broadcasts the 128 bytes over the process group,
then every rank calls remoe_sps_build with its contiguous row shard.  All data-path
exchange (candidate all-gather, winner-row all-reduce) happens inside the library
over NCCL.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .sps import Sps, remoe_nccl_unique_id


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row shard of `rank`: (global offset, rows), the balanced split
    offset_g = floor(n_total * g / world).  Ranks tile [0, n_total); every shard is
    non-empty whenever n_total >= world (a ceil(n/world) split can leave the last ranks
    empty, e.g. n = 9 over 4 ranks)."""
    lo = n_total * rank // world
    hi = n_total * (rank + 1) // world
    return lo, hi - lo


def broadcast_unique_id(group=None, device=None) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank returns the same 128 bytes."""
    rank = dist.get_rank(group)
    dev = device if device is not None else torch.device("cpu")
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(remoe_nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0, group=group)
    return bytes(t.cpu().numpy())


def build_sharded(emb_shard, act_shard, n_total: int, *, group=None, device: int = 0, **kw) -> Sps:
    """Collective: build this rank's handle over its shard of an n_total-row store."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    off, n = shard_range(n_total, world, rank)
    assert emb_shard.shape[0] == n, f"rank {rank}: expected {n} rows, got {emb_shard.shape[0]}"
    backend = dist.get_backend(group)
    bdev = torch.device("cuda", device) if backend == "nccl" else None
    uid = broadcast_unique_id(group, bdev) if world > 1 else None
    return Sps(emb_shard, act_shard, device=device, rank=rank, world=world, global_offset=off,
               nccl_unique_id=uid, **kw)
