"""Multi-GPU plumbing for the batch-sharded path (torch.distributed; no data-path collective).

Batches of independent images shard trivially: each rank solves its
own images with its own per-image iPiano state, so the only cross-rank traffic is the
timing barrier and the max-over-ranks reduction of the measured time.
"""
from __future__ import annotations

import os
from typing import List, Sequence


def world() -> tuple:
    """(rank, world_size, local_rank) from the torchrun environment (1-process defaults)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init_process_group(backend: str = "nccl"):
    """Initialise torch.distributed from the environment when WORLD_SIZE > 1."""
    import torch.distributed as dist
    rank, ws, local = world()
    if ws > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        kw = {}
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend=backend, rank=rank, world_size=ws, **kw)
    return rank, ws, local


def weak_shard(images_per_rank: int, rank: int) -> List[int]:
    """Weak scaling: rank r owns global images [r*n, (r+1)*n) -- per-GPU work fixed as N grows."""
    return list(range(rank * images_per_rank, (rank + 1) * images_per_rank))


def balanced_shard(looks: Sequence[int], rank: int, world_size: int) -> List[int]:
    """Strong scaling of a fixed batch: images sorted by looks L (which sets lambda and the
    trial counts), then dealt round-robin, so every rank gets the same L mix (+-1 image)."""
    order = sorted(range(len(looks)), key=lambda i: (looks[i], i))
    return sorted(order[rank::world_size])


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (identity without an initialised process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# ------------------------------------------------------------------ row slabs (c5)

def slab_rows(H_global: int, world_size: int, rank: int, band: int = 64) -> tuple:
    """Rows [r0, r1) of rank's slab: equal slabs of whole 64-row bands (include/foe.h
    ipiano_slabs_create), ranks in ring order top to bottom."""
    if H_global % (band * world_size):
        raise ValueError(f"H_global={H_global} is not a multiple of {band} x {world_size}")
    rows = H_global // world_size
    return rank * rows, (rank + 1) * rows


def ring_neighbours(rank: int, world_size: int) -> tuple:
    """(up, down): the slabs above and below in the periodic ring."""
    return (rank - 1) % world_size, (rank + 1) % world_size


def share_bytes(payload, src: int = 0) -> bytes:
    """Broadcast a small byte string (e.g. the NCCL unique id) from rank src to all ranks."""
    import torch.distributed as dist
    obj = [payload]
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast_object_list(obj, src=src)
    return obj[0]


def all_true(flag: bool) -> bool:
    """True on every rank iff the flag is true on every rank (collective decisions)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return bool(flag)
    vals = [None] * dist.get_world_size()
    dist.all_gather_object(vals, bool(flag))
    return all(vals)
