"""Multi-GPU driver pieces: windows are independent units, so the batch is
sharded into contiguous window ranges, one process per GPU, with no collective in the data
path.  Collectives (torch.distributed; NCCL on GPUs, gloo in the CPU tests) are used only for
the barrier around the timed region, the max-over-ranks reduction of elapsed time, and the
optional gather of per-window digests used to check that a sharded run reproduces the
single-GPU results bit for bit.
"""
from __future__ import annotations

import hashlib
import os

import numpy as np


def dist_env():
    """(world, rank, local_rank) from the torchrun environment (1, 0, 0 when absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n_windows: int, world: int, rank: int) -> range:
    """Contiguous, balanced range of window indices owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    q, r = divmod(n_windows, world)
    start = rank * q + min(rank, r)
    return range(start, start + q + (1 if rank < r else 0))


def window_digest(surface) -> int:
    """64-bit digest of one window's fp32 surface bits."""
    a = np.ascontiguousarray(np.asarray(surface, dtype=np.float32))
    return int.from_bytes(hashlib.blake2b(a.tobytes(), digest_size=8).digest(), "little")


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. elapsed ms of the timed region) over all ranks."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_digests(first_window: int, digests: list[int]) -> dict[int, int] | None:
    """Gather {window index: digest} from every rank; returned on rank 0, None elsewhere."""
    import torch.distributed as dist

    mine = {first_window + i: d for i, d in enumerate(digests)}
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return mine
    out = [None] * dist.get_world_size() if dist.get_rank() == 0 else None
    dist.gather_object(mine, out, dst=0)
    if dist.get_rank() != 0:
        return None
    merged = {}
    for part in out:
        overlap = merged.keys() & part.keys()
        if overlap:
            raise RuntimeError(f"windows processed twice: {sorted(overlap)[:5]}")
        merged.update(part)
    return merged
