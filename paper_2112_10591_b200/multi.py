"""Multi-GPU driver pieces: windows are independent units,
so the batch is sharded into contiguous window ranges, one process per GPU, with no collective
in the data path.  Collectives (torch.distributed; NCCL on GPUs, gloo in the CPU tests) are
used only for the barrier around the timed region, the max-over-ranks reduction of elapsed
time, and the gather of per-window digests that checks a sharded run against a single-rank
recompute bit for bit.

This module imports neither the package's native library nor the oracle: bench.py loads it by
path, so its reference arm never maps libieds.so.
"""
from __future__ import annotations

import hashlib
import os
import socket
import subprocess
import sys

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


def sample_windows(rng: range, k: int = 3) -> list[int]:
    """Up to k global window indices spread over a rank's shard: first, evenly spaced, last."""
    n = len(rng)
    if n == 0:
        return []
    if n <= k:
        return list(rng)
    return sorted({rng[(i * (n - 1)) // (k - 1)] for i in range(k)})


def window_digest(surface) -> int:
    """64-bit digest of one window's surface bytes (dtype preserved: fp32, fp16 or uint8)."""
    a = np.ascontiguousarray(np.asarray(surface))
    return int.from_bytes(hashlib.blake2b(a.tobytes(), digest_size=8).digest(), "little")


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. elapsed ms of the timed region) over all ranks."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_digest_map(mine: dict[int, int]) -> dict[int, int] | None:
    """Gather {global window index: digest} from every rank; the union on rank 0, None elsewhere.
    A window reported by two ranks is an error (the shards must partition the batch)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return dict(mine)
    out = [None] * dist.get_world_size() if dist.get_rank() == 0 else None
    dist.gather_object(dict(mine), out, dst=0)
    if dist.get_rank() != 0:
        return None
    merged: dict[int, int] = {}
    for part in out:
        overlap = merged.keys() & part.keys()
        if overlap:
            raise RuntimeError(f"windows processed twice: {sorted(overlap)[:5]}")
        merged.update(part)
    return merged


def gather_digests(first_window: int, digests: list[int]) -> dict[int, int] | None:
    """gather_digest_map for a contiguous shard starting at first_window."""
    return gather_digest_map({first_window + i: d for i, d in enumerate(digests)})


def cross_rank_check(mine: dict[int, int], recompute) -> dict | None:
    """Gather every rank's sampled digests to rank 0 and compare them with `recompute(indices)`,
    a single-rank recompute returning {index: digest}.  Rank 0 gets a summary dict, the other
    ranks None.  recompute runs on rank 0 only."""
    merged = gather_digest_map(mine)
    if merged is None:
        return None
    idx = sorted(merged)
    ref = recompute(idx)
    bad = [i for i in idx if ref.get(i) != merged[i]]
    return {"windows_checked": len(idx), "match": not bad, "mismatched": bad[:8]}


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def torchrun_command(nproc: int, script: str, argv: list[str], port: int | None = None) -> list[str]:
    """The driver's launch line for N ranks on one node (rendezvous on 127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr", "127.0.0.1", f"--master-port={port or free_port()}", script] + list(argv)


def relaunch_under_torchrun(nproc: int, script: str, argv: list[str]) -> int:
    """`python bench.py --gpus N` without torchrun: re-run the same command as N ranks under
    torch.distributed.run and return its exit code (rank 0's JSON line passes through)."""
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(torchrun_command(nproc, script, argv), env=env)
