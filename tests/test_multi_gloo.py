"""Multi-process (world_size 2, gloo, CPU) tests of the sharding / timing / digest logic.

The per-window work on each rank is stood in for by the CPU oracle on tiny windows: this is a
test-only mock of the device path (the product path never calls the oracle); what is under
test is the host logic -- shard arithmetic, max-over-ranks timing, digest gather -- and that a
sharded run reproduces the single-process results bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2112_10591_b200.multi import shard, window_digest
from synth.events import SceneConfig, batch_events

CFG = SceneConfig(64, 48, 600, n_prims=6, len_range=(8.0, 30.0), sigma=0.5)
N_WIN = 7
SEED = 11


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _surfaces(k0, n):
    import oracle

    xy, off = batch_events(CFG, SEED, k0, n)
    a = oracle.alpha_from_dsat(6.0)
    return [oracle.build_window(xy[off[b]:off[b + 1]], CFG.width, CFG.height, 1, 4, a, want=("S",))["S"]
            .astype(np.float32) for b in range(n)]


def _xcheck_worker(rank, world, port, q, corrupt):
    """bench.py's cross-rank parity check: sampled digests of each rank's shard, gathered to
    rank 0 and compared with rank 0's single-rank recompute (here: the oracle stands in for the
    device path on tiny windows, test-only)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist

    from paper_2112_10591_b200.multi import cross_rank_check, sample_windows

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = shard(N_WIN, world, rank)
        S = _surfaces(rng.start, len(rng))
        if corrupt and rank == 1:
            S[-1] = S[-1].copy()
            S[-1][0, 0] = np.nextafter(S[-1][0, 0], np.float32(2))
        mine = {i: window_digest(S[i - rng.start]) for i in sample_windows(rng, 3)}
        res = cross_rank_check(mine, lambda idx: {i: window_digest(_surfaces(i, 1)[0]) for i in idx})
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _run_two(target, *extra):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, 2, port, q) + extra) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        got = q.get(timeout=240)
        res[got[0]] = got[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("corrupt", [False, True])
def test_cross_rank_check_two_ranks(corrupt):
    res = _run_two(_xcheck_worker, corrupt)
    assert res[1][0] is None
    r0 = res[0][0]
    # rank 0 holds windows 0..3, rank 1 windows 4..6: 3 samples each
    assert r0["windows_checked"] == 6
    assert r0["match"] is (not corrupt)
    if corrupt:
        assert r0["mismatched"] == [N_WIN - 1]


def test_sample_windows():
    from paper_2112_10591_b200.multi import sample_windows

    assert sample_windows(range(0), 3) == []
    assert sample_windows(range(5, 7), 3) == [5, 6]
    assert sample_windows(range(100, 200), 3) == [100, 149, 199]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist

    from paper_2112_10591_b200.multi import gather_digests, max_over_ranks

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = shard(N_WIN, world, rank)
        S = _surfaces(rng.start, len(rng))
        dig = [window_digest(s) for s in S]
        merged = gather_digests(rng.start, dig)
        t = max_over_ranks(10.0 + rank)
        dist.barrier()
        q.put((rank, merged, t))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_partition():
    for n in (0, 1, 7, 1000, 16000):
        for world in (1, 2, 3, 4, 8):
            rs = [shard(n, world, r) for r in range(world)]
            got = [i for r in rs for i in r]
            assert got == list(range(n))
            sizes = [len(r) for r in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(10, 2, 2)


def test_digest_is_bitwise():
    a = np.random.default_rng(0).random((5, 7)).astype(np.float32)
    b = a.copy()
    assert window_digest(a) == window_digest(b)
    b[2, 3] = np.nextafter(b[2, 3], np.float32(2))
    assert window_digest(a) != window_digest(b)


def test_two_rank_gloo_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        rank, merged, t = q.get(timeout=240)
        res[rank] = (merged, t)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    merged0, t0 = res[0]
    assert res[1][0] is None
    assert t0 == 11.0 and res[1][1] == 11.0          # max over ranks, on every rank
    single = {i: window_digest(s) for i, s in enumerate(_surfaces(0, N_WIN))}
    assert merged0 == single
