#!/usr/bin/env python
"""Benchmark of the batched IEDS build (BASELINE.json metric: IEDS surfaces/s and Mev/s at
1280x720, % of HBM peak).

One "step" = the whole hot path (scatter -> denoise -> fill -> exact EDT -> Eq. (1)) over one
batch of synthetic windows already resident in HBM: workload C3 (1280x720 Gen4-like, 1000
windows x 75k events per GPU; N_d=2, N_f=3, d_sat=6).  Multi-GPU: one
process per GPU (torchrun), each rank processes its own 1000 distinct windows (weak scaling,
windows are independent: no collective in the data path); timing = max over ranks.
--config C4 is BASELINE's sharded config instead: 16,000 windows in total split across the
ranks (strong scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3]

--impl reference times the CPU oracle (the reference arm of this tier) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth.events import WORKLOADS, batch_events  # noqa: E402


def _load_multi():
    """paper_2112_10591_b200/multi.py loaded by path: importing the package would map
    libieds.so, and the reference arm must not load the product's native code."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "_ieds_multi", os.path.join(ROOT, "paper_2112_10591_b200", "multi.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


multi = _load_multi()
shard = multi.shard

EDT_KERNEL_NAME = "window_kernel<C> (a4 EDT, saturation-aware register window + a5 surface)"
METRIC = "IEDS surfaces/sec and Mev/s at 1280x720 (1/2/4/8 B200), % HBM peak"
UNIT = "surfaces/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy test)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_per_launch(override, windows_per_launch):
    """dram read+write bytes per launch of the dominant kernel from the committed ncu capture
    (profiles/*_traffic.json, scaled to this run's windows per launch), or None."""
    if override is not None:
        return override
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    if not files:
        return None
    try:
        with open(files[-1]) as f:
            t = json.load(f)
        return t["dram_bytes_per_launch"] / t["windows_per_launch"] * windows_per_launch
    except Exception:
        return None


# ------------------------------------------------------------------------------- inputs

def _gen_part(args):
    name, k0, n = args
    wl = WORKLOADS[name]
    return batch_events(wl.scene, wl.seed, k0, n)


def generate(name: str, k0: int, n: int, procs: int | None = None):
    """Windows k0..k0+n-1 of workload `name` as CSR, generated on a process pool."""
    import multiprocessing as mp

    procs = procs or max(1, min(len(os.sched_getaffinity(0)), 32))
    per = max(1, math.ceil(n / (procs * 4)))
    parts = [(name, k0 + i, min(per, n - i)) for i in range(0, n, per)]
    if procs == 1 or len(parts) == 1:
        res = [_gen_part(p) for p in parts]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_gen_part, parts)
    xy = np.concatenate([r[0] for r in res])
    off = np.zeros(n + 1, np.int64)
    pos, i = 0, 0
    for r in res:
        m = len(r[1]) - 1
        off[i + 1:i + m + 1] = r[1][1:] + pos
        pos += len(r[0])
        i += m
    return xy, off


# ------------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
                pw.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(pw) if pw else None}


# ------------------------------------------------------------------------------- oracle baseline

def _oracle_windows(args):
    name, k0, n = args
    import oracle

    wl = WORKLOADS[name]
    c = wl.scene
    xy, off = batch_events(c, wl.seed, k0, n)
    a = oracle.alpha_from_dsat(wl.d_sat)
    t = time.perf_counter()
    for b in range(n):
        oracle.build_window(xy[off[b]:off[b + 1]], c.width, c.height, wl.n_d, wl.n_f, a, want=("S",))
    return time.perf_counter() - t


def oracle_rate(name: str, n_windows: int, cores: int, pool=None):
    """Time the oracle (as it stands) on `n_windows` windows spread over `cores` processes.
    Event generation happens inside the workers before their clock starts."""
    import multiprocessing as mp

    per = max(1, n_windows // cores)
    jobs = [(name, 7919 * i, per) for i in range(cores)]
    own = pool is None
    if own:
        pool = mp.get_context("fork").Pool(cores)
    t0 = time.perf_counter()
    per_times = pool.map(_oracle_windows, jobs)
    wall = time.perf_counter() - t0
    if own:
        pool.close()
        pool.join()
    done = per * cores
    # the workers' compute time excludes their generation time
    busy = max(per_times)
    return done / busy, done, wall


# ------------------------------------------------------------------------------- arms

def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.lower().startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def resolve_config(args, world: int) -> str:
    """BASELINE.json's metric config: C3 (configs[2], 1000 windows) on one GPU; C4 (configs[3],
    16,000 windows sharded across the ranks) when N > 1.  --config overrides."""
    if args.config:
        return args.config
    return "C4" if world > 1 else "C3"


def workload_config(name: str, world: int, rank: int, windows: int = 0, events_per_gpu=None) -> dict:
    """The line's `config` for workload `name` at this world size: the same dict in both arms, so
    the reference arm reports exactly our arm's config (its bounded per-step sample is stated in
    its cpu_baseline.sample and reference_windows_per_step)."""
    wl = WORKLOADS[name]
    c = wl.scene
    strong = name == "C4"
    if strong:
        total = windows or wl.n_windows
        nwin = len(shard(total, world, rank))
    else:
        nwin = windows or wl.n_windows
        total = nwin * world
    n_ev = events_per_gpu if events_per_gpu is not None else c.events_per_window * nwin
    return {"workload": (f"{wl.name}: {c.width}x{c.height} Gen4-like, {total} windows sharded over {world} GPU(s), "
                         if strong else f"{wl.name}: {c.width}x{c.height} Gen4-like, {nwin} windows per GPU, ")
                        + f"{c.events_per_window} events per window",
            "windows_total": total, "windows_per_gpu": nwin, "events_per_gpu": int(n_ev), "width": c.width,
            "height": c.height, "n_d": wl.n_d, "n_f": wl.n_f, "d_sat": wl.d_sat,
            "alpha": wl.d_sat / math.log(255.0),   # Eq. (2)-(3)
            "l2": "inputs+outputs larger than L2 (events %.0f MB, surfaces %.0f MB per step)" % (
                4 * n_ev / 1e6, 4 * c.width * c.height * nwin / 1e6)}


_REF_EVENTS = []   # the reference arm's pre-generated windows (inherited by the forked workers)


def _ref_window(i):
    import oracle

    xy, name = _REF_EVENTS[i]
    wl = WORKLOADS[name]
    c = wl.scene
    oracle.build_window(xy, c.width, c.height, wl.n_d, wl.n_f, oracle.alpha_from_dsat(wl.d_sat), want=("S",))
    return i


def run_reference(args):
    """This tier's reference arm: the fp64 C oracle as it stands, on the host cores.  Each step
    is one batch of `cores` distinct windows of the same workload as our arm (one per worker
    process); events are generated before timing, so value = windows per step / ms_per_step
    over exactly the timed region.  Under torchrun rank 0 alone runs it."""
    world, rank, local = dist_setup()
    if rank != 0:
        return 0
    import multiprocessing as mp

    name = resolve_config(args, world)
    wl = WORKLOADS[name]
    c = wl.scene
    cores = len(os.sched_getaffinity(0))
    per_step = cores
    nsteps = args.warmup + args.steps
    xy, off = generate(name, 0, per_step * nsteps)   # distinct windows for every step (untimed)
    _REF_EVENTS.clear()
    _REF_EVENTS.extend((xy[off[b]:off[b + 1]], name) for b in range(len(off) - 1))
    pool = mp.get_context("fork").Pool(cores)
    walls = []
    for s in range(nsteps):
        t0 = time.perf_counter()
        pool.map(_ref_window, range(s * per_step, (s + 1) * per_step), chunksize=1)
        if s >= args.warmup:
            walls.append(time.perf_counter() - t0)
    pool.close()
    pool.join()
    ms = 1e3 * statistics.median(walls)
    value = per_step / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if name == "C4" else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_config(name, world, 0, args.windows),
        "reference_windows_per_step": per_step,
        "mev_per_s": value * c.events_per_window / 1e6,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "cpu": cpu_model(), "kind": "oracle",
                         "sample": f"each step: {per_step} distinct windows of {wl.name}, one process per core, "
                                   "C oracle (fp64) as it stands; value = windows per step / median step wall time"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "repo_native_libs_mapped": repo_libs_mapped(),
    }
    print(json.dumps(line), flush=True)
    return 0


def repo_libs_mapped() -> list[str]:
    """Shared objects under this repo mapped into this process (the reference arm must show no
    libieds.so: it runs the oracle only, in forked workers)."""
    try:
        with open("/proc/self/maps") as f:
            paths = {ln.split()[-1] for ln in f if ln.rstrip().endswith(".so") or ".so." in ln}
    except OSError:
        return []
    return sorted(os.path.relpath(p, ROOT) for p in paths if p.startswith(ROOT))


def cycled_batch(name, k0, nwin, pool, dev):
    """Device CSR batch of nwin windows of `name` whose events cycle through `pool` distinct
    generated windows k0 .. k0+pool-1 (window i carries the events of window k0 + i % pool).
    Used where generating every window on the host would dominate the run (C5: ~120 ms per
    window); the pool's events (>= 150 MB) exceed the 126 MB L2, so a repeat is an HBM read."""
    import torch

    pool = max(1, min(pool, nwin))
    pxy, poff = generate(name, k0, pool)
    lens = np.diff(poff)
    reps, rem = divmod(nwin, pool)
    txy_pool = torch.from_numpy(pxy.view(np.int32)).to(dev)
    parts = [txy_pool] * reps + ([txy_pool[:int(poff[rem])]] if rem else [])
    txy = torch.cat(parts) if len(parts) > 1 else parts[0].clone()
    off = np.zeros(nwin + 1, np.int64)
    off[1:] = np.cumsum(np.concatenate([np.tile(lens, reps), lens[:rem]]))
    return txy, torch.from_numpy(off).to(dev), int(off[-1]), pool


def run_weak_c3(args, dev, stream, world, local, peak, txy, off, n):
    """Weak scaling at N > 1: each rank builds the first n windows of its resident C4 shard (C3's
    per-GPU batch shape), timed like the main line, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2112_10591_b200 as ieds

    wl = WORKLOADS["C3"]
    c = wl.scene
    toff = torch.from_numpy(np.ascontiguousarray(off[:n + 1])).to(dev)
    S = torch.empty((n, c.height, c.width), dtype=torch.float32, device=dev)
    with ieds.Builder(c.width, c.height, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=local) as bld:
        for _ in range(max(1, args.warmup)):
            bld.build_batch(txy, toff, S)
        ksteps = max(1, min(args.steps, 10))
        dist.barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ksteps):
            bld.build_batch(txy, toff, S)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        bld.sync()
    tm = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ms = float(tm.item()) / ksteps
    del S
    return {"workload": f"C3 per GPU: {n} windows on each of {world} GPUs (first windows of each rank's C4 shard)",
            "windows_total": n * world, "windows_per_gpu": n, "scaling": "weak",
            "value": n * world / (ms / 1e3), "unit": "surfaces/s", "ms_per_step": ms, "steps": ksteps}


def run_c4_single(args, dev, stream, peak, xy, off, total=16000):
    """C4 (BASELINE configs[3]: 16,000 1280x720 windows) on one GPU -- the R = 1 point of its
    strong-scaling curve -- with the events of the 1000 resident C3 windows cycled 16 times."""
    import torch

    import paper_2112_10591_b200 as ieds

    wl = WORKLOADS["C4"]
    c = wl.scene
    pool = len(off) - 1
    reps, rem = divmod(total, pool)
    txy_pool = torch.from_numpy(xy.view(np.int32)).to(dev)
    txy = torch.cat([txy_pool] * reps + ([txy_pool[:int(off[rem])]] if rem else []))
    lens = np.diff(off)
    o = np.zeros(total + 1, np.int64)
    o[1:] = np.cumsum(np.concatenate([np.tile(lens, reps), lens[:rem]]))
    toff = torch.from_numpy(o).to(dev)
    S = torch.empty((total, c.height, c.width), dtype=torch.float32, device=dev)
    with ieds.Builder(c.width, c.height, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=dev.index) as bld:
        for _ in range(max(1, args.warmup)):
            bld.build_batch(txy, toff, S)
        ksteps = max(1, min(args.steps, 5))
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ksteps):
            bld.build_batch(txy, toff, S)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        bld.sync()
    ms = e0.elapsed_time(e1) / ksteps
    n_ev = int(o[-1])
    bytes_step = 4.0 * n_ev + 4.0 * c.width * c.height * total + 8.0 * (total + 1)
    del S, txy, toff
    return {"workload": f"C4: 1280x720, {total} windows on 1 GPU (R = 1), 75000 events per window",
            "windows_total": total, "distinct_windows": pool, "scaling": "strong", "value": total / (ms / 1e3),
            "unit": "surfaces/s", "ms_per_step": ms, "steps": ksteps,
            "hbm_frac_path": bytes_step / (ms / 1e3) / 1e9 / peak,
            "note": "the R = 1 baseline of BASELINE's C4 strong scaling; N > 1 runs report C4 as the main line"}


def run_config_brief(args, name, dev, stream, world, local, peak, nwin=None, total=None, pool=None):
    """Another §8(d) workload (C2: 346x260; C5: the 1280x720 dense burst) on the same device:
    surfaces/s and the whole-path HBM fraction over a few steps, inputs resident (not the
    metric's config).  nwin = windows per GPU (weak scaling), or total = windows sharded across
    the ranks (strong scaling, BASELINE's C5 shape: 16k windows on the 8 GPUs); pool = distinct
    generated windows per rank, cycled (cycled_batch)."""
    import torch
    import torch.distributed as dist

    import paper_2112_10591_b200 as ieds

    wl = WORKLOADS[name]
    c = wl.scene
    rank = int(os.environ.get("RANK", "0"))
    if total:
        rng = shard(total, world, rank)
        k0, nwin = rng.start, len(rng)
    else:
        nwin = nwin or wl.n_windows
        k0 = rank * nwin
    if pool:
        txy, toff, n_ev, npool = cycled_batch(name, k0, nwin, pool, dev)
    else:
        xy, off = generate(name, k0, nwin)
        txy = torch.from_numpy(xy.view(np.int32)).to(dev)
        toff = torch.from_numpy(off).to(dev)
        n_ev, npool = int(off[-1]), nwin
        del xy
    S = torch.empty((nwin, c.height, c.width), dtype=torch.float32, device=dev)
    bld = ieds.Builder(c.width, c.height, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=local)
    for _ in range(max(1, args.warmup)):
        bld.build_batch(txy, toff, S)
    ksteps = max(1, min(args.steps, 10))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(ksteps):
        bld.build_batch(txy, toff, S)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    bld.sync()
    bld.close()
    tm = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ms = float(tm.item()) / ksteps
    bytes_step = 4.0 * n_ev + 4.0 * c.width * c.height * nwin + 8.0 * (nwin + 1)
    del S, txy, toff
    all_windows = total if total else nwin * max(1, world)
    return {"workload": f"{name}: {c.width}x{c.height}, " + (
                f"{total} windows sharded over {world} GPU(s) ({nwin} on rank {rank})" if total else
                f"{nwin} windows per GPU") + f" x {c.events_per_window} events",
            "windows_total": all_windows, "windows_per_gpu": nwin, "distinct_windows_per_gpu": npool,
            "scaling": "strong" if total else "weak",
            "value": all_windows / (ms / 1e3), "unit": "surfaces/s", "ms_per_step": ms, "steps": ksteps,
            "mev_per_s": all_windows * (n_ev / nwin) / (ms / 1e3) / 1e6,
            "hbm_frac_path": bytes_step / (ms / 1e3) / 1e9 / peak,
            "note": "SURVEY §8(d) ceiling at the measured peak (4 B/event + 4 B/px): "
                    f"{peak * 1e9 / (bytes_step / nwin) / 1e6:.2f} M surfaces/s per GPU"}


def run_f2_windowing(args, dev, stream, world, local, wl, off, peak):
    """Row f2: on-device Delta-T windowing (ieds_window_offsets) of the C3 stream: 1000 windows of
    15 ms over 75 M time-ordered timestamps resident on the device.  The kernel binary-searches
    each window start and checks the whole stream's order, so its algorithmic bytes are 8 B per
    event (+ 8 B per offset).  The timestamps are synthetic, laid out so that the windows are
    exactly the C3 batch's CSR windows, which the result is checked against."""
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_2112_10591_b200 as ieds
    from paper_2112_10591_b200._lib import load

    dt = 15000
    nwin = len(off) - 1
    counts = np.diff(off)
    k = np.repeat(np.arange(nwin, dtype=np.int64), counts)
    j = np.arange(int(off[-1]), dtype=np.int64) - np.repeat(off[:-1], counts)
    t = k * dt + (j * dt) // np.maximum(1, counts)[k]
    tt = torch.from_numpy(t).to(dev)
    del k, j, t
    out = torch.empty(nwin + 1, dtype=torch.int64, device=dev)
    bld = ieds.Builder(wl.scene.width, wl.scene.height, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=local)
    lib = load()
    n = tt.numel()

    def call():
        rc = lib.ieds_window_offsets(bld._h, ctypes.c_void_p(tt.data_ptr()), n, 0, dt, nwin,
                                     ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream.cuda_stream))
        assert rc == 0, rc

    for _ in range(max(1, args.warmup)):
        call()
    torch.cuda.synchronize(dev)
    ok = bool(torch.equal(out.cpu(), torch.from_numpy(off)))
    ksteps = max(1, min(args.steps, 10))
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(ksteps):
        call()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    bld.sync()
    bld.close()
    tm = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ms = float(tm.item()) / ksteps
    gbs = (8.0 * n + 8.0 * (nwin + 1)) / (ms / 1e3) / 1e9
    del tt, out
    return {"metric": "Delta-T windowing of a resident event stream (ieds_window_offsets)",
            "value": n * max(1, world) / (ms / 1e3) / 1e6, "unit": "Mev/s", "ms_per_step": ms, "steps": ksteps,
            "windows": nwin, "events": n, "hbm_gbs": gbs, "hbm_frac": gbs / peak, "offsets_match_batch": ok,
            "note": "algorithmic bytes 8 B/event (the order check reads every timestamp) + 8 B/offset"}


def run_f2_stream(args, dev, world, local, wl, xy, off, nwin=200, chunk_events=1_000_000):
    """Row f2 streaming ingest (ieds_stream_push, Fig. 1 / P:117): the first nwin C3 windows as a
    live time-ordered stream, pushed from pinned host memory in chunks of chunk_events events
    (~13 windows; the open window carried across pushes on the device), surfaces returned into a
    pinned host buffer as windows close.  Host in, host out, like e2e: PCIe-bound (3.7 MB of
    surface per window)."""
    import ctypes

    import torch

    import paper_2112_10591_b200 as ieds
    from paper_2112_10591_b200._lib import load

    c = wl.scene
    dt = 15000
    nwin = min(nwin, len(off) - 1)
    counts = np.diff(off[:nwin + 1])
    n = int(off[nwin])
    k = np.repeat(np.arange(nwin, dtype=np.int64), counts)
    j = np.arange(n, dtype=np.int64) - np.repeat(off[:nwin], counts)
    t_pin = torch.from_numpy(np.ascontiguousarray(k * dt + (j * dt) // np.maximum(1, counts)[k])).pin_memory()
    ev_pin = torch.from_numpy(np.ascontiguousarray(xy[:n]).view(np.int32)).pin_memory()
    t, ev = t_pin.numpy(), ev_pin.numpy()
    lib = load()
    cap = chunk_events // 10_000 + 4   # windows one push can close (C3 windows hold ~75k events)
    hS = torch.empty((cap, c.height, c.width), dtype=torch.float32).pin_memory()
    got = ctypes.c_int32()
    bld = ieds.Builder(c.width, c.height, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=local)

    st = bld.stream(dt)   # created once: its device buffers are allocated outside the timed region

    def run_once():   # one whole stream: push every chunk, then flush (which resets the stream)
        done = 0
        for a in range(0, n, chunk_events):
            b = min(n, a + chunk_events)
            rc = lib.ieds_stream_push(st._s, t[a:].ctypes.data_as(ctypes.c_void_p),
                                      ev[a:].ctypes.data_as(ctypes.c_void_p), b - a,
                                      ctypes.c_void_p(hS.data_ptr()), cap, ctypes.byref(got))
            assert rc == 0, rc
            done += got.value
        rc = lib.ieds_stream_flush(st._s, ctypes.c_void_p(hS.data_ptr()), cap, ctypes.byref(got))
        assert rc == 0, rc
        return done + got.value

    run_once()
    t0 = time.perf_counter()
    done = run_once()
    el = time.perf_counter() - t0
    st.close()
    bld.close()
    return {"metric": "streaming ingest windows/s (ieds_stream_push: host (t, xy) chunks in, host surfaces out)",
            "value": done / el, "unit": "windows/s", "windows": done, "events": n, "chunk_events": chunk_events,
            "mev_per_s": n / el / 1e6, "ms_per_window": 1e3 * el / done,
            "note": "wall clock; the first C3 windows as one time-ordered stream (15 ms windows), pushed in fixed-size "
                    "chunks that cut windows at arbitrary points; surfaces into a pinned host buffer; PCIe-bound like e2e"}


def run_f4_pipeline(args, dev, world, local, wl, xy, off, nwin=60, chunk_events=1_000_000):
    """The Fig. 1 pipeline (ieds_pipeline_push): the first nwin C3 windows as one live
    stream pushed from pinned host memory in chunks; per closed window its flow (float32 [H][W][2])
    and valid mask come back into pinned host buffers.  Surfaces of later windows are built while
    earlier windows' flow runs; each window's flow is copied out while the next is computed."""
    import ctypes

    import torch

    import paper_2112_10591_b200 as ieds
    from paper_2112_10591_b200._lib import load

    c = wl.scene
    dt = 15000
    nwin = min(nwin, len(off) - 1)
    counts = np.diff(off[:nwin + 1])
    n = int(off[nwin])
    k = np.repeat(np.arange(nwin, dtype=np.int64), counts)
    j = np.arange(n, dtype=np.int64) - np.repeat(off[:nwin], counts)
    t = torch.from_numpy(np.ascontiguousarray(k * dt + (j * dt) // np.maximum(1, counts)[k])).pin_memory().numpy()
    ev = torch.from_numpy(np.ascontiguousarray(xy[:n]).view(np.int32)).pin_memory().numpy()
    cap = chunk_events // 10_000 + 4
    hF = torch.empty((cap, c.height, c.width, 2), dtype=torch.float32).pin_memory()
    hV = torch.empty((cap, c.height, c.width), dtype=torch.uint8).pin_memory()
    lib = load()
    got = ctypes.c_int32()
    bld = ieds.Builder(c.width, c.height, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=local)
    fe = ieds.FlowEstimator(c.width, c.height, device=local)
    pl = ieds.Pipeline(bld, fe, dt)   # device buffers allocated here, outside the timed region
    outs = (ctypes.c_void_p(hF.data_ptr()), ctypes.c_void_p(hV.data_ptr()), None)

    def run_once():
        done = 0
        for a in range(0, n, chunk_events):
            b = min(n, a + chunk_events)
            rc = lib.ieds_pipeline_push(pl._p, t[a:].ctypes.data_as(ctypes.c_void_p),
                                        ev[a:].ctypes.data_as(ctypes.c_void_p), b - a, *outs, cap, ctypes.byref(got))
            assert rc == 0, rc
            done += got.value
        rc = lib.ieds_pipeline_flush(pl._p, *outs, cap, ctypes.byref(got))
        assert rc == 0, rc
        return done + got.value

    run_once()
    t0 = time.perf_counter()
    done = run_once()
    el = time.perf_counter() - t0
    pl.close()
    fe.close()
    bld.close()
    return {"metric": "pipeline windows/s (ieds_pipeline_push: host events in, flow + valid mask out per window)",
            "value": done / el, "unit": "windows/s", "windows": done, "events": n, "chunk_events": chunk_events,
            "ms_per_window": 1e3 * el / done,
            "note": "wall clock; events -> surfaces -> 3-level flow (P:260 settings) -> host, 8.3 MB out per window "
                    "(flow + mask); the build of later windows overlaps earlier windows' flow, and each flow's "
                    "copy-out the next flow step"}


def run_f4(args, dev, stream, world, local, wl):
    """Row f4: the stateful flow consumer (ieds_flow_step, reading R21) at the
    paper's HD settings (3 levels, weight 500, 20 sweeps) over the surfaces and
    denoised edge bits of consecutive C3 windows (a moving scene), built on the device by the
    hot path.  Sequential by nature: windows/s of one stream; plus one window's surface + flow
    latency (the paper's whole-pipeline real-time figure)."""
    import torch

    import paper_2112_10591_b200 as ieds
    from synth.events import batch_events

    c = wl.scene
    W, H = c.width, c.height
    n = 24
    rank = int(os.environ.get("RANK", "0"))
    xy, off = batch_events(c, wl.seed, 5000 + rank * n, n)
    txy = torch.from_numpy(xy.view(np.int32)).to(dev)
    toff = torch.from_numpy(off).to(dev)
    NW = (W + 31) // 32
    bld = ieds.Builder(W, H, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=local)
    S = torch.empty((n, H, W), dtype=torch.float32, device=dev)
    Ed = torch.empty((n, H, NW), dtype=torch.int32, device=dev)
    bld.build_batch(txy, toff, S, denoised_bits=Ed)
    bld.sync()
    fe = ieds.FlowEstimator(W, H, device=local)
    flow = torch.empty((H, W, 2), dtype=torch.float32, device=dev)
    for k in range(4):   # warm-up (captures both graph parities)
        fe.step(S[k], Ed[k], out=flow)
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(4, n):
        fe.step(S[k], Ed[k], out=flow)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / (n - 4)
    # one window end to end on the device: surface (frame + window kernels) then flow
    lat = []
    one_off = torch.tensor([0, int(off[1] - off[0])], dtype=torch.int64, device=dev)
    for k in range(6):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        bld.build_batch(txy[:int(off[1])], one_off, S[:1], denoised_bits=Ed[:1])
        fe.step(S[0], Ed[0], out=flow)
        b.record(stream)
        torch.cuda.synchronize(dev)
        lat.append(a.elapsed_time(b))
    bld.sync()
    launches = fe.launches_per_step()
    fe.close()
    bld.close()
    return {"metric": "flow windows/s (3-level update-prediction flow, P:241-248, one sequence)",
            "value": 1e3 / ms, "unit": "windows/s", "ms_per_window": ms, "windows_timed": n - 4,
            "launches_per_step": launches, "graph": "per-level kernels (prep, grad, 4 Jacobi sweeps per halo-tiled launch; the coarse levels' sweeps in one cooperative launch) replayed from one CUDA graph per step",
            "surface_plus_flow_ms_p50": float(np.median(lat[1:])),
            "note": "paper: 16.88 ms per 1280x720 window for the whole pipeline incl. its third-party flow on an "
                    "RTX 5000 (P:555); this estimator is the R21 substitute, so the timing is context, not parity"}


def run_f3(args, dev, stream, world, local, peak):
    """Row f3: ieds_fwl_batch over C3-geometry windows of a scene moving under a known dense
    affine flow (synth/flowscene.py), inputs resident on the device.  Algorithmic bytes per
    event: 4 (xy) + 8 (t) + 1 (p) + 8 (the flow gathered at the event pixel)."""
    import torch
    import torch.distributed as dist

    import paper_2112_10591_b200 as ieds
    from synth.flowscene import F3_SCENE, flow_batch

    cfg = F3_SCENE
    nwin = max(1, args.f3_windows)
    rank = int(os.environ.get("RANK", "0"))
    xy, t, p, off, flows, _fl, t_ref = flow_batch(cfg, 3, rank * nwin, nwin)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    txy, tt, tp, toff = T(xy.view(np.int32)), T(t), T(p), T(off)
    tflow, tref = T(flows), T(t_ref)
    del flows
    bld = ieds.Builder(cfg.width, cfg.height, 1, 4, device=local)
    for _ in range(max(1, args.warmup)):
        r = bld.fwl_batch(txy, tt, tp, toff, tflow, tref, cfg.dt_us)
    bld.sync()
    ksteps = max(1, min(args.steps, 10))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(ksteps):
        r = bld.fwl_batch(txy, tt, tp, toff, tflow, tref, cfg.dt_us)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    bld.sync()
    fwl_mean = float(r["fwl"].mean().item())
    bld.close()
    tm = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ms = float(tm.item()) / ksteps
    n_ev = int(off[-1])
    bytes_alg = 21.0 * n_ev + 8.0 * (nwin + 1) + 16.0 * nwin
    ceil = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_f3_atomic_ceiling.json")) as f:
            ceil = json.load(f)["events_per_s"]
    except Exception:
        pass
    out = {"metric": "FWL windows/s (flow-compensated event image + variance ratio, P:293-297)",
           "value": nwin * max(1, world) / (ms / 1e3), "unit": "windows/s", "ms_per_step": ms, "steps": ksteps,
           "windows": nwin, "mev_per_s": n_ev * max(1, world) / (ms / 1e3) / 1e6,
           "hbm_gbs": bytes_alg / (ms / 1e3) / 1e9, "hbm_frac": bytes_alg / (ms / 1e3) / 1e9 / peak,
           "fwl_mean": fwl_mean,
           "atomic_ceiling": None if ceil is None else {
               "events_per_s": ceil, "frac_whole_call": n_ev * max(1, world) / (ms / 1e3) / ceil,
               "source": "profiles/r02_f3_atomic_ceiling.json (tools/atomic_ceiling.cu: the splat's 1 int32 + 4 fp64 "
                         "atomics per event with no arithmetic); the splat kernel alone runs at ~0.97 of it, the "
                         "whole call adds the scratch re-zeroing and the finalize"},
           "note": "algorithmic bytes 21 B/event (xy, t, p, flow gather); the I_comp/I_uncomp images are "
                   "L2 scratch (12 B/px, 16 windows per pass) that is never read back: sum I and sum I^2 come "
                   "from the atomics' old values; the bound is the L2 atomic rate, not HBM"}
    if world == 1 and not args.no_cpu_baseline:   # the oracle is timed at N = 1 only
        import time as _time

        import oracle

        t0 = _time.perf_counter()
        nsamp = min(4, nwin)
        for b in range(nsamp):
            sl = slice(off[b], off[b + 1])
            oracle.fwl(xy[sl], t[sl], p[sl], cfg.width, cfg.height,
                       flow_batch(cfg, 3, rank * nwin + b, 1)[4][0], t_ref[b], cfg.dt_us)
        dt_o = _time.perf_counter() - t0
        out["cpu_baseline"] = {"value": nsamp / dt_o, "unit": "windows/s", "cores": 1, "kind": "oracle",
                               "sample": f"{nsamp} windows, one core, C oracle fp64 (incl. regenerating each field)"}
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_setup()
    dist_info = None
    # IEDS_BENCH_SHARE_GPU=1 (code-path check only, never a measurement): every rank on cuda:0
    # with the gloo backend, so the N > 1 path can be exercised on a one-GPU box
    share = os.environ.get("IEDS_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    if world > 1:
        # NCCL's own communicator-init log (stderr) shows the N ranks and their transports
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()   # forces the communicator up before anything is timed
        ws = dist.get_world_size()
        print(f"[bench rank {rank}] process group up: backend={dist.get_backend()} world_size={ws} "
              f"device=cuda:{local} ({torch.cuda.get_device_name(local)})", file=sys.stderr, flush=True)
        if ws != world:
            raise RuntimeError(f"WORLD_SIZE {world} but the process group has {ws} ranks")
        try:
            nccl_v = ".".join(str(x) for x in torch.cuda.nccl.version())
        except Exception:
            nccl_v = None
        dist_info = {"backend": dist.get_backend(), "world_size": ws, "nccl_version": nccl_v,
                     "shared_gpu_code_path_check": share,
                     "collectives": "barrier + all_reduce(MAX) of elapsed ms + gather of sampled window digests; "
                                    "none in the data path (windows are independent, P:113, S:198)"}
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2112_10591_b200 as ieds

    if args.gpus > 1 and world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    name = resolve_config(args, world)
    wl = WORKLOADS[name]
    c = wl.scene
    W, H = c.width, c.height
    # C4 (BASELINE configs[3]) is a fixed total of windows sharded across the ranks (strong
    # scaling); every other config gives each rank its own nwin distinct windows (weak scaling)
    strong = name == "C4"
    if strong:
        total_windows = args.windows or wl.n_windows
        rng = shard(total_windows, world, rank)
        k0, nwin = rng.start, len(rng)
    else:
        nwin = args.windows or wl.n_windows
        rng = shard(nwin * world, world, rank)
        k0 = rng.start
        total_windows = nwin * world
    xy, off = generate(name, k0, nwin)
    n_ev = len(xy)
    txy = torch.from_numpy(xy.view(np.int32)).to(dev)
    toff = torch.from_numpy(off).to(dev)
    S = torch.empty((nwin, H, W), dtype=torch.float32, device=dev)
    bld = ieds.Builder(W, H, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=local, chunk_windows=args.chunk)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        bld.build_batch(txy, toff, S)
    bld.sync()
    torch.cuda.synchronize(dev)

    launches_per_step = bld.launches_per_batch(nwin)
    bld.profile(True)
    bld.profile_read()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        bld.build_batch(txy, toff, S)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    prof = bld.profile_read()
    bld.profile(False)
    bld.sync()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = total_windows / (ms_step / 1e3)

    # roofline of the dominant kernel (EDT + surface, a4-a5): algorithmic bytes = 4 B/px fp32 surface
    peak, peak_src = peaks()
    edt_ms, edt_n = prof["edt"]
    fr_ms, fr_n = prof["frame"]
    chunk_windows = math.ceil(nwin / max(1, edt_n // max(1, args.steps)))
    edt_avg_ms = edt_ms / max(1, edt_n)
    edt_bytes_per_launch = 4.0 * W * H * (nwin / max(1, edt_n // args.steps))
    edt_gbs = edt_bytes_per_launch / (edt_avg_ms / 1e3) / 1e9
    fr_avg_ms = fr_ms / max(1, fr_n)
    fr_bytes_per_launch = 4.0 * n_ev / max(1, fr_n // args.steps)
    path_bytes = 4.0 * n_ev + 4.0 * W * H * nwin + 8.0 * (nwin + 1)
    path_gbs = path_bytes / (ms_step / 1e3) / 1e9

    # end to end through the C ABI with host buffers (copies inside the timed region)
    # (at N > 1 on the first e2e_windows windows of each rank's shard: pinned host buffers for a
    # whole 16k-window C4 shard would pin ~60 GB of host memory across the ranks)
    e2e = None
    if not args.no_e2e:
        en = min(nwin, args.e2e_windows) if world > 1 else nwin
        hxy = torch.from_numpy(xy[:int(off[en])].view(np.int32)).pin_memory()
        hoff = torch.from_numpy(off[:en + 1]).pin_memory()
        hS = torch.empty((en, H, W), dtype=torch.float32).pin_memory()
        nxy, noff, nS = hxy.numpy().view(np.uint32), hoff.numpy(), hS.numpy()
        bld.build_batch_host(nxy, noff, nS)
        esteps = max(1, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(esteps):
            bld.build_batch_host(nxy, noff, nS)
        el = (time.perf_counter() - t0) / esteps
        te = torch.tensor([el], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        el = float(te.item())
        e2e = {"value": en * world / el, "unit": UNIT, "h2d_bytes_per_step": int(4 * off[en] + 8 * (en + 1)),
               "d2h_bytes_per_step": int(4 * W * H * en), "steps": esteps, "windows_per_rank": en,
               "note": "ieds_build_batch_host: pinned host events in, pinned host surfaces out, per rank; "
                       "wall clock, max over ranks"}
        del hxy, hoff, hS

    bld.close()

    # cross-rank parity: digests of sampled windows of every rank's shard (from the timed run's
    # surfaces), gathered to rank 0 and compared with rank 0's own recompute of those windows
    # from regenerated events in a separate batch -- a sharded run must reproduce the
    # single-rank results bit for bit (windows are pure functions of their events)
    def recompute(indices):
        out = {}
        with ieds.Builder(W, H, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=local) as br:
            for i in indices:
                rxy, roff = generate(name, i, 1, procs=1)
                rS = br.build_batch(torch.from_numpy(rxy.view(np.int32)).to(dev), torch.from_numpy(roff).to(dev))
                br.sync()
                out[i] = multi.window_digest(rS[0].cpu().numpy())
        return out

    mine = {i: multi.window_digest(S[i - k0].cpu().numpy()) for i in multi.sample_windows(rng, 3)}
    xcheck = multi.cross_rank_check(mine, recompute)
    if xcheck is not None and not xcheck["match"]:
        print(f"cross-rank digest mismatch: {xcheck}", file=sys.stderr, flush=True)

    # the uncapped exact-EDT kernel on the same inputs (reported beside the headline path)
    exact = None
    if not args.no_exact:
        bx = ieds.Builder(W, H, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=local, exact_edt=True)
        for _ in range(max(1, args.warmup)):
            bx.build_batch(txy, toff, S)
        torch.cuda.synchronize(dev)
        bx.profile(True)
        bx.profile_read()
        ksteps = max(1, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        x0 = torch.cuda.Event(enable_timing=True)
        x1 = torch.cuda.Event(enable_timing=True)
        x0.record(stream)
        for _ in range(ksteps):
            bx.build_batch(txy, toff, S)
        x1.record(stream)
        torch.cuda.synchronize(dev)
        xp = bx.profile_read()
        bx.sync()
        bx.close()
        tx = torch.tensor([x0.elapsed_time(x1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tx, op=dist.ReduceOp.MAX)
        xms = float(tx.item()) / ksteps
        xe_ms, xe_n = xp["edt"]
        xe_avg = xe_ms / max(1, xe_n)
        xe_bytes = 4.0 * W * H * (nwin / max(1, xe_n // ksteps))
        exact = {"value": total_windows / (xms / 1e3), "unit": UNIT, "ms_per_step": xms, "steps": ksteps,
                 "kernel": "edt_kernel (uncapped exact EDT)",
                 "achieved_gbs": xe_bytes / (xe_avg / 1e3) / 1e9, "frac": xe_bytes / (xe_avg / 1e3) / 1e9 / peak,
                 "note": "IEDS_FLAG_EXACT_EDT: D2 exact everywhere (the kernel sqdist requests use)"}
        # the sqdist request itself: surfaces + exact integer D2 written (8 B/px), default handle
        D2 = torch.empty((nwin, H, W), dtype=torch.int32, device=dev)
        bd = ieds.Builder(W, H, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=local)
        for _ in range(max(1, args.warmup)):
            bd.build_batch(txy, toff, S, sqdist=D2)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        x0.record(stream)
        for _ in range(ksteps):
            bd.build_batch(txy, toff, S, sqdist=D2)
        x1.record(stream)
        torch.cuda.synchronize(dev)
        bd.sync()
        bd.close()
        td = torch.tensor([x0.elapsed_time(x1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(td, op=dist.ReduceOp.MAX)
        dms = float(td.item()) / ksteps
        dbytes = 4.0 * n_ev + 8.0 * W * H * nwin
        exact["sqdist"] = {"value": total_windows / (dms / 1e3), "unit": UNIT, "ms_per_step": dms,
                           "path_gbs": dbytes / (dms / 1e3) / 1e9, "path_frac": dbytes / (dms / 1e3) / 1e9 / peak,
                           "note": "build_batch(..., sqdist=): fp32 surface + exact uint32 D2 (4 B/event + 8 B/px)"}
        del D2

    # row f1: the same workload with the epilogue variants (1 or 2 B/px written)
    def time_variant(out, transfer, odt, bpp, label, note, kernel_frac=True):
        Q = torch.empty((nwin, H, W), dtype=odt, device=dev)
        bq = ieds.Builder(W, H, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=local, out=out, transfer=transfer)
        for _ in range(max(1, args.warmup)):
            bq.build_batch(txy, toff, Q)
        torch.cuda.synchronize(dev)
        bq.profile(True)
        bq.profile_read()
        ksteps = max(1, min(args.steps, 10))
        if world > 1:
            dist.barrier()
        q0 = torch.cuda.Event(enable_timing=True)
        q1 = torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        for _ in range(ksteps):
            bq.build_batch(txy, toff, Q)
        q1.record(stream)
        torch.cuda.synchronize(dev)
        qp = bq.profile_read()
        bq.sync()
        bq.close()
        tq = torch.tensor([q0.elapsed_time(q1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tq, op=dist.ReduceOp.MAX)
        qms = float(tq.item()) / ksteps
        path_q = (4.0 * n_ev + bpp * W * H * nwin) / (qms / 1e3) / 1e9
        r = {"variant": label, "value": total_windows / (qms / 1e3), "unit": UNIT, "ms_per_step": qms,
             "steps": ksteps, "path_gbs": path_q, "path_frac": path_q / peak, "note": note}
        if kernel_frac:
            qe_ms, qe_n = qp["edt"]
            q_bytes = bpp * W * H * (nwin / max(1, qe_n // ksteps))
            q_gbs = q_bytes / (qe_ms / max(1, qe_n) / 1e3) / 1e9
            r["window_kernel_gbs"] = q_gbs
            r["window_kernel_frac"] = q_gbs / peak
        del Q
        return r

    f1 = f1_f16 = f1_norm = None
    if not args.no_f1:
        f1 = time_variant("u8", "invexp", torch.uint8, 1.0, "8-bit coded surface q = round(255*S) (P:231)",
                          "algorithmic bytes 4 B/event + 1 B/px; saturation radius C = 8 (q = 255 from D2 >= 46)")
        f1_f16 = time_variant("f16", "invexp", torch.float16, 2.0, "float16 surface (Eq. (1) rounded to nearest even)",
                              "algorithmic bytes 4 B/event + 2 B/px; saturation radius C = 10 (fp16 1.0 from D2 >= 82)")
        f1_norm = time_variant("u8", "log", torch.uint8, 1.0,
                               "8-bit ln(d+1) normalised by the frame maximum (S:254, S:271)",
                               "exact EDT -> D2 scratch -> per-window max -> quantise (fp64 table); "
                               "algorithmic bytes 4 B/event + 1 B/px", kernel_frac=False)

    # row f3: flow-compensated event image + FWL on C3-geometry moving scenes
    # (rows f2-f4 are single-stream / latency measurements: N = 1 only)
    single = world == 1
    f3 = None
    if not args.no_f3 and single:
        f3 = run_f3(args, dev, stream, world, local, peak)

    # the low-resolution config of SURVEY §8(d) (C2: 346x260, 10,000 windows per GPU; 2,000
    # distinct generated windows per GPU, cycled: 160 MB of events)
    c2 = None
    if not args.no_c2 and name != "C2":
        c2 = run_config_brief(args, "C2", dev, stream, world, local, peak, pool=2000)

    # BASELINE's C4 at R = 1 ("16,000 windows ... plus R=1 baseline"): at N = 1 the
    # main line is C3, so the 16,000-window batch is timed here on the one GPU, its events cycling
    # through the 1000 generated C3 windows (300 MB > L2); at N > 1 C4 is the main line itself
    c4_r1 = None
    if not args.no_c4_r1 and world == 1 and name == "C3":
        c4_r1 = run_c4_single(args, dev, stream, peak, xy, off)
    # and at N > 1 the weak-scaling view of the same path: every rank builds 1000 windows of its
    # resident shard (C3's per-GPU batch), value = all ranks' windows / the slowest rank's time
    c3_weak = None
    if world > 1 and name == "C4" and nwin >= 1:
        c3_weak = run_weak_c3(args, dev, stream, world, local, peak, txy, off, min(nwin, 1000))

    # the dense burst config at BASELINE's shape (configs[4]: 300k events per 1280x720 window,
    # fill 13 %; 16,000 windows sharded across the ranks; 256 distinct windows per GPU, cycled)
    c5 = None
    if not args.no_c5 and name != "C5":
        c5 = run_config_brief(args, "C5", dev, stream, world, local, peak, total=args.c5_windows, pool=256)

    # row f4: the flow consumer on consecutive C3 surfaces
    f4 = f4p = None
    if not args.no_f4 and single:
        f4 = run_f4(args, dev, stream, world, local, wl)
        f4p = run_f4_pipeline(args, dev, world, local, wl, xy, off)

    # row f2: on-device windowing of the resident stream, and the streaming ingest from the host
    f2w = f2s = None
    if not args.no_latency and single:
        f2w = run_f2_windowing(args, dev, stream, world, local, wl, off, peak)
        f2s = run_f2_stream(args, dev, world, local, wl, xy, off)

    # row f2: single-window latency (the paper's real-time mode): one window's
    # events -> surface, (a) events resident on the device, (b) through the host-buffer API
    lat = None
    if not args.no_latency and single:
        bl = ieds.Builder(W, H, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=local, chunk_windows=1)
        S1 = torch.empty((1, H, W), dtype=torch.float32, device=dev)
        hS1 = torch.empty((1, H, W), dtype=torch.float32).pin_memory().numpy()
        dev_ms, host_ms, gpu_ms = [], [], []
        for i in range(60):
            k = i % nwin
            o = off[k:k + 2].copy()
            xs = xy[o[0]:o[1]]
            ta = toff[k:k + 2]
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            ev0.record(stream)
            bl.build_batch(txy, ta, S1)
            ev1.record(stream)
            torch.cuda.synchronize(dev)
            dev_ms.append(1e3 * (time.perf_counter() - t0))
            gpu_ms.append(ev0.elapsed_time(ev1))
            t0 = time.perf_counter()
            bl.build_batch_host(xs, o - o[0], hS1)
            host_ms.append(1e3 * (time.perf_counter() - t0))
        # the same call captured once in a CUDA graph (ieds_build_batch enqueues only: no host sync,
        # no allocation) and replayed per window; the window is chosen by a 16-byte device copy of
        # its CSR offsets into the graph's static offsets buffer
        graph_ms = []
        try:
            g_off = toff[0:2].clone()
            cap = torch.cuda.Stream(device=dev)
            cap.wait_stream(stream)
            with torch.cuda.stream(cap):
                bl.build_batch(txy, g_off, S1)   # warm-up on the capture stream
            cap.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=cap):
                bl.build_batch(txy, g_off, S1)
            for i in range(60):
                k = i % nwin
                torch.cuda.synchronize(dev)
                t0 = time.perf_counter()
                g_off.copy_(toff[k:k + 2], non_blocking=True)
                graph.replay()
                torch.cuda.synchronize(dev)
                graph_ms.append(1e3 * (time.perf_counter() - t0))
            bl.sync()
        except Exception as ex:   # report, never fall back
            graph_ms = []
            print(f"graph replay unavailable: {ex}", file=sys.stderr)
        bl.close()
        dev_ms, host_ms, gpu_ms = np.array(dev_ms[10:]), np.array(host_ms[10:]), np.array(gpu_ms[10:])
        lat = {"device_ms_p50": float(np.median(dev_ms)), "device_ms_p99": float(np.percentile(dev_ms, 99)),
               "graph_replay_ms_p50": float(np.median(graph_ms[10:])) if graph_ms else None,
               "gpu_ms_p50": float(np.median(gpu_ms)),
               "host_e2e_ms_p50": float(np.median(host_ms)), "host_e2e_ms_p99": float(np.percentile(host_ms, 99)),
               "windows": len(dev_ms),
               "note": "one 1280x720 window per call; device_ms = wall clock of the call with its events resident, "
                       "incl. launch + sync; graph_replay_ms = the same, the call replayed from a CUDA graph; gpu_ms = CUDA "
                       "events around the call's kernels; host_e2e adds the H2D of "
                       "its events and the D2H of its 3.7 MB surface (paper: 16.88 ms per window for the "
                       "whole pipeline incl. flow on an RTX 5000, P:555)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0))
        n_s = max(cores, args.cpu_windows)
        r, done, wall = oracle_rate(name, n_s, cores)
        cpu = {"value": r, "unit": UNIT, "cores": cores, "cpu": cpu_model(), "kind": "oracle",
               "sample": f"{done} windows of {wl.name} (distinct seeds), {cores} processes, "
                         f"C oracle fp64 as it stands, {wall:.1f} s wall"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "u32+i32+f32", "data": "synthetic",
        "config": workload_config(name, world, 0, args.windows, events_per_gpu=n_ev),
        "mev_per_s": value * (n_ev / nwin) / 1e6,
        "hbm_frac_path": {"achieved_gbs": path_gbs, "peak": peak, "frac": path_gbs / peak,
                          "frac_nominal_8tbs": path_gbs / 8000.0,
                          "bytes_per_window": path_bytes / nwin,
                          "note": "algorithmic bytes of the whole path: 4 B/event + 4 B/px + offsets"},
        "roofline": {"bound": "hbm", "kernel": EDT_KERNEL_NAME,
                     "achieved": edt_gbs, "peak": peak, "unit": "GB/s", "frac": edt_gbs / peak,
                     "traffic": traffic_per_launch(args.traffic, nwin / max(1, edt_n // args.steps)),
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": edt_bytes_per_launch, "avg_launch_ms": edt_avg_ms,
                     "share_of_step": edt_ms / max(1e-9, ms_max),
                     "ncu_summary": args.ncu_summary},
        "kernels": {"frame_kernel": {"avg_ms": fr_avg_ms, "launches": fr_n,
                                     "achieved_gbs": fr_bytes_per_launch / (fr_avg_ms / 1e3) / 1e9 if fr_avg_ms else None,
                                     "share_of_step": fr_ms / max(1e-9, ms_max)},
                    "window_kernel": {"avg_ms": edt_avg_ms, "launches": edt_n,
                                      "share_of_step": edt_ms / max(1e-9, ms_max)}},
        "gpu_launches": int(launches_per_step * args.steps),
        "dist": dist_info,
        "cross_rank_check": xcheck,
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "exact_edt_path": exact,
        "f1_u8_surface": f1,
        "f1_f16_surface": f1_f16,
        "f1_u8_normalised_log": f1_norm,
        "f2_latency": lat,
        "f2_windowing": f2w,
        "f2_stream": f2s,
        "f3_fwl": f3,
        "f4_flow": f4,
        "f4_pipeline": f4p,
        "c2_lowres": c2,
        "c5_burst": c5,
        "c4_r1_baseline": c4_r1,
        "c3_weak_scaling": c3_weak,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=None, choices=sorted(WORKLOADS),
                    help="workload (default: C3 on one GPU, C4 = 16k windows sharded when N > 1)")
    ap.add_argument("--windows", type=int, default=0,
                    help="override windows per GPU (C4: total windows) (default: config)")
    ap.add_argument("--c5-windows", type=int, default=16000,
                    help="C5 dense-burst windows in total, sharded across the ranks (BASELINE configs[4])")
    ap.add_argument("--e2e-windows", type=int, default=1000, help="windows per rank of the e2e run when N > 1")
    ap.add_argument("--ncu-summary", default="profiles/r02_ncu_full_frame_window.md",
                    help="committed ncu --set full summary of the dominant kernel (limiter evidence)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-exact", action="store_true", help="skip the exact-EDT comparison run")
    ap.add_argument("--no-f1", action="store_true", help="skip the 8-bit surface (row f1) run")
    ap.add_argument("--no-f3", action="store_true", help="skip the FWL (row f3) run")
    ap.add_argument("--no-f4", action="store_true", help="skip the flow consumer (row f4) run")
    ap.add_argument("--no-c2", action="store_true", help="skip the low-resolution C2 run")
    ap.add_argument("--no-c5", action="store_true", help="skip the dense-burst C5 run")
    ap.add_argument("--no-c4-r1", action="store_true", help="skip the one-GPU 16k-window C4 run (N = 1)")
    ap.add_argument("--f3-windows", type=int, default=128, help="C3-geometry windows of the FWL (row f3) run")
    ap.add_argument("--no-latency", action="store_true", help="skip the single-window latency (row f2) run")
    ap.add_argument("--chunk", type=int, default=0, help="windows per launch pair (0 = library default)")
    ap.add_argument("--cpu-windows", type=int, default=512,
                    help="oracle windows timed for cpu_baseline (~15 core-seconds at 1280x720 on the GPU box)")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per EDT launch (from profiles/), reported in roofline.traffic")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing protocol", file=sys.stderr)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # the driver launches N > 1 under torchrun; a bare `bench.py --gpus N` re-runs itself that way
        return multi.relaunch_under_torchrun(args.gpus, os.path.abspath(__file__), sys.argv[1:])
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
