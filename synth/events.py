"""Seeded synthetic event-window generator (shared by the oracle tests and the CUDA path).

This module produces *inputs only*: packed event coordinates grouped by time window.
It holds none of the method's arithmetic (no accumulation, filtering, distance
transform or transfer function) — see DESIGN.md "Input recipe".

Workload shape (BASELINE.json configs): a persistent "driving scene"
of edge primitives (line segments and circular arcs) that translate by a per-primitive
velocity each window, so consecutive windows correlate; events are sampled on the
primitives with Gaussian jitter sigma (edge thickness) and a uniform noise fraction
eta (event cameras are noisy sensors, §III-B).  Duplicated pixels are
common, as they are in real windows.  Timestamps are uniform inside the window and
polarity is random; both stay host-side (polarity is ignored by the edge image,
PAPER.md §III-A) and are only produced on request.

Per-window seeds follow SURVEY.md §8(d): seed_k = splitmix64(config_seed XOR k), so any
rank (or the oracle) can regenerate any window independently and byte-identically.
The per-window stream is numpy's counter-based Philox keyed by seed_k.
"""
from __future__ import annotations

import dataclasses
import functools

import numpy as np

MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """SplitMix64 finaliser (Steele et al. 2014) on a 64-bit integer."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def window_seed(config_seed: int, k: int) -> int:
    return splitmix64((config_seed ^ k) & MASK64)


@dataclasses.dataclass(frozen=True)
class SceneConfig:
    """Shape of a synthetic event stream.

    width/height: sensor geometry (346x260 DAVIS-like, 1280x720 Gen4-like).
    events_per_window: rate x Delta T (e.g. 5 Mev/s x 15 ms = 75k).
    n_prims: number of edge primitives in the persistent scene.
    len_range: primitive length range (pixels).
    sigma: Gaussian jitter of events around the edge (pixels).
    noise_frac: fraction of uniformly distributed noise events.
    vmax: max |velocity| per axis (pixels / window).
    count_jitter: per-window event count is events_per_window * U(1-j, 1+j) (0 = fixed).
    dt_us: window length Delta T in microseconds (timestamps only).
    """

    width: int
    height: int
    events_per_window: int
    n_prims: int
    len_range: tuple = (20.0, 200.0)
    sigma: float = 0.6
    noise_frac: float = 0.10
    vmax: float = 8.0
    count_jitter: float = 0.0
    dt_us: int = 15000


@dataclasses.dataclass(frozen=True)
class Workload:
    """A named benchmark/parity configuration (BASELINE.json configs[0..4]).

    n_d, n_f and d_sat are the method's parameters as the paper states them
    (§IV-A P:258 low-res: N_d=1, N_f=4, d_sat=6; P:260 HD: N_d=2, N_f=3, d_sat=6).
    They are carried here as plain numbers; each side derives alpha itself.
    """

    name: str
    scene: SceneConfig
    n_windows: int
    seed: int
    n_d: int
    n_f: int
    d_sat: float = 6.0


DAVIS = SceneConfig(346, 260, 20_000, n_prims=28, len_range=(15.0, 120.0), sigma=0.45,
                    noise_frac=0.10, vmax=4.0, dt_us=32000)
GEN4 = SceneConfig(1280, 720, 75_000, n_prims=90, len_range=(30.0, 260.0), sigma=0.55,
                   noise_frac=0.10, vmax=8.0, dt_us=15000)
GEN4_BURST = SceneConfig(1280, 720, 300_000, n_prims=720, len_range=(40.0, 320.0), sigma=2.0,
                         noise_frac=0.10, vmax=8.0, dt_us=15000)

WORKLOADS = {
    "C1": Workload("C1", DAVIS, 1, seed=1, n_d=1, n_f=4),
    "C2": Workload("C2", DAVIS, 10_000, seed=2, n_d=1, n_f=4),
    "C3": Workload("C3", GEN4, 1_000, seed=3, n_d=2, n_f=3),
    "C4": Workload("C4", GEN4, 16_000, seed=4, n_d=2, n_f=3),
    "C5": Workload("C5", GEN4_BURST, 16_000, seed=5, n_d=2, n_f=3),
}


@functools.lru_cache(maxsize=16)
def _scene(cfg: SceneConfig, seed: int):
    """Persistent primitives of a scene (depends on the config seed only)."""
    rng = np.random.Generator(np.random.Philox(key=splitmix64(seed ^ 0x5CE9E)))
    m = cfg.n_prims
    kind = rng.integers(0, 2, m)                       # 0 = segment, 1 = arc
    cx = rng.uniform(0, cfg.width, m)
    cy = rng.uniform(0, cfg.height, m)
    length = rng.uniform(cfg.len_range[0], cfg.len_range[1], m)
    ang = rng.uniform(0, 2 * np.pi, m)
    # arcs: radius from length and span
    span = rng.uniform(0.5 * np.pi, 2 * np.pi, m)
    radius = np.maximum(length / span, 3.0)
    vel = rng.uniform(-cfg.vmax, cfg.vmax, (m, 2))
    w = np.where(kind == 0, length, radius * span)
    cw = np.cumsum(w)
    cw /= cw[-1]
    return kind, cx, cy, length, ang, span, radius, vel, cw


def window_events(cfg: SceneConfig, config_seed: int, k: int, with_tp: bool = False):
    """Events of window k: packed uint32 xy = x | (y << 16), plus (t_us, p) if requested."""
    kind, cx, cy, length, ang, span, radius, vel, cw = _scene(cfg, config_seed)
    rng = np.random.Generator(np.random.Philox(key=window_seed(config_seed, k)))
    n = cfg.events_per_window
    if cfg.count_jitter > 0:
        n = int(round(n * rng.uniform(1 - cfg.count_jitter, 1 + cfg.count_jitter)))
    n_noise = int(round(n * cfg.noise_frac))
    n_edge = n - n_noise
    idx = np.searchsorted(cw, rng.random(n_edge), side="right")
    idx = np.minimum(idx, len(cw) - 1)
    u = rng.random(n_edge)
    seg = kind[idx] == 0
    # segment: start + u*L*(cos,sin); arc: centre + r*(cos,sin)(ang + u*span)
    th_seg = ang[idx]
    th_arc = ang[idx] + u * span[idx]
    px = np.where(seg, cx[idx] + u * length[idx] * np.cos(th_seg), cx[idx] + radius[idx] * np.cos(th_arc))
    py = np.where(seg, cy[idx] + u * length[idx] * np.sin(th_seg), cy[idx] + radius[idx] * np.sin(th_arc))
    px = px + k * vel[idx, 0] + rng.normal(0.0, cfg.sigma, n_edge)
    py = py + k * vel[idx, 1] + rng.normal(0.0, cfg.sigma, n_edge)
    ex = np.mod(np.floor(px + 0.5).astype(np.int64), cfg.width)
    ey = np.mod(np.floor(py + 0.5).astype(np.int64), cfg.height)
    nx = rng.integers(0, cfg.width, n_noise)
    ny = rng.integers(0, cfg.height, n_noise)
    x = np.concatenate([ex, nx])
    y = np.concatenate([ey, ny])
    perm = rng.permutation(n)
    xy = (x[perm].astype(np.uint32) | (y[perm].astype(np.uint32) << np.uint32(16))).astype(np.uint32)
    if not with_tp:
        return xy
    t = np.sort(rng.integers(k * cfg.dt_us, (k + 1) * cfg.dt_us, n)).astype(np.int64)
    p = rng.integers(0, 2, n).astype(np.int8) * 2 - 1
    return xy, t, p


def batch_events(cfg: SceneConfig, config_seed: int, k0: int, n_windows: int):
    """Windows k0 .. k0+n_windows-1 as CSR: (xy uint32[total], offsets int64[n_windows+1])."""
    parts = [window_events(cfg, config_seed, k0 + i) for i in range(n_windows)]
    offsets = np.zeros(n_windows + 1, dtype=np.int64)
    offsets[1:] = np.cumsum([len(p) for p in parts])
    xy = np.concatenate(parts) if parts else np.zeros(0, dtype=np.uint32)
    return xy, offsets


def workload_batch(name: str, k0: int = 0, n_windows: int | None = None):
    wl = WORKLOADS[name]
    nw = wl.n_windows if n_windows is None else n_windows
    return batch_events(wl.scene, wl.seed, k0, nw)


def unpack_xy(xy: np.ndarray):
    xy = np.asarray(xy, dtype=np.uint32)
    return (xy & np.uint32(0xFFFF)).astype(np.int64), (xy >> np.uint32(16)).astype(np.int64)


def pack_xy(x, y) -> np.ndarray:
    x = np.asarray(x, dtype=np.int64)
    y = np.asarray(y, dtype=np.int64)
    return ((x & 0xFFFF) | ((y & 0xFFFF) << 16)).astype(np.uint32)


# ---- small structured frames for parity edge cases (inputs only) -------------------------

def random_frame_events(width: int, height: int, density: float, seed: int, dup: float = 0.5):
    """Events whose distinct pixels are a Bernoulli(density) frame, with ~dup extra duplicates."""
    rng = np.random.Generator(np.random.Philox(key=splitmix64(seed ^ 0xF4A3E)))
    mask = rng.random((height, width)) < density
    ys, xs = np.nonzero(mask)
    ndup = int(len(xs) * dup)
    if ndup and len(xs):
        j = rng.integers(0, len(xs), ndup)
        xs = np.concatenate([xs, xs[j]])
        ys = np.concatenate([ys, ys[j]])
    perm = rng.permutation(len(xs))
    return pack_xy(xs[perm], ys[perm])


def pattern_events(width: int, height: int, pattern: str, seed: int = 0):
    """Degenerate/structured windows: empty, single, all, checker, row, col, corners."""
    if pattern == "empty":
        return np.zeros(0, dtype=np.uint32)
    if pattern == "single":
        rng = np.random.Generator(np.random.Philox(key=splitmix64(seed ^ 0x51)))
        return pack_xy([rng.integers(0, width)], [rng.integers(0, height)])
    yy, xx = np.mgrid[0:height, 0:width]
    if pattern == "all":
        m = np.ones((height, width), bool)
    elif pattern == "checker":
        m = ((xx + yy) & 1) == 0
    elif pattern == "row":
        m = yy == height // 2
    elif pattern == "col":
        m = xx == width // 2
    elif pattern == "corners":
        m = np.zeros((height, width), bool)
        m[0, 0] = True
        m[height - 1, width - 1] = True
    else:
        raise ValueError(pattern)
    ys, xs = np.nonzero(m)
    return pack_xy(xs, ys)
