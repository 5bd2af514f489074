"""Seeded synthetic inputs for row f3 (flow-compensated event image / Flow Warping Loss).

INPUTS ONLY: a scene of edge primitives that moves during each window under a known dense
affine flow field, and that field itself.  The method's arithmetic (the warp, the bilinear
splat, the variances) lives in oracle/ and in the CUDA path; nothing here computes it.

Motion model: the flow of window k is F(x, y) = v + A (x - cx, y - cy) pixels per window,
with |F| <= vmax over the frame (a translation plus a small rotation / zoom, the ego-motion
shape of the paper's driving scenes).  An edge point at p0 at the window start is at
p0 + F(p0) * tau at time t = t_k + tau * dt (first order in the motion), so compensating each
event by F at its pixel to t_ref = the window end brings the events of one point together.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .events import GEN4, SceneConfig, _scene, splitmix64, window_seed


@dataclass(frozen=True)
class AffineFlow:
    vx: float
    vy: float
    a11: float
    a12: float
    a21: float
    a22: float
    cx: float
    cy: float

    def at(self, x, y):
        dx = np.asarray(x, np.float64) - self.cx
        dy = np.asarray(y, np.float64) - self.cy
        return self.vx + self.a11 * dx + self.a12 * dy, self.vy + self.a21 * dx + self.a22 * dy


def affine_flow(width: int, height: int, seed: int, k: int, vmax: float = 24.0) -> AffineFlow:
    """The flow of window k: a translation of up to vmax/2 plus a rotation/zoom whose
    contribution stays below vmax/2 over the frame."""
    rng = np.random.Generator(np.random.Philox(key=splitmix64(window_seed(seed, k) ^ 0xF10F)))
    r = 0.5 * float(np.hypot(width, height))
    s = 0.5 * vmax / r
    v = rng.uniform(-0.5 * vmax, 0.5 * vmax, 2) / np.sqrt(2.0)
    A = rng.uniform(-s, s, (2, 2)) / 2.0
    return AffineFlow(float(v[0]), float(v[1]), float(A[0, 0]), float(A[0, 1]), float(A[1, 0]), float(A[1, 1]),
                      0.5 * (width - 1), 0.5 * (height - 1))


def flow_field(width: int, height: int, fl: AffineFlow) -> np.ndarray:
    """Dense float32 [H][W][2] (dx, dy) field of an affine flow, pixels per window."""
    yy, xx = np.mgrid[0:height, 0:width]
    fx, fy = fl.at(xx, yy)
    return np.stack([fx, fy], axis=-1).astype(np.float32)


def flow_window(cfg: SceneConfig, config_seed: int, k: int, fl: AffineFlow):
    """Events of window k of a scene moving under `fl`: (xy uint32, t_us int64 sorted,
    p int8 +-1, t_start_us).  Edge events sit at p0 + F(p0) tau (+ jitter) with their
    primitive's polarity, noise events are uniform with random polarity; events that leave
    the frame are not emitted."""
    kind, cx, cy, length, ang, span, radius, _vel, cw = _scene(cfg, config_seed)
    rng = np.random.Generator(np.random.Philox(key=splitmix64(window_seed(config_seed, k) ^ 0xF3)))
    n = cfg.events_per_window
    n_noise = int(round(n * cfg.noise_frac))
    n_edge = n - n_noise
    idx = np.minimum(np.searchsorted(cw, rng.random(n_edge), side="right"), len(cw) - 1)
    u = rng.random(n_edge)
    seg = kind[idx] == 0
    th_arc = ang[idx] + u * span[idx]
    px = np.where(seg, cx[idx] + u * length[idx] * np.cos(ang[idx]), cx[idx] + radius[idx] * np.cos(th_arc))
    py = np.where(seg, cy[idx] + u * length[idx] * np.sin(ang[idx]), cy[idx] + radius[idx] * np.sin(th_arc))
    px = np.mod(px, cfg.width)
    py = np.mod(py, cfg.height)
    tau = rng.random(n_edge)
    fx, fy = fl.at(px, py)
    ex = np.floor(px + fx * tau + rng.normal(0.0, cfg.sigma, n_edge) + 0.5).astype(np.int64)
    ey = np.floor(py + fy * tau + rng.normal(0.0, cfg.sigma, n_edge) + 0.5).astype(np.int64)
    nx = rng.integers(0, cfg.width, n_noise)
    ny = rng.integers(0, cfg.height, n_noise)
    ntau = rng.random(n_noise)
    # polarity is coherent along an edge (one sign per primitive, as a moving contrast edge
    # emits); noise events have random polarity
    pol = np.random.Generator(np.random.Philox(key=splitmix64(config_seed ^ 0x9017))).integers(0, 2, len(cw))
    pe = pol[idx].astype(np.int8) * 2 - 1
    pn = rng.integers(0, 2, n_noise).astype(np.int8) * 2 - 1
    x = np.concatenate([ex, nx])
    y = np.concatenate([ey, ny])
    tt = np.concatenate([tau, ntau])
    pp = np.concatenate([pe, pn])
    keep = (x >= 0) & (x < cfg.width) & (y >= 0) & (y < cfg.height)
    x, y, tt, pp = x[keep], y[keep], tt[keep], pp[keep]
    t0 = k * cfg.dt_us
    t = t0 + np.minimum((tt * cfg.dt_us).astype(np.int64), cfg.dt_us - 1)
    order = np.argsort(t, kind="stable")
    xy = (x[order].astype(np.uint32) | (y[order].astype(np.uint32) << np.uint32(16))).astype(np.uint32)
    return xy, t[order].astype(np.int64), pp[order].astype(np.int8), t0


def flow_batch(cfg: SceneConfig, config_seed: int, k0: int, n_windows: int, with_fields: bool = True):
    """Windows k0.. as CSR plus per-window flow fields and reference times (window ends):
    (xy, t, p, offsets, flows [B][H][W][2] or None, affine params, t_ref [B])."""
    parts, fls = [], []
    for i in range(n_windows):
        fl = affine_flow(cfg.width, cfg.height, config_seed, k0 + i)
        fls.append(fl)
        parts.append(flow_window(cfg, config_seed, k0 + i, fl))
    off = np.zeros(n_windows + 1, np.int64)
    off[1:] = np.cumsum([len(q[0]) for q in parts])
    xy = np.concatenate([q[0] for q in parts]) if parts else np.zeros(0, np.uint32)
    t = np.concatenate([q[1] for q in parts]) if parts else np.zeros(0, np.int64)
    p = np.concatenate([q[2] for q in parts]) if parts else np.zeros(0, np.int8)
    t_ref = np.array([q[3] + cfg.dt_us for q in parts], np.int64)
    flows = np.stack([flow_field(cfg.width, cfg.height, fl) for fl in fls]) if with_fields else None
    return xy, t, p, off, flows, fls, t_ref


F3_SCENE = GEN4   # C3 geometry: 1280x720, 75k events per 15 ms window
