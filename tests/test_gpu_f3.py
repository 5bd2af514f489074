"""GPU parity of SURVEY §8 row f3: the flow-compensated event image and the Flow Warping Loss
 through ieds_fwl_batch, against the fp64 oracle.

The warp is the oracle's fp64 arithmetic operation for operation (same drop / floor decisions,
same weights); only the order of the per-pixel fp64 sums differs (atomics), so I_comp matches
to 1e-12 absolute and FWL / variances to 1e-9 relative (SPEC S:567's oracle tolerance).
"""
import numpy as np
import pytest

import oracle
from synth.events import DAVIS, GEN4
from synth.flowscene import flow_batch

pytestmark = pytest.mark.gpu


def _gpu_fwl(xy, t, p, off, flows, t_ref, dt, W, H, comp=True):
    import torch

    import paper_2112_10591_b200 as ieds

    dev = torch.device("cuda", 0)
    T = lambda a, dt_: torch.from_numpy(np.ascontiguousarray(a)).to(dev) if dt_ is None else \
        torch.from_numpy(np.ascontiguousarray(a).view(dt_)).to(dev)
    with ieds.Builder(W, H, 1, 4, device=0) as bld:
        r = bld.fwl_batch(T(xy, np.int32), T(t, None), T(p, None), T(off, None), T(flows, None), T(t_ref, None), dt,
                          variances=True, comp_image=comp)
        bld.sync()
        return {k: v.cpu().numpy() for k, v in r.items()}


def _check(xy, t, p, off, flows, t_ref, dt, W, H, comp_tol=1e-12):
    g = _gpu_fwl(xy, t, p, off, flows, t_ref, dt, W, H)
    for b in range(len(off) - 1):
        sl = slice(off[b], off[b + 1])
        r = oracle.fwl(xy[sl], t[sl], p[sl], W, H, flows[b], t_ref[b], dt, images=True)
        if np.isnan(r["fwl"]):
            assert np.isnan(g["fwl"][b])
        else:
            assert abs(g["fwl"][b] - r["fwl"]) <= 1e-9 * abs(r["fwl"]), (b, g["fwl"][b], r["fwl"])
        for k in ("var_comp", "var_uncomp"):
            assert abs(g[k][b] - r[k]) <= 1e-9 * abs(r[k]) + 1e-15, (b, k)
        err = np.max(np.abs(g["comp_image"][b] - r["I_comp"]))
        assert err <= comp_tol, (b, err)
    return g


def test_fwl_parity_generated_scenes_davis():
    xy, t, p, off, flows, _fl, t_ref = flow_batch(DAVIS, 1, 0, 5)
    _check(xy, t, p, off, flows, t_ref, DAVIS.dt_us, DAVIS.width, DAVIS.height)


def test_fwl_parity_hand_cases_and_degenerates():
    """Unit shift, half-pixel splat, border drop / W-1 boundary, an empty window (NaN),
    zero flow (FWL = 1) and a random |F| = 10 field, in one batch."""
    W, H, dt = 12, 10, 1000
    wins, flows = [], []

    def add(points, F):
        a = np.array(points, np.int64).reshape(-1, 4)
        wins.append(a)
        flows.append(F.astype(np.float32))

    F = np.zeros((H, W, 2), np.float32)
    F1 = F.copy(); F1[5, 5] = (1.0, 0.0)
    add([(5, 5, 0, 1), (2, 3, 400, -1)], F1)
    F2 = F.copy(); F2[5, 5] = (0.5, 0.25)
    add([(5, 5, 0, 1), (5, 5, 500, 0)], F2)
    F3 = F.copy(); F3[0, 0] = (-0.5, 0.0)
    add([(0, 0, 0, 1), (W - 1, 0, 0, 1), (W - 1, H - 1, 999, -1)], F3)
    add([], F)
    rng = np.random.default_rng(1)
    pts = [(int(rng.integers(0, W)), int(rng.integers(0, H)), int(rng.integers(0, dt)), int(rng.integers(0, 2)))
           for _ in range(300)]
    add(pts, F)
    add(pts, rng.uniform(-10, 10, (H, W, 2)))
    off = np.zeros(len(wins) + 1, np.int64)
    off[1:] = np.cumsum([len(a) for a in wins])
    allp = np.concatenate([a for a in wins if len(a)])
    xy = (allp[:, 0] | (allp[:, 1] << 16)).astype(np.uint32)
    t = allp[:, 2].astype(np.int64)
    p = allp[:, 3].astype(np.int8)
    t_ref = np.full(len(wins), dt, np.int64)
    g = _check(xy, t, p, off, np.stack(flows), t_ref, dt, W, H)
    assert np.isnan(g["fwl"][3])
    assert abs(g["fwl"][4] - 1.0) <= 1e-12           # zero flow
    assert g["comp_image"][0][5, 6] == 1.0           # S:400 unit shift


def test_fwl_parity_c3_geometry_and_chunking():
    """C3 geometry (1280x720, 75k events per window) over more windows than one scratch
    pass (4 by default), so the re-zeroed scratch is reused; results do not depend on the batch."""
    xy, t, p, off, flows, _fl, t_ref = flow_batch(GEN4, 3, 0, 10)
    g = _check(xy, t, p, off, flows, t_ref, GEN4.dt_us, GEN4.width, GEN4.height)
    # the same windows one call at a time give the same values (to the fp64 summation order)
    for b in (0, 9):
        sl = slice(off[b], off[b + 1])
        g1 = _gpu_fwl(xy[sl], t[sl], p[sl], np.array([0, off[b + 1] - off[b]], np.int64), flows[b:b + 1],
                      t_ref[b:b + 1], GEN4.dt_us, GEN4.width, GEN4.height, comp=False)
        assert abs(g1["fwl"][0] - g["fwl"][b]) <= 1e-12 * abs(g["fwl"][b])
    assert np.all(np.isfinite(g["fwl"])) and np.all(g["fwl"] > 0.0)


def test_fwl_out_of_frame_event_latched():
    import torch

    import paper_2112_10591_b200 as ieds

    W, H, dt = 8, 8, 100
    dev = torch.device("cuda", 0)
    xy = torch.tensor([1 | (1 << 16), 9 | (1 << 16)], dtype=torch.int32, device=dev)   # x = 9 >= W
    t = torch.zeros(2, dtype=torch.int64, device=dev)
    p = torch.ones(2, dtype=torch.int8, device=dev)
    off = torch.tensor([0, 2], dtype=torch.int64, device=dev)
    flow = torch.zeros((1, H, W, 2), dtype=torch.float32, device=dev)
    tr = torch.full((1,), dt, dtype=torch.int64, device=dev)
    with ieds.Builder(W, H, 1, 4, device=0) as bld:
        r = bld.fwl_batch(xy, t, p, off, flow, tr, dt, variances=True)
        with pytest.raises(ieds.IedsRangeError):
            bld.sync()
        # the in-frame event alone: 1 on 64 pixels, var = 63/64^2 for both images
        assert abs(r["var_uncomp"].item() - 63.0 / 4096.0) < 1e-15


def test_fwl_pileup_precision():
    """Sum of squares from the atomics' old values (fwl_kernel.cuh): 60k events on 3 pixels
    with fractional weights, so each compensated pixel sees ~20k adds and reaches |I| ~ 1e4.
    The telescoped sum must still give the variances within 1e-9 relative; a second window has
    nearly every event dropped at the border.  I_comp itself differs from the oracle only by the
    order of its fp64 sums: n adds of weights |w| <= 1 bound that by n * u * n (u = 2^-53)."""
    W, H, dt = 64, 48, 10000
    rng = np.random.default_rng(7)
    n = 60000
    xs = rng.choice([10, 11, 40], n)
    ys = rng.choice([20, 21, 5], n)
    ts = rng.integers(0, dt, n)
    ps = (rng.random(n) < 0.8).astype(np.int8)   # mostly positive: large signed sums
    F = np.zeros((H, W, 2), np.float32)
    F[:, :, 0] = 0.37
    F[:, :, 1] = -0.21
    F2 = np.zeros((H, W, 2), np.float32)
    F2[:, :, 0] = 80.0                           # almost everything warps out of the frame
    xy = np.concatenate([xs | (ys << 16), xs | (ys << 16)]).astype(np.uint32)
    t = np.concatenate([ts, ts]).astype(np.int64)
    p = np.concatenate([ps, ps])
    off = np.array([0, n, 2 * n], np.int64)
    t_ref = np.full(2, dt, np.int64)
    g = _check(xy, t, p, off, np.stack([F, F2]), t_ref, dt, W, H, comp_tol=float(n) * n * 2.0 ** -53)
    assert np.isfinite(g["fwl"]).all()


def test_fwl_first_call_on_a_side_stream():
    """the f3 scratch is zeroed on the caller's stream at the first call, so a first
    call issued on a non-blocking torch side stream sees zeroed images (FWL equals the oracle's)."""
    import torch

    import paper_2112_10591_b200 as ieds

    xy, t, p, off, flows, _fl, t_ref = flow_batch(DAVIS, 2, 0, 3)
    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    args = (T(xy.view(np.int32)), T(t), T(p), T(off), T(flows), T(t_ref))
    torch.cuda.synchronize()
    side = torch.cuda.Stream(device=dev)
    with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, device=0) as bld:
        with torch.cuda.stream(side):
            r = bld.fwl_batch(*args, DAVIS.dt_us)
            bld.sync(stream=side)
        g = r["fwl"].cpu().numpy()
    for b in range(len(off) - 1):
        sl = slice(off[b], off[b + 1])
        ref = oracle.fwl(xy[sl], t[sl], p[sl], DAVIS.width, DAVIS.height, flows[b], t_ref[b], DAVIS.dt_us)["fwl"]
        assert abs(g[b] - ref) <= 1e-9 * abs(ref)


def test_fwl_scratch_sets_alternate_across_passes_and_calls():
    """The f3 scratch is two image sets, one re-zeroed on an internal stream while the other is
    splatted: 3 calls of 37 windows (3 passes of <= 16 windows each) must all equal the oracle,
    so every pass starts from zeroed images whichever set and call it falls in."""
    import torch

    import paper_2112_10591_b200 as ieds

    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, device=0) as bld:
        for call in range(3):
            xy, t, p, off, flows, _fl, t_ref = flow_batch(DAVIS, 5 + call, 0, 37)
            r = bld.fwl_batch(T(xy.view(np.int32)), T(t), T(p), T(off), T(flows), T(t_ref), DAVIS.dt_us)
            bld.sync()
            g = r["fwl"].cpu().numpy()
            for b in (0, 15, 16, 31, 32, 36):
                sl = slice(off[b], off[b + 1])
                ref = oracle.fwl(xy[sl], t[sl], p[sl], DAVIS.width, DAVIS.height, flows[b], t_ref[b], DAVIS.dt_us)["fwl"]
                assert abs(g[b] - ref) <= 1e-9 * abs(ref), (call, b)
