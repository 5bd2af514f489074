"""GPU parity of SURVEY §8 row f4: the flow consumer (DESIGN reading R21) through
ieds_flow_step, against the fp64 oracle on the same fp32 surfaces.

Tolerances (row f4): the device is fp32, the oracle fp64.  One step's rounding
(255-scaled images, |J| <= 255, ~1e-5 absolute) moves the flow by ~1e-6-1e-5 px; the state
feeds each window's flow into the next one's prediction and every coarse level is upsampled
x2, so the difference grows over a sequence (measured: <= 7e-4 px through the first three
estimated windows, mean 1e-6 px and max 2e-2 px over ten).  Bars: bit-exact zeros on the first
window and on a static scene; <= 2e-3 px for the first three estimated windows; over the whole
sequence mean <= 1e-4 px and max <= 5e-2 px; the valid mask equals E_d exactly.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _seq(W, H, v, n):
    from tests.test_oracle_pins import _square_sequence

    return _square_sequence(W, H, v, n)


def _bits(E):
    H, W = E.shape
    NW = (W + 31) // 32
    words = np.zeros((H, NW), np.uint32)
    for x in range(W):
        words[:, x // 32] |= (E[:, x].astype(np.uint32) << np.uint32(x % 32))
    return words


def _run(seq, W, H, levels=3, use_mask=True, iters=(20, 20, 20)):
    import torch

    import paper_2112_10591_b200 as ieds

    dev = torch.device("cuda", 0)
    fo = oracle.FlowOracle(W, H, levels=levels, iters=iters)
    out = []
    with ieds.FlowEstimator(W, H, levels=levels, iterations=iters, device=0) as fe:
        for S, E in seq:
            S32 = S.astype(np.float32)
            Fo = fo.step(S32.astype(np.float64))
            eb = torch.from_numpy(_bits(E).view(np.int32)).to(dev) if use_mask else None
            Fg, vg = fe.step(torch.from_numpy(S32).to(dev), eb)
            torch.cuda.synchronize()
            out.append((Fo, Fg.cpu().numpy().astype(np.float64), vg.cpu().numpy(), E))
    return out


@pytest.mark.parametrize("W,H,v,levels", [(256, 192, 1, 3), (384, 192, 8, 3), (256, 192, 1, 1)])
def test_flow_sequence_parity(W, H, v, levels):
    res = _run(_seq(W, H, v, 10), W, H, levels)
    Fo0, Fg0, v0, _ = res[0]
    assert not Fg0.any() and not v0.any()                   # first window: zero, nothing valid
    diffs = []
    for k, (Fo, Fg, vg, E) in enumerate(res[1:], start=1):
        Fom, vo = oracle.mask_flow(Fo, E.astype(np.uint8))
        assert np.array_equal(vg, vo), k                     # valid = E_d
        assert not Fg[~E].any(), k                           # flow off the mask is 0
        d = np.abs(Fg - Fom)
        if k <= 3:
            assert d.max() <= 2e-3, (k, d.max())
        diffs.append(d)
    d = np.stack(diffs)
    assert d.mean() <= 1e-4 and d.max() <= 5e-2, (d.mean(), d.max())


@pytest.mark.parametrize("iters", [(7, 5, 3), (1, 0, 2), (13, 9, 6)])
def test_flow_sweep_counts(iters):
    """The Jacobi sweeps run up to 4 per launch on halo tiles (temporal blocking); sweep counts
    that are not multiples of 4, a single sweep and none at all match the oracle's plain
    per-sweep iteration.  Frames of 200 x 136 leave ragged 64 x 16 tiles on every level."""
    W, H = 200, 136
    res = _run(_seq(W, H, 2, 6), W, H, 3, iters=iters)
    for k, (Fo, Fg, vg, E) in enumerate(res[1:], start=1):
        Fom, vo = oracle.mask_flow(Fo, E.astype(np.uint8))
        assert np.array_equal(vg, vo), k
        d = np.abs(Fg - Fom)
        assert d.max() <= 2e-3, (iters, k, d.max())


def test_flow_static_scene_and_dense_output():
    """A static scene gives exactly zero flow on the device too (the warp by 0 is exact); with
    no mask the dense field is returned and everything after the first window is valid."""
    W, H = 128, 96
    res = _run(_seq(W, H, 0, 4), W, H, use_mask=False)
    for k, (Fo, Fg, vg, _E) in enumerate(res):
        assert not Fg.any()
        assert vg.all() == (k > 0)
    res = _run(_seq(W, H, 1, 4), W, H, use_mask=False)
    for k, (Fo, Fg, vg, _E) in enumerate(res[1:], start=1):
        assert np.abs(Fg - Fo).max() <= 2e-3


def test_flow_reset_starts_a_new_sequence():
    import torch

    import paper_2112_10591_b200 as ieds

    W, H = 64, 48
    seq = _seq(W, H, 1, 3)
    with ieds.FlowEstimator(W, H, device=0) as fe:
        for S, _ in seq:
            fe.step(torch.from_numpy(S.astype(np.float32)).cuda())
        fe.reset()
        F, v = fe.step(torch.from_numpy(seq[0][0].astype(np.float32)).cuda())
        assert not F.any().item() and not v.any().item()
        assert fe.launches_per_step() > 0


@pytest.mark.parametrize("iters", [(20, 20, 20), (7, 5, 13)])
def test_flow_cooperative_sweeps_bit_identical(iters, monkeypatch):
    """Levels whose sweep tiles are all co-resident run their sweeps as one cooperative launch
    (grid-wide barriers between 4-sweep chunks); the same tiles and operations as one launch per
    chunk (IEDS_FLOW_COOP=0, read at create), so the flow is identical bit for bit."""
    import torch

    import paper_2112_10591_b200 as ieds

    W, H = 640, 360
    seq = _seq(W, H, 3, 5)
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("IEDS_FLOW_COOP", mode)
        out = []
        with ieds.FlowEstimator(W, H, iterations=iters, device=0) as fe:
            for S, E in seq:
                F, v = fe.step(torch.from_numpy(S.astype(np.float32)).cuda())
                out.append(F.clone())
            res[mode] = (out, fe.launches_per_step())
    for a, b in zip(res["0"][0], res["1"][0]):
        assert torch.equal(a, b)
    assert res["1"][1] <= res["0"][1]


def test_flow_step_validates_arguments():
    """step() rejects a wrong-shaped/typed `out`, short or mistyped edge bits and
    accepts a torch.cuda.Stream object as the stream."""
    import torch

    import paper_2112_10591_b200 as ieds

    dev = torch.device("cuda", 0)
    W, H = 64, 48
    S = torch.rand((H, W), dtype=torch.float32, device=dev)
    with ieds.FlowEstimator(W, H, device=0) as fe:
        with pytest.raises(ValueError):
            fe.step(S, out=torch.empty((H, W), dtype=torch.float32, device=dev))
        with pytest.raises(ValueError):
            fe.step(S, out=torch.empty((H, W, 2), dtype=torch.float64, device=dev))
        with pytest.raises(ValueError):
            fe.step(S, edge_bits=torch.zeros(H * 2 - 1, dtype=torch.int32, device=dev))
        with pytest.raises(ValueError):
            fe.step(S, edge_bits=torch.zeros(H * 2, dtype=torch.float32, device=dev))
        with pytest.raises(ValueError):
            fe.step(torch.rand((2, H, W), dtype=torch.float32, device=dev))
        side = torch.cuda.Stream(device=dev)
        F, valid = fe.step(S, edge_bits=torch.zeros(H * 2, dtype=torch.int32, device=dev), stream=side)
        side.synchronize()
        assert F.shape == (H, W, 2) and int(valid.sum()) == 0
