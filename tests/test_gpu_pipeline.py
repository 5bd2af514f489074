"""GPU tests of the Fig. 1 pipeline (ieds_pipeline_*, include/ieds.h): host chunks of a live event
stream in, each closed window's flow out (the blocks run concurrently; the image is
built when its window has expired).  The pipeline must give, bit for bit, what the batched path
gives -- ieds_window_offsets + ieds_build_batch (with the denoised edge bits) followed by one
ieds_flow_step per window in order -- wherever the stream is cut, and start a new sequence after
flush().  The batched path and the flow consumer are checked against the oracle elsewhere
(test_gpu_parity.py, test_gpu_f4.py).
"""
import numpy as np
import pytest

from synth.events import DAVIS, GEN4, window_events

pytestmark = pytest.mark.gpu


def _stream(cfg, seed, n_win, drop=()):
    xs, ts = [], []
    for k in range(n_win):
        if k in drop:
            continue
        xy, t, _ = window_events(cfg, seed, k, with_tp=True)
        xs.append(xy)
        ts.append(t)
    return np.concatenate(xs), np.concatenate(ts)


def _batched_flow(cfg, nd, nf, xy, t):
    import torch

    import paper_2112_10591_b200 as ieds

    dev = torch.device("cuda", 0)
    W, H = cfg.width, cfg.height
    with ieds.Builder(W, H, nd, nf, d_sat=6.0, device=0) as bld:
        off = bld.window_offsets(torch.from_numpy(t).to(dev), cfg.dt_us)
        B = off.numel() - 1
        Ed = torch.empty((B, H, (W + 31) // 32), dtype=torch.int32, device=dev)
        S = bld.build_batch(torch.from_numpy(xy.view(np.int32)).to(dev), off, denoised_bits=Ed)
        bld.sync()
    flows, valids = [], []
    with ieds.FlowEstimator(W, H, device=0) as fe:
        for k in range(B):
            F, V = fe.step(S[k], Ed[k])
            flows.append(F.cpu().numpy())
            valids.append(V.cpu().numpy())
    return S.cpu().numpy(), np.stack(flows), np.stack(valids)


def _pipelined(cfg, nd, nf, xy, t, cuts, repeats=1):
    import paper_2112_10591_b200 as ieds

    W, H = cfg.width, cfg.height
    outs = []
    with ieds.Builder(W, H, nd, nf, d_sat=6.0, device=0) as bld, ieds.FlowEstimator(W, H, device=0) as fe:
        with ieds.Pipeline(bld, fe, cfg.dt_us, surfaces=True) as pl:
            for _ in range(repeats):
                parts = []
                b = [0] + sorted(cuts) + [len(t)]
                for i in range(len(b) - 1):
                    parts.append(pl.push(t[b[i]:b[i + 1]], xy[b[i]:b[i + 1]]))
                parts.append(pl.flush())
                outs.append({k: np.concatenate([p[k] for p in parts]) for k in ("flow", "valid", "surfaces")})
    return outs


@pytest.mark.parametrize("cfg,nd,nf,nwin", [(DAVIS, 1, 4, 9), (GEN4, 2, 3, 6)])
def test_pipeline_matches_batched_surfaces_and_flow(cfg, nd, nf, nwin):
    xy, t = _stream(cfg, 3, nwin, drop=(2,))
    S, F, V = _batched_flow(cfg, nd, nf, xy, t)
    rng = np.random.default_rng(5)
    cuts = sorted(set(rng.integers(1, len(t), 7).tolist()))
    for out in _pipelined(cfg, nd, nf, xy, t, cuts, repeats=2):   # the second run: a new sequence
        assert out["surfaces"].shape == S.shape
        assert np.array_equal(out["surfaces"], S)
        assert np.array_equal(out["valid"], V)
        assert np.array_equal(out["flow"].view(np.uint32), F.view(np.uint32))
    assert np.abs(F[0]).max() == 0.0 and np.abs(F[-1]).max() > 0.0   # first window: zero flow


def test_pipeline_one_push_and_single_event_chunks():
    xy, t = _stream(DAVIS, 8, 4)
    S, F, V = _batched_flow(DAVIS, 1, 4, xy, t)
    n = len(t)
    for cuts in ([], [1, 2, n - 1]):
        out = _pipelined(DAVIS, 1, 4, xy, t, cuts)[0]
        assert np.array_equal(out["flow"].view(np.uint32), F.view(np.uint32)) and np.array_equal(out["surfaces"], S)


def test_pipeline_rejects_mismatched_handles():
    import ctypes

    import paper_2112_10591_b200 as ieds
    from paper_2112_10591_b200._lib import IEDS_EINVAL, load

    lib = load()
    p = ctypes.c_void_p()
    with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, device=0) as bld, \
            ieds.FlowEstimator(DAVIS.width + 2, DAVIS.height, device=0) as fe:
        assert lib.ieds_pipeline_create(bld._h, fe._h, 1000, ctypes.byref(p)) == IEDS_EINVAL and not p.value
    with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, device=0, out="u8") as bld, \
            ieds.FlowEstimator(DAVIS.width, DAVIS.height, device=0) as fe:
        assert lib.ieds_pipeline_create(bld._h, fe._h, 1000, ctypes.byref(p)) == IEDS_EINVAL and not p.value
