"""GPU tests of SURVEY §8 row f2's streaming ingest (ieds_stream_*, include/ieds.h) and the
library-side window count (ieds_window_count).

The paper's accumulation thread fills a buffer per event and a second thread builds the image
"when the time window has expired" (Fig. 1's concurrent blocks).  A stream cut at
arbitrary points and pushed chunk by chunk must give the same windows (reading R16: t0 = the
first event, window k = floor((t - t0)/dt) == k, empty interior windows emitted) and the same
surfaces, bit for bit, as the batched path over the whole stream -- which the parity suite
checks against the oracle.
"""
import ctypes

import numpy as np
import pytest

import oracle
from synth.events import DAVIS, GEN4, window_events

pytestmark = pytest.mark.gpu


def _stream(cfg, seed, n_win, drop=(), dt=None):
    """A time-ordered stream: the generator's windows laid end to end in time, the windows in
    `drop` removed (empty interior windows)."""
    xs, ts = [], []
    for k in range(n_win):
        if k in drop:
            continue
        xy, t, _ = window_events(cfg, seed, k, with_tp=True)
        xs.append(xy)
        ts.append(t)
    return np.concatenate(xs), np.concatenate(ts), dt or cfg.dt_us


def _batched(bld, xy, t, dt):
    import torch

    dev = bld.device
    off = bld.window_offsets(torch.from_numpy(t).to(dev), dt)
    S = bld.build_batch(torch.from_numpy(xy.view(np.int32)).to(dev), off)
    bld.sync()
    return S.cpu().numpy(), off.cpu().numpy()


def _pushed(bld, xy, t, dt, cuts):
    parts = []
    with bld.stream(dt) as st:
        b = [0] + sorted(cuts) + [len(t)]
        for i in range(len(b) - 1):
            parts.append(st.push(t[b[i]:b[i + 1]], xy[b[i]:b[i + 1]]))
        parts.append(st.flush())
    return np.concatenate([p for p in parts if len(p)]) if parts else None


@pytest.mark.parametrize("cfg,nd,nf,out", [(DAVIS, 1, 4, "f32"), (GEN4, 2, 3, "f32"), (DAVIS, 1, 4, "u8"),
                                           (GEN4, 2, 3, "f16")])
def test_stream_matches_batched_at_arbitrary_cuts(cfg, nd, nf, out):
    import paper_2112_10591_b200 as ieds

    xy, t, dt = _stream(cfg, 3, 9, drop=(4, 5))
    rng = np.random.default_rng(7)
    n = len(t)
    ref_off = oracle.window_offsets(t, dt)
    bounds = ref_off[1:-1]
    cut_sets = [
        [],                                                  # one push, everything closes at flush
        sorted(set(rng.integers(1, n, 13).tolist())),        # random cuts
        sorted(set(bounds.tolist()) - {0, n}),               # exactly at window starts
        sorted({int(b) + d for b in bounds for d in (-1, 1) if 0 < int(b) + d < n}),   # one event either side
        [1, 2, 3, n - 2, n - 1],                             # single-event chunks at both ends
    ]
    with ieds.Builder(cfg.width, cfg.height, nd, nf, d_sat=6.0, device=0, out=out) as bld:
        S_ref, off = _batched(bld, xy, t, dt)
        assert np.array_equal(off, ref_off)
        assert len(S_ref) == len(ref_off) - 1
        for cuts in cut_sets:
            got = _pushed(bld, xy, t, dt, cuts)
            assert got.shape == S_ref.shape, (cuts[:5], got.shape, S_ref.shape)
            assert np.array_equal(got.view(np.uint8), S_ref.view(np.uint8)), cuts[:5]


def test_stream_windows_against_the_oracle():
    """Spot check of the pushed surfaces against the fp64 oracle (2e-6), including the empty
    interior window (S = 1 everywhere, reading R5)."""
    import paper_2112_10591_b200 as ieds

    xy, t, dt = _stream(DAVIS, 5, 6, drop=(2,))
    off = oracle.window_offsets(t, dt)
    a = oracle.alpha_from_dsat(6.0)
    with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, d_sat=6.0, device=0) as bld:
        got = _pushed(bld, xy, t, dt, [len(t) // 3, len(t) // 2])
    assert len(got) == len(off) - 1
    for k in range(len(got)):
        ref = oracle.build_window(xy[off[k]:off[k + 1]], DAVIS.width, DAVIS.height, 1, 4, a)
        assert np.abs(got[k].astype(np.float64) - ref["S"]).max() <= 2e-6, k
    assert np.all(got[2] == 1.0)   # the dropped window: empty, saturated


def test_stream_rejects_out_of_order_chunks_and_recovers():
    import paper_2112_10591_b200 as ieds

    xy, t, dt = _stream(DAVIS, 9, 5)
    n = len(t)
    with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, d_sat=6.0, device=0) as bld:
        S_ref, _ = _batched(bld, xy, t, dt)
        with bld.stream(dt) as st:
            a = st.push(t[:n // 2], xy[:n // 2])
            # a chunk that starts before the stream's last timestamp: rejected, stream unchanged
            with pytest.raises(ieds.IedsOrderError):
                st.push(t[n // 2 - 10:n // 2 + 5], xy[n // 2 - 10:n // 2 + 5])
            # an inversion inside a chunk (ends ordered): found by the device check, rejected
            bad = t[n // 2:n // 2 + 100].copy()
            bad[41] = bad[40] - 1
            assert bad[0] <= bad[-1]
            with pytest.raises(ieds.IedsOrderError):
                st.push(bad, xy[n // 2:n // 2 + 100])
            b = st.push(t[n // 2:], xy[n // 2:])
            c = st.flush()
        got = np.concatenate([p for p in (a, b, c) if len(p)])
        assert np.array_equal(got, S_ref)


def test_stream_capacity_and_reuse_after_flush():
    """ECAPACITY leaves the stream unchanged; after flush the next push starts a new stream with
    its own t0; ieds_stream_closing counts the windows a push would close."""
    import paper_2112_10591_b200 as ieds
    from paper_2112_10591_b200._lib import IEDS_ECAPACITY, load

    xy, t, dt = _stream(DAVIS, 11, 4)
    lib = load()
    with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, d_sat=6.0, device=0) as bld:
        S_ref, off = _batched(bld, xy, t, dt)
        with bld.stream(dt) as st:
            assert st.closing(int(t[0]), int(t[0])) == 0              # nothing pushed yet
            assert st.closing(int(t[0]), int(t[-1])) == len(off) - 2
            first = st.push(t[:10], xy[:10])
            assert len(first) == 0
            k = st.closing(int(t[10]), int(t[-1]))
            assert k == len(off) - 2                                  # all but the last window
            buf = np.empty((k - 1, DAVIS.height, DAVIS.width), np.float32)
            got = ctypes.c_int32()
            rc = lib.ieds_stream_push(st._s, t[10:].ctypes.data_as(ctypes.c_void_p),
                                      xy[10:].ctypes.data_as(ctypes.c_void_p), len(t) - 10,
                                      buf.ctypes.data_as(ctypes.c_void_p), k - 1, ctypes.byref(got))
            assert rc == IEDS_ECAPACITY and got.value == 0
            rest = st.push(t[10:], xy[10:])
            last = st.flush()
            assert np.array_equal(np.concatenate([rest, last]), S_ref)
            # a second stream on the same object, shifted in time: same surfaces
            again = [st.push(t + 10**9, xy), st.flush()]
            assert np.array_equal(np.concatenate(again), S_ref)


def test_window_count_matches_reading_r16():
    import torch

    import paper_2112_10591_b200 as ieds

    xy, t, dt = _stream(GEN4, 3, 5, drop=(1,))
    dev = torch.device("cuda", 0)
    with ieds.Builder(1280, 720, 2, 3, device=0) as bld:
        t0, K = bld.window_count(torch.from_numpy(t).to(dev), dt)
        assert t0 == int(t[0]) and K == len(oracle.window_offsets(t, dt)) - 1
        assert bld.window_count(torch.zeros(0, dtype=torch.int64, device=dev), dt) == (0, 0)
        with pytest.raises(ieds.IedsOrderError):
            bld.window_count(torch.from_numpy(t[::-1].copy()).to(dev), dt)
