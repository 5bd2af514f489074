"""GPU parity of SURVEY §8 row f1: the ablation transfers of §IV-D (Fig. 4) and the
8-bit coded surface, against the oracle, on both the default (saturation-aware, when
the transfer saturates) and the exact-EDT kernel.

Tolerances: 8-bit codes are bit-exact (both sides round the fp64 value); fp32 transfers within
atol 2e-6 + rtol 2^-23 (one rounding of a value up to ~1.5e3 for Id(d)).
"""
import numpy as np
import pytest

import oracle
from synth.events import WORKLOADS, batch_events, pattern_events, random_frame_events

pytestmark = pytest.mark.gpu


def _run(xy, off, W, H, n_d, n_f, transfer, out, with_d2, bound=6.0, d_sat=6.0):
    import torch

    import paper_2112_10591_b200 as ieds

    dev = torch.device("cuda", 0)
    B = len(off) - 1
    txy = torch.from_numpy(np.ascontiguousarray(xy).view(np.int32)).to(dev)
    toff = torch.from_numpy(np.asarray(off, np.int64)).to(dev)
    d2 = torch.empty((B, H, W), dtype=torch.int32, device=dev) if with_d2 else None
    with ieds.Builder(W, H, n_d, n_f, d_sat=d_sat, device=0, transfer=transfer, bound=bound, out=out) as bld:
        S = bld.build_batch(txy, toff, sqdist=d2)
        bld.sync()
    return S.cpu().numpy(), (d2.cpu().numpy().view(np.uint32) if with_d2 else None)


def _windows():
    wl = WORKLOADS["C1"]
    c = wl.scene
    xy, off = batch_events(c, wl.seed, 3, 3)
    wins = [xy[off[b]:off[b + 1]] for b in range(3)]
    wins += [pattern_events(c.width, c.height, "empty"), pattern_events(c.width, c.height, "corners"),
             random_frame_events(c.width, c.height, 0.003, seed=5)]
    off = np.zeros(len(wins) + 1, np.int64)
    off[1:] = np.cumsum([len(w) for w in wins])
    return np.concatenate(wins).astype(np.uint32), off, c.width, c.height


@pytest.mark.parametrize("transfer", ["invexp", "linear", "bounded", "log"])
def test_transfer_variants_f32(transfer):
    xy, off, W, H = _windows()
    a = oracle.alpha_from_dsat(6.0)
    S_def, _ = _run(xy, off, W, H, 0, 5, transfer, "f32", with_d2=False)
    S_exact, D2 = _run(xy, off, W, H, 0, 5, transfer, "f32", with_d2=True)
    for b in range(len(off) - 1):
        ref = oracle.build_window(xy[off[b]:off[b + 1]], W, H, 0, 5, a)
        exp = oracle.transfer(ref["D2"], transfer, alpha=a, bound=6.0)
        for S in (S_def[b], S_exact[b]):
            fin = np.isfinite(exp)
            assert np.array_equal(np.isinf(S), ~fin), (transfer, b)
            err = np.abs(S[fin].astype(np.float64) - exp[fin])
            assert np.all(err <= 2e-6 + np.abs(exp[fin]) * 2.0 ** -23), (transfer, b, float(err.max()))
    assert np.array_equal(S_def, S_exact)   # both kernels give the same fp32 bits


def test_surface_u8_bit_exact():
    xy, off, W, H = _windows()
    a = oracle.alpha_from_dsat(6.0)
    Q_def, _ = _run(xy, off, W, H, 1, 4, "invexp", "u8", with_d2=False)
    Q_exact, _ = _run(xy, off, W, H, 1, 4, "invexp", "u8", with_d2=True)
    assert Q_def.dtype == np.uint8
    for b in range(len(off) - 1):
        ref = oracle.build_window(xy[off[b]:off[b + 1]], W, H, 1, 4, a)
        q = oracle.quantize_u8(ref["S"])
        assert np.array_equal(Q_def[b], q), b
        assert np.array_equal(Q_exact[b], q), b


def test_u8_workload_c3_sampled():
    wl = WORKLOADS["C3"]
    c = wl.scene
    a = oracle.alpha_from_dsat(wl.d_sat)
    xy, off = batch_events(c, wl.seed, 40, 4)
    Q, _ = _run(xy, off, c.width, c.height, wl.n_d, wl.n_f, "invexp", "u8", with_d2=False)
    for b in range(4):
        ref = oracle.build_window(xy[off[b]:off[b + 1]], c.width, c.height, wl.n_d, wl.n_f, a)
        assert np.array_equal(Q[b], oracle.quantize_u8(ref["S"])), b


# ----------------------------------------------------------------------------- row f2

def _stream(n_win=6, dt=15000):
    """A time-ordered Gen4-like stream: the generator's windows k laid end to end in time,
    with one empty interior window (events of window 3 dropped)."""
    from synth.events import GEN4, window_events

    xs, ts = [], []
    for k in range(n_win):
        xy, t, _ = window_events(GEN4, 3, k, with_tp=True)
        if k == 3:
            continue
        xs.append(xy)
        ts.append(t)
    return np.concatenate(xs), np.concatenate(ts), dt


def test_window_offsets_match_oracle_and_build():
    import torch

    import paper_2112_10591_b200 as ieds

    xy, t, dt = _stream()
    ref_off = oracle.window_offsets(t, dt)
    dev = torch.device("cuda", 0)
    with ieds.Builder(1280, 720, 2, 3, d_sat=6.0, device=0) as bld:
        off = bld.window_offsets(torch.from_numpy(t).to(dev), dt)
        S = bld.build_batch(torch.from_numpy(xy.view(np.int32)).to(dev), off)
        bld.sync()
        got = off.cpu().numpy()
        assert np.array_equal(got, ref_off)
        assert got[4] == got[3]                       # the empty interior window is emitted
        a = oracle.alpha_from_dsat(6.0)
        S = S.cpu().numpy()
        for k in (0, 3, 5):
            ref = oracle.build_window(xy[ref_off[k]:ref_off[k + 1]], 1280, 720, 2, 3, a)
            assert np.abs(S[k] - ref["S"]).max() <= 2e-6
        # unordered timestamps are latched as an ordering error
        bad = t.copy()
        bad[10], bad[11] = bad[11] + 1, bad[10]
        bld.window_offsets(torch.from_numpy(bad).to(dev), dt)
        with pytest.raises(ieds.IedsOrderError):
            bld.sync()


# ----------------------------------------------------------------------------- row f1: fp16 and normalised 8-bit

def _windows_all():
    """_windows() plus an all-set frame (every pixel an edge pixel: D2 = 0 everywhere)."""
    xy, off, W, H = _windows()
    full = pattern_events(W, H, "all")
    xy2 = np.concatenate([xy, full]).astype(np.uint32)
    off2 = np.concatenate([off, [off[-1] + len(full)]]).astype(np.int64)
    return xy2, off2, W, H


@pytest.mark.parametrize("transfer", ["invexp", "linear", "bounded", "log"])
def test_transfer_variants_f16(transfer):
    """float16 surfaces: the fp64 transfer value rounded to nearest even (numpy's float16
    conversion) -- bit for bit from the fp64 table and at saturation; beyond the table (Id
    and ln only, exact kernel) the fp32 value rounded to fp16, within one fp16 ulp."""
    xy, off, W, H = _windows()
    a = oracle.alpha_from_dsat(6.0)
    S_def, _ = _run(xy, off, W, H, 0, 5, transfer, "f16", with_d2=False)
    S_exact, D2 = _run(xy, off, W, H, 0, 5, transfer, "f16", with_d2=True)
    assert S_def.dtype == np.float16
    for b in range(len(off) - 1):
        ref = oracle.build_window(xy[off[b]:off[b + 1]], W, H, 0, 5, a)
        exp16 = oracle.transfer(ref["D2"], transfer, alpha=a, bound=6.0).astype(np.float16)
        in_table = (ref["D2"] >= 0) & (ref["D2"] < 1024)
        for S in (S_def[b], S_exact[b]):
            same = S.view(np.uint16) == exp16.view(np.uint16)
            if transfer in ("invexp", "bounded"):
                assert same.all(), (transfer, b)
            else:
                assert same[in_table].all() and np.array_equal(np.isinf(S), np.isinf(exp16)), (transfer, b)
                fin = np.isfinite(exp16)
                ulp = np.spacing(np.abs(exp16[fin])).astype(np.float64)
                assert np.all(np.abs(S[fin].astype(np.float64) - exp16[fin].astype(np.float64)) <= ulp), (transfer, b)
    if transfer in ("invexp", "bounded"):
        assert np.array_equal(S_def.view(np.uint16), S_exact.view(np.uint16))


@pytest.mark.parametrize("transfer", ["linear", "bounded", "log"])
def test_u8_normalised_by_frame_max_bit_exact(transfer):
    """8-bit view of the ablation transfers normalised by the frame maximum (SPEC S:254,
    S:271, R17): bit-exact against the oracle, including the empty (255) and all-edge (0)
    frames; identical with and without the D2 output."""
    xy, off, W, H = _windows_all()
    a = oracle.alpha_from_dsat(6.0)
    Q, _ = _run(xy, off, W, H, 0, 5, transfer, "u8", with_d2=False, bound=4.0)
    Q2, D2 = _run(xy, off, W, H, 0, 5, transfer, "u8", with_d2=True, bound=4.0)
    assert Q.dtype == np.uint8 and np.array_equal(Q, Q2)
    for b in range(len(off) - 1):
        ref = oracle.build_window(xy[off[b]:off[b + 1]], W, H, 0, 5, a)
        assert np.array_equal(D2[b].astype(np.int64), np.where(ref["D2"] < 0, 0xFFFFFFFF, ref["D2"]))
        assert np.array_equal(Q[b], oracle.quantize_norm_u8(ref["D2"], transfer, bound=4.0)), (transfer, b)
    assert (Q[3] == 255).all()      # the empty window
    assert (Q[-1] == 0).all()       # every pixel an edge pixel


def test_u8_normalised_workload_c3_sampled():
    wl = WORKLOADS["C3"]
    c = wl.scene
    a = oracle.alpha_from_dsat(wl.d_sat)
    xy, off = batch_events(c, wl.seed, 70, 3)
    Q, _ = _run(xy, off, c.width, c.height, wl.n_d, wl.n_f, "log", "u8", with_d2=False)
    for b in range(3):
        ref = oracle.build_window(xy[off[b]:off[b + 1]], c.width, c.height, wl.n_d, wl.n_f, a)
        assert np.array_equal(Q[b], oracle.quantize_norm_u8(ref["D2"], "log")), b


@pytest.mark.parametrize("out", ["u8", "f16"])
def test_variants_bulk_batch_sampled(out):
    """u8 / f16 in the bulk launch configuration (300 windows: one row band per window, the
    shape bench.py times) -- sampled windows against the oracle, bit-exact."""
    import torch

    import paper_2112_10591_b200 as ieds

    wl = WORKLOADS["C3"]
    c = wl.scene
    a = oracle.alpha_from_dsat(wl.d_sat)
    xy, off = batch_events(c, wl.seed, 400, 300)
    dev = torch.device("cuda", 0)
    with ieds.Builder(c.width, c.height, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=0, out=out) as bld:
        Q = bld.build_batch(torch.from_numpy(xy.view(np.int32)).to(dev), torch.from_numpy(off).to(dev))
        bld.sync()
    for b in (0, 151, 299):
        ref = oracle.build_window(xy[off[b]:off[b + 1]], c.width, c.height, wl.n_d, wl.n_f, a)
        got = Q[b].cpu().numpy()
        if out == "u8":
            assert np.array_equal(got, oracle.quantize_u8(ref["S"])), b
        else:
            exp16 = ref["S"].astype(np.float16)
            assert np.array_equal(got.view(np.uint16), exp16.view(np.uint16)), b


@pytest.mark.parametrize("out", ["u8", "f16"])
def test_host_entry_point_variants_match_device(out):
    """ieds_build_batch_host (pinned copies pipelined with the kernels over several chunks)
    returns the same u8 / f16 surfaces as the device entry point."""
    import torch

    import paper_2112_10591_b200 as ieds

    wl = WORKLOADS["C1"]
    c = wl.scene
    xy, off = batch_events(c, wl.seed, 30, 9)
    dev = torch.device("cuda", 0)
    with ieds.Builder(c.width, c.height, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=0, out=out,
                      chunk_windows=4) as bld:
        Sd = bld.build_batch(torch.from_numpy(xy.view(np.int32)).to(dev), torch.from_numpy(off).to(dev))
        bld.sync()
        Sh = bld.build_batch_host(xy, off)
    assert Sh.dtype == {"u8": np.uint8, "f16": np.float16}[out]
    assert np.array_equal(Sd.cpu().numpy().view(np.uint8), Sh.view(np.uint8))


def test_window_order_check_every_boundary():
    """The order check of ieds_window_offsets (16-byte pair loads, the previous element from the
    lane below): one inversion placed inside a pair, between pairs, across lane, warp-chunk
    and grid-iteration boundaries and at the unpaired last element, on 16-byte aligned and
    misaligned streams of odd and even length, is latched exactly when present; ordered streams
    give the oracle's offsets."""
    import torch

    import paper_2112_10591_b200 as ieds

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    dt = 1000
    with ieds.Builder(64, 48, 1, 4, device=0) as bld:
        for n in (1, 2, 3, 257, 4096, 300001):
            t = np.sort(rng.integers(0, 50 * dt, n)).astype(np.int64)
            for shift in (0, 1):                       # 16-byte aligned / 8-byte aligned start
                base = torch.zeros(n + 2, dtype=torch.int64, device=dev)
                base[shift:shift + n] = torch.from_numpy(t).to(dev)
                tt = base[shift:shift + n]
                off = bld.window_offsets(tt, dt)
                bld.sync()
                assert np.array_equal(off.cpu().numpy(), oracle.window_offsets(t, dt)), (n, shift)
                for i in sorted({1, 2, 63, 64, 65, 255, 256, 257, n - 1} & set(range(1, n))):
                    bad = t.copy()
                    bad[i] = bad[i - 1] - 1                # t[i] < t[i-1]
                    base[shift:shift + n] = torch.from_numpy(bad).to(dev)
                    bld.window_offsets(tt, dt)
                    with pytest.raises(ieds.IedsOrderError):
                        bld.sync()
