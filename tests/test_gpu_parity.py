"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Bar (BASELINE.json north_star): E, E_d, E_df bit-exact; D2 exact (integer); surface within
max-abs 2e-6 of the oracle's fp64 values.
"""
import numpy as np
import pytest

import oracle
from synth.events import (WORKLOADS, SceneConfig, batch_events, pack_xy, pattern_events,
                          random_frame_events)

pytestmark = pytest.mark.gpu
TOL = 2e-6


def _torch():
    import torch
    return torch


def ieds():
    import paper_2112_10591_b200 as m
    return m


def unpack(bits, W, H):
    nw = (W + 31) // 32
    a = np.ascontiguousarray(bits).view(np.uint32).reshape(H, nw)
    full = np.unpackbits(a.view(np.uint8), bitorder="little").reshape(H, nw * 32)
    assert not full[:, W:].any(), "padding bits must stay 0"
    return full[:, :W]


def run_gpu(xy, off, W, H, n_d, n_f, alpha, chunk=0, xy_shift=0, debug=True, exact_edt=False, bands=False):
    """Run the CUDA path.  With debug=True the intermediate frames and D2 are requested (this
    selects the exact-EDT kernel) and the surface-only call (default streaming kernel) is run
    as well: the two surfaces must be bit-identical."""
    torch = _torch()
    dev = torch.device("cuda", 0)
    B = len(off) - 1
    nw = (W + 31) // 32
    base = torch.zeros(len(xy) + xy_shift + 4, dtype=torch.int32, device=dev)
    if len(xy):
        base[xy_shift:xy_shift + len(xy)] = torch.from_numpy(np.ascontiguousarray(xy).view(np.int32)).to(dev)
    txy = base[xy_shift:xy_shift + len(xy)]
    toff = torch.from_numpy(np.asarray(off, np.int64)).to(dev)
    outs = {}
    if debug:
        for k in ("E", "E_d", "E_df"):
            outs[k] = torch.full((B, H, nw), -1, dtype=torch.int32, device=dev)
        outs["D2"] = torch.full((B, H, W), 7, dtype=torch.int32, device=dev)
    S = torch.full((B, H, W), -5.0, dtype=torch.float32, device=dev)
    S2 = torch.full((B, H, W), -5.0, dtype=torch.float32, device=dev)
    with ieds().Builder(W, H, n_d, n_f, alpha=alpha, chunk_windows=chunk, device=0, exact_edt=exact_edt,
                        _test_bands=bands) as bld:
        bld.build_batch(txy, toff, S2)
        if debug:
            bld.build_batch(txy, toff, S, edge_bits=outs.get("E"), denoised_bits=outs.get("E_d"),
                            filtered_bits=outs.get("E_df"), sqdist=outs.get("D2"))
        bld.sync()
    res = {"S": (S if debug else S2).cpu().numpy()}
    if debug:
        S2 = S2.cpu().numpy()
        bad = S2 != res["S"]
        assert not bad.any(), ("surface-only path differs from the exact path", int(bad.sum()),
                               np.argwhere(bad)[:5])
    for k, v in outs.items():
        res[k] = v.cpu().numpy().view(np.uint32)
    return res


def check_window(gpu, b, xy_w, W, H, n_d, n_f, alpha, debug=True):
    ref = oracle.build_window(xy_w, W, H, n_d, n_f, alpha)
    if debug:
        for k in ("E", "E_d", "E_df"):
            got = unpack(gpu[k][b], W, H)
            assert np.array_equal(got, ref[k]), (k, b, int((got != ref[k]).sum()))
        ref_d2 = np.where(ref["D2"] < 0, 0xFFFFFFFF, ref["D2"]).astype(np.uint32)
        bad = gpu["D2"][b] != ref_d2
        assert not bad.any(), ("D2", b, int(bad.sum()), np.argwhere(bad)[:5])
    err = np.abs(gpu["S"][b].astype(np.float64) - ref["S"])
    assert err.max() <= TOL, ("S", b, float(err.max()))
    # exact structure: 0 exactly on E_df pixels, 1.0 exactly for empty frames
    assert np.all((gpu["S"][b] == 0) == (ref["E_df"] == 1))
    return ref


def csr(windows):
    off = np.zeros(len(windows) + 1, np.int64)
    off[1:] = np.cumsum([len(w) for w in windows])
    xy = np.concatenate(windows).astype(np.uint32) if windows else np.zeros(0, np.uint32)
    return xy, off


# ----------------------------------------------------------------------------- configs

@pytest.mark.parametrize("name,nwin", [("C1", 1), ("C2", 24), ("C3", 6), ("C5", 3)])
def test_parity_workload_configs(name, nwin):
    wl = WORKLOADS[name]
    c = wl.scene
    alpha = oracle.alpha_from_dsat(wl.d_sat)
    xy, off = batch_events(c, wl.seed, 0, nwin)
    gpu = run_gpu(xy, off, c.width, c.height, wl.n_d, wl.n_f, alpha)
    for b in range(nwin):
        check_window(gpu, b, xy[off[b]:off[b + 1]], c.width, c.height, wl.n_d, wl.n_f, alpha)


def test_parity_alpha_printed_value():
    # the paper prints alpha = 1.08; parity must hold for that exact value too
    wl = WORKLOADS["C1"]
    c = wl.scene
    xy, off = batch_events(c, wl.seed, 5, 2)
    gpu = run_gpu(xy, off, c.width, c.height, wl.n_d, wl.n_f, 1.08)
    for b in range(2):
        check_window(gpu, b, xy[off[b]:off[b + 1]], c.width, c.height, wl.n_d, wl.n_f, 1.08)


# ----------------------------------------------------------------------------- edge cases

@pytest.mark.parametrize("W,H", [(1, 1), (1, 40), (37, 1), (33, 17), (64, 64), (346, 260), (100, 70)])
def test_parity_patterns_and_sizes(W, H):
    wins = [pattern_events(W, H, p, seed=i) for i, p in
            enumerate(["empty", "single", "all", "checker", "row", "col", "corners"])]
    for i, d in enumerate([0.001, 0.01, 0.1, 0.3, 0.5]):
        wins.append(random_frame_events(W, H, d, seed=100 + i))
    xy, off = csr(wins)
    for n_d, n_f in [(0, 5), (0, 2), (1, 4), (2, 3)]:
        gpu = run_gpu(xy, off, W, H, n_d, n_f, 1.0827855)
        for b in range(len(wins)):
            check_window(gpu, b, xy[off[b]:off[b + 1]], W, H, n_d, n_f, 1.0827855)


def test_parity_isolated_event_closed_form():
    # single event, N_d = 0, N_f = 2: S(x,y) = 1 - exp(-|(x,y)-(x0,y0)|/alpha)  (Eq. (1))
    W, H, x0, y0 = 300, 200, 123, 77
    alpha = oracle.alpha_from_dsat(6.0)
    xy, off = csr([pack_xy([x0], [y0])])
    gpu = run_gpu(xy, off, W, H, 0, 2, alpha)
    yy, xx = np.mgrid[0:H, 0:W]
    exp = 1.0 - np.exp(-np.hypot(xx - x0, yy - y0) / alpha)
    assert np.abs(gpu["S"][0] - exp).max() <= TOL
    assert gpu["D2"][0][y0, x0] == 0 and gpu["D2"][0][0, 0] == x0 * x0 + y0 * y0


def test_parity_max_distance_corners():
    # two far corner points: maximal D2 = (W-1)^2 + (H-1)^2 is reached at the far corners
    W, H = 1280, 720
    xy, off = csr([pack_xy([0], [0])])
    gpu = run_gpu(xy, off, W, H, 0, 5, 2.0)
    assert gpu["D2"][0][H - 1, W - 1] == (W - 1) ** 2 + (H - 1) ** 2
    check_window(gpu, 0, xy, W, H, 0, 5, 2.0)


def test_parity_parameter_grid():
    # sensitivity grid of Fig. 9: N_d 0-4, N_f 1-5, d_sat 3/6/9/12
    W, H = 83, 61
    wins = [random_frame_events(W, H, d, seed=200 + i) for i, d in enumerate([0.02, 0.15, 0.4])]
    xy, off = csr(wins)
    for n_d in range(5):
        for n_f in range(1, 6):
            for d_sat in (3.0, 6.0, 9.0, 12.0):
                a = oracle.alpha_from_dsat(d_sat)
                gpu = run_gpu(xy, off, W, H, n_d, n_f, a)
                for b in range(len(wins)):
                    check_window(gpu, b, xy[off[b]:off[b + 1]], W, H, n_d, n_f, a)


def test_parity_large_alpha_mufu_path():
    # alpha large enough that the saturation index exceeds the 1024-entry table
    W, H = 200, 150
    xy, off = csr([random_frame_events(W, H, 0.002, seed=9)])
    for a in (10.0, 40.0):
        gpu = run_gpu(xy, off, W, H, 0, 5, a)
        check_window(gpu, 0, xy, W, H, 0, 5, a)


# ----------------------------------------------------------------------------- batching

def test_chunking_and_ragged_windows_identical():
    cfg = SceneConfig(346, 260, 20_000, n_prims=28, len_range=(15.0, 120.0), sigma=0.45,
                      count_jitter=0.9)
    xy, off = batch_events(cfg, 77, 0, 11)
    # insert empty windows
    off = np.concatenate([off[:3], [off[2]], off[3:7], [off[6], off[6]], off[7:]])
    a = oracle.alpha_from_dsat(6.0)
    g1 = run_gpu(xy, off, 346, 260, 1, 4, a, chunk=0)
    g2 = run_gpu(xy, off, 346, 260, 1, 4, a, chunk=3, xy_shift=1)   # unaligned events, 5 chunks
    for k in g1:
        assert np.array_equal(g1[k], g2[k]), k
    for b in range(len(off) - 1):
        check_window(g1, b, xy[off[b]:off[b + 1]], 346, 260, 1, 4, a)


def test_surface_only_path_matches_debug_path():
    wl = WORKLOADS["C3"]
    c = wl.scene
    a = oracle.alpha_from_dsat(wl.d_sat)
    xy, off = batch_events(c, wl.seed, 10, 4)
    g1 = run_gpu(xy, off, c.width, c.height, wl.n_d, wl.n_f, a, debug=True)
    g2 = run_gpu(xy, off, c.width, c.height, wl.n_d, wl.n_f, a, debug=False)
    assert np.array_equal(g1["S"], g2["S"])


def test_host_entry_point_matches_device():
    wl = WORKLOADS["C1"]
    c = wl.scene
    a = oracle.alpha_from_dsat(wl.d_sat)
    xy, off = batch_events(c, wl.seed, 0, 9)
    g = run_gpu(xy, off, c.width, c.height, wl.n_d, wl.n_f, a, debug=False)
    with ieds().Builder(c.width, c.height, wl.n_d, wl.n_f, alpha=a, chunk_windows=4, device=0) as bld:
        S = bld.build_batch_host(xy, off)
    assert np.array_equal(S, g["S"])


# ----------------------------------------------------------------------------- errors

def test_out_of_frame_event_latched_and_dropped():
    torch = _torch()
    ie = ieds()
    W, H = 64, 32
    good = random_frame_events(W, H, 0.2, seed=1)
    bad = np.concatenate([good, pack_xy([W], [0]), pack_xy([0], [H])])
    xy, off = csr([bad])
    dev = torch.device("cuda", 0)
    with ie.Builder(W, H, 0, 5, alpha=1.0, device=0) as bld:
        S = bld.build_batch(torch.from_numpy(xy.view(np.int32)).to(dev), torch.from_numpy(off).to(dev))
        with pytest.raises(ie.IedsRangeError):
            bld.sync()
        bld.sync()   # cleared
        ref = oracle.build_window(good, W, H, 0, 5, 1.0)
        assert np.abs(S.cpu().numpy()[0] - ref["S"]).max() <= TOL
        off_bad = torch.tensor([0, 5, 3], dtype=torch.int64, device=dev)
        bld.build_batch(torch.from_numpy(xy.view(np.int32)).to(dev), off_bad)
        with pytest.raises(ie.IedsOrderError):
            bld.sync()


def test_invalid_configs_rejected():
    ie = ieds()
    for args in [(0, 10, 1, 4), (10, 0, 1, 4), (10, 10, 5, 4), (10, 10, 1, 0), (10, 10, 1, 6),
                 (5000, 10, 1, 4), (10, 5000, 1, 4)]:
        with pytest.raises(ie.IedsError):
            ie.Builder(*args, alpha=1.0, device=0)
    with pytest.raises(ie.IedsError):
        ie.Builder(10, 10, 1, 4, alpha=-1.0, device=0)


# ----------------------------------------------------------------------------- full size

def test_full_size_bench_config_sampled():
    """C3 at its full BASELINE size (1000 windows) in the bench launch configuration; a
    sample of windows across all chunks is checked against the oracle one by one."""
    torch = _torch()
    wl = WORKLOADS["C3"]
    c = wl.scene
    a = oracle.alpha_from_dsat(wl.d_sat)
    xy, off = batch_events(c, wl.seed, 0, wl.n_windows)
    dev = torch.device("cuda", 0)
    with ieds().Builder(c.width, c.height, wl.n_d, wl.n_f, alpha=a, device=0) as bld:
        S = bld.build_batch(torch.from_numpy(xy.view(np.int32)).to(dev), torch.from_numpy(off).to(dev))
        bld.sync()
    sample = [0, 1, 147, 148, 295, 296, 511, 700, 888, 999]
    Sh = S[sample].cpu().numpy()
    refs = oracle.build_batch(xy, off, c.width, c.height, wl.n_d, wl.n_f, a, windows=sample,
                              want=("S", "E_df"))
    for i, b in enumerate(sample):
        err = np.abs(Sh[i].astype(np.float64) - refs[i]["S"]).max()
        assert err <= TOL, (b, err)
        assert np.all((Sh[i] == 0) == (refs[i]["E_df"] == 1))


def test_c5_bulk_launch_sampled():
    """C5 (the dense burst, 300k events per window) in the bench's bulk launch configuration: 296
    windows (two waves of frame CTAs, so the events of the next wave are L2-prefetched, capped per
    window) cycling 12 generated windows, sampled against the oracle; surfaces also bit-identical
    to the exact-EDT kernel's."""
    torch = _torch()
    wl = WORKLOADS["C5"]
    c = wl.scene
    a = oracle.alpha_from_dsat(wl.d_sat)
    xy0, off0 = batch_events(c, wl.seed, 100, 12)
    ws = [xy0[off0[i % 12]:off0[i % 12 + 1]] for i in range(296)]
    xy, off = csr(ws)
    dev = torch.device("cuda", 0)
    txy, toff = torch.from_numpy(xy.view(np.int32)).to(dev), torch.from_numpy(off).to(dev)
    with ieds().Builder(c.width, c.height, wl.n_d, wl.n_f, alpha=a, device=0) as bld:
        S = bld.build_batch(txy, toff)
        bld.sync()
    with ieds().Builder(c.width, c.height, wl.n_d, wl.n_f, alpha=a, device=0, exact_edt=True) as bx:
        Sx = bx.build_batch(txy, toff)
        bx.sync()
    assert torch.equal(S, Sx)
    for b in (0, 5, 147, 148, 150, 295):
        ref = oracle.build_window(ws[b], c.width, c.height, wl.n_d, wl.n_f, a, want=("S",))["S"]
        assert np.abs(S[b].cpu().numpy().astype(np.float64) - ref).max() <= TOL, b


# ----------------------------------------------------------------------------- streaming vs exact

def _stress_windows(W, H, seed):
    rng = np.random.default_rng(seed)
    wins = []
    yy, xx = np.mgrid[0:H, 0:W]
    masks = [
        (yy % 23 == 0), (xx % 29 == 0), ((xx + yy) % 37 == 0), ((xx - 2 * yy) % 41 == 0),
        (yy == H // 2) & (xx % 3 == 0), ((xx // 7 + yy // 5) % 2 == 0) & (rng.random((H, W)) < 0.05),
        rng.random((H, W)) < 0.0005, rng.random((H, W)) < 0.003, rng.random((H, W)) < 0.02,
        (np.hypot(xx - W / 2, yy - H / 2).astype(int) % 31 == 0),
    ]
    for m in masks:
        ys, xs = np.nonzero(m)
        wins.append(pack_xy(xs, ys))
    return wins


@pytest.mark.parametrize("d_sat", [1.0, 3.0, 6.0, 8.0, 9.5, 11.0, 12.0])
def test_streaming_surface_bit_identical_to_exact(d_sat):
    """The saturation-aware streaming kernel (default when D2 is not requested) must produce the
    same fp32 surface bits as the exact-EDT kernel, for every saturation radius it serves."""
    W, H = 300, 211
    wins = _stress_windows(W, H, int(d_sat * 10))
    xy, off = csr(wins)
    a = oracle.alpha_from_dsat(d_sat)
    g_stream = run_gpu(xy, off, W, H, 0, 5, a, debug=False)
    g_exact = run_gpu(xy, off, W, H, 0, 5, a, debug=False, exact_edt=True)
    assert np.array_equal(g_stream["S"], g_exact["S"])
    for b in (0, 6, 9):
        ref = oracle.build_window(xy[off[b]:off[b + 1]], W, H, 0, 5, a)
        assert np.abs(g_stream["S"][b] - ref["S"]).max() <= TOL


# ----------------------------------------------------------------------------- banded frames

@pytest.mark.parametrize("name,nwin", [("C1", 4), ("C3", 2), ("C5", 1)])
def test_banded_frame_kernel_forced(name, nwin):
    """IEDS_FLAG_TEST_BANDS splits the frame into 64-row bands (one CTA each, halo of 2 rows):
    E / E_d / E_df / D2 bit-exact and the surface within 2e-6 on both the exact and the
    streaming path, exactly as with one band."""
    wl = WORKLOADS[name]
    c = wl.scene
    a = oracle.alpha_from_dsat(wl.d_sat)
    xy, off = batch_events(c, wl.seed, 11, nwin)
    gpu = run_gpu(xy, off, c.width, c.height, wl.n_d, wl.n_f, a, bands=True)
    one = run_gpu(xy, off, c.width, c.height, wl.n_d, wl.n_f, a, bands=False)
    for b in range(nwin):
        check_window(gpu, b, xy[off[b]:off[b + 1]], c.width, c.height, wl.n_d, wl.n_f, a)
    for k in ("S", "E", "E_d", "E_df", "D2"):
        assert np.array_equal(gpu[k], one[k]), k


def test_full_hd_1920x1080_uses_bands():
    """1920x1080 does not fit one CTA's shared memory: the frame kernel splits it into row
    bands.  Parity against the oracle on two windows of a Gen4-like scene at that size."""
    c = SceneConfig(1920, 1080, 150_000, n_prims=140, len_range=(30.0, 300.0), sigma=0.55,
                    noise_frac=0.10, vmax=8.0, dt_us=15000)
    a = oracle.alpha_from_dsat(6.0)
    xy, off = batch_events(c, 21, 0, 2)
    gpu = run_gpu(xy, off, c.width, c.height, 2, 3, a)
    for b in range(2):
        check_window(gpu, b, xy[off[b]:off[b + 1]], c.width, c.height, 2, 3, a)


def test_largest_frames_create():
    """The header's largest geometry (4096 x 2048) builds a handle and an empty window."""
    torch = _torch()
    with ieds().Builder(4096, 2048, 1, 4, device=0) as bld:
        S = bld.build_batch(torch.zeros(4, dtype=torch.int32, device="cuda"),
                            torch.zeros(2, dtype=torch.int64, device="cuda"))
        bld.sync()
        assert bool((S == 1.0).all())



def test_small_batch_bands_match_bulk_batch():
    """Row f2 latency mode: a batch smaller than the GPU spreads each window over row bands
    (frame kernel and window kernel); the same windows inside a 300-window batch use one band
    each.  Surfaces (and, on the exact path, D2) are identical bit for bit."""
    torch = _torch()
    wl = WORKLOADS["C3"]
    c = wl.scene
    a = oracle.alpha_from_dsat(wl.d_sat)
    xy, off = batch_events(c, wl.seed, 200, 300)
    dev = torch.device("cuda", 0)
    txy = torch.from_numpy(xy.view(np.int32)).to(dev)
    toff = torch.from_numpy(off).to(dev)
    pick = [0, 137, 299]
    with ieds().Builder(c.width, c.height, wl.n_d, wl.n_f, alpha=a, device=0) as bld:
        S_all = bld.build_batch(txy, toff)
        D_all = torch.empty((300, c.height, c.width), dtype=torch.int32, device=dev)
        bld.build_batch(txy, toff, sqdist=D_all)
        for k in pick:
            one = torch.tensor([0, int(off[k + 1] - off[k])], dtype=torch.int64, device=dev)
            ev = txy[int(off[k]):int(off[k + 1])]
            S1 = bld.build_batch(ev, one)
            D1 = torch.empty((1, c.height, c.width), dtype=torch.int32, device=dev)
            bld.build_batch(ev, one, sqdist=D1)
            bld.sync()
            assert torch.equal(S1[0], S_all[k]), k
            assert torch.equal(D1[0], D_all[k]), k
    ref = oracle.build_window(xy[off[0]:off[1]], c.width, c.height, wl.n_d, wl.n_f, a)
    assert np.abs(S_all[0].cpu().numpy().astype(np.float64) - ref["S"]).max() <= TOL


@pytest.mark.parametrize("name,nwin,d_sat", [("C2", 300, None), ("C3", 20, None), ("C1", 7, 12.0), ("C2", 5, 2.5)])
def test_packed_window_ctas_bit_identical(name, nwin, d_sat, monkeypatch):
    """Packed window-kernel CTAs (8 strips of consecutive windows, per-warp staging; the default
    for narrow frames such as 346 wide) against per-window CTAs (forced with IEDS_WIN_PACKED,
    read at create): surfaces identical bit for bit, in bulk and small batches (row bands), at
    C3 width too, and for d_sat = 12 (C = 31, the widest one-word window)."""
    torch = _torch()
    wl = WORKLOADS[name]
    c = wl.scene
    a = oracle.alpha_from_dsat(d_sat if d_sat is not None else wl.d_sat)
    xy, off = batch_events(c, wl.seed, 300, nwin)
    dev = torch.device("cuda", 0)
    txy = torch.from_numpy(xy.view(np.int32)).to(dev)
    toff = torch.from_numpy(off).to(dev)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("IEDS_WIN_PACKED", mode)
        with ieds().Builder(c.width, c.height, wl.n_d, wl.n_f, alpha=a, device=0) as bld:
            S = bld.build_batch(txy, toff)
            one = torch.tensor([0, int(off[1] - off[0])], dtype=torch.int64, device=dev)
            S1 = bld.build_batch(txy[:int(off[1])], one)
            bld.sync()
        out[mode] = (S, S1)
    assert torch.equal(out["0"][0], out["1"][0])
    assert torch.equal(out["0"][1], out["1"][1])
    assert torch.equal(out["1"][1][0], out["1"][0][0])
    k = nwin // 2
    check_window({"S": out["1"][0].cpu().numpy()}, k, xy[off[k]:off[k + 1]], c.width, c.height, wl.n_d, wl.n_f, a,
                 debug=False)


@pytest.mark.parametrize("name,nwin,chunk", [("C2", 40, 6), ("C2", 23, 0), ("C1", 17, 4)])
def test_chunk_overlap_bit_identical(name, nwin, chunk, monkeypatch):
    """Small frames, several chunks per build_batch: the frame kernel of chunk c + 1 runs on a side
    stream under the window kernel of chunk c, into a second E_df scratch set (ieds_build_batch).
    Against the serial chunk order (IEDS_CHUNK_OVERLAP=0, read at create): identical bit for bit,
    with empty windows and a ragged last chunk, repeated back to back on one handle (the set a
    frame kernel writes was read by the window kernel two chunks earlier); one window per chunk
    against the oracle."""
    torch = _torch()
    wl = WORKLOADS[name]
    c = wl.scene
    a = oracle.alpha_from_dsat(wl.d_sat)
    xy, off = batch_events(c, wl.seed, 40, nwin)
    off = np.concatenate([off[:5], [off[4], off[4]], off[5:]])   # two empty windows
    B = len(off) - 1
    dev = torch.device("cuda", 0)
    txy = torch.from_numpy(xy.view(np.int32)).to(dev)
    toff = torch.from_numpy(off).to(dev)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("IEDS_CHUNK_OVERLAP", mode)
        with ieds().Builder(c.width, c.height, wl.n_d, wl.n_f, alpha=a, chunk_windows=chunk, device=0) as bld:
            S = [bld.build_batch(txy, toff) for _ in range(3)]
            bld.sync()
        assert torch.equal(S[0], S[1]) and torch.equal(S[0], S[2])
        out[mode] = S[0]
    assert torch.equal(out["0"], out["1"])
    step = chunk if chunk else B
    for b in list(range(0, B, max(1, step)))[:6] + [B - 1]:
        check_window({"S": out["1"].cpu().numpy()}, b, xy[off[b]:off[b + 1]], c.width, c.height, wl.n_d, wl.n_f,
                     a, debug=False)


def test_multi_chunk_batch_captured_in_cuda_graph():
    """ieds_build_batch enqueues only (no host sync, no allocation), also when it forks the next
    chunk's frame kernel onto its side stream: the whole multi-chunk call captured in a CUDA graph
    (the side stream joins the capture through the fork event and is joined back at the end) and
    replayed gives the directly launched surfaces bit for bit, for two different input batches
    copied into the graph's static buffers."""
    torch = _torch()
    wl = WORKLOADS["C2"]
    c = wl.scene
    a = oracle.alpha_from_dsat(wl.d_sat)
    dev = torch.device("cuda", 0)
    batches = []
    for k0 in (0, 50):
        xy, off = batch_events(c, wl.seed, k0, 13)
        batches.append((torch.from_numpy(xy.view(np.int32)).to(dev), torch.from_numpy(off).to(dev), xy, off))
    n_max = max(int(b[3][-1]) for b in batches)
    with ieds().Builder(c.width, c.height, wl.n_d, wl.n_f, alpha=a, chunk_windows=4, device=0) as bld:
        direct = []
        for txy, toff, _, _ in batches:
            direct.append(bld.build_batch(txy, toff).clone())
        bld.sync()
        g_xy = torch.zeros(n_max, dtype=torch.int32, device=dev)
        g_off = torch.zeros_like(batches[0][1])
        S = torch.empty((13, c.height, c.width), dtype=torch.float32, device=dev)
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(cap):
            bld.build_batch(g_xy, g_off, S)   # warm-up on the capture stream
        cap.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            bld.build_batch(g_xy, g_off, S)
        for (txy, toff, xy, off), ref in zip(batches, direct):
            g_xy[:txy.numel()].copy_(txy)
            g_off.copy_(toff)
            graph.replay()
            torch.cuda.synchronize(dev)
            assert torch.equal(S, ref)
        bld.sync()
    b = 7
    check_window({"S": direct[1].cpu().numpy()}, b, batches[1][2][batches[1][3][b]:batches[1][3][b + 1]], c.width,
                 c.height, wl.n_d, wl.n_f, a, debug=False)


def test_c4_on_one_gpu_two_chunks_sampled():
    """BASELINE's C4 batch (16,000 Gen4 windows) on one GPU in the bench's launch configuration
    (bench.py c4_r1_baseline): the default chunk splits it into two launch pairs, the second
    chunk's frame kernel overlapping the first chunk's window kernel.  Windows cycle 64 generated
    ones; every sampled window (both chunks, both sides of the chunk edge) equals the same window
    built alone, bit for bit, and two are checked against the oracle."""
    torch = _torch()
    wl = WORKLOADS["C4"]
    c = wl.scene
    a = oracle.alpha_from_dsat(wl.d_sat)
    pool = 64
    xy0, off0 = batch_events(c, wl.seed, 200, pool)
    lens = np.diff(off0)
    n = 16_000
    reps = n // pool
    dev = torch.device("cuda", 0)
    txy = torch.from_numpy(xy0.view(np.int32)).to(dev).repeat(reps)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(np.tile(lens, reps))
    toff = torch.from_numpy(off).to(dev)
    with ieds().Builder(c.width, c.height, wl.n_d, wl.n_f, alpha=a, device=0) as bld:
        assert bld.launches_per_batch(n) == 4   # two chunks
        S = bld.build_batch(txy, toff)
        Sp = bld.build_batch(torch.from_numpy(xy0.view(np.int32)).to(dev), torch.from_numpy(off0).to(dev))
        bld.sync()
    for b in (0, 63, 5000, 10803, 10804, 10805, 12345, 15999):
        assert torch.equal(S[b], Sp[b % pool]), b
    for b in (10803, 10804):
        ref = oracle.build_window(xy0[off0[b % pool]:off0[b % pool + 1]], c.width, c.height, wl.n_d, wl.n_f, a,
                                  want=("S",))["S"]
        assert np.abs(S[b].cpu().numpy().astype(np.float64) - ref).max() <= TOL, b


@pytest.mark.parametrize("env", [{"IEDS_FRAME_THREADS": "256"}, {"IEDS_FRAME_THREADS": "640"},
                                 {"IEDS_FRAME_PREFETCH": "0"}])
def test_frame_kernel_knobs_bit_identical(env, monkeypatch):
    """The frame kernel's A/B knobs (block size, read per launch; the L2 prefetch of the next
    wave's events) change the schedule, never the bits: 160 C3 windows (more than one wave of
    frame CTAs, so windows are prefetched) against the default launch."""
    torch = _torch()
    wl = WORKLOADS["C3"]
    c = wl.scene
    a = oracle.alpha_from_dsat(wl.d_sat)
    xy0, off0 = batch_events(c, wl.seed, 400, 16)
    ws = [xy0[off0[i % 16]:off0[i % 16 + 1]] for i in range(160)]
    xy, off = csr(ws)
    dev = torch.device("cuda", 0)
    txy, toff = torch.from_numpy(xy.view(np.int32)).to(dev), torch.from_numpy(off).to(dev)
    out = []
    for knobs in ({}, env):
        for k, v in knobs.items():
            monkeypatch.setenv(k, v)
        with ieds().Builder(c.width, c.height, wl.n_d, wl.n_f, alpha=a, device=0) as bld:
            S = bld.build_batch(txy, toff)
            bld.sync()
        out.append(S)
    assert torch.equal(out[0], out[1])
