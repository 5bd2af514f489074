#!/usr/bin/env python
"""Small invocations of every kernel of libieds.so, for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck).  Each case is tiny so the instrumented run stays short; the
results are compared with the oracle where one exists, so a sanitizer-clean run is also a
correct one.  Run as `compute-sanitizer --tool <tool> python tools/sanitize_cases.py [case ...]`
(tools/sanitize.sh runs all four tools over all cases).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2112_10591_b200 as ieds  # noqa: E402
from synth.events import DAVIS, GEN4, batch_events, window_events  # noqa: E402

dev = torch.device("cuda", 0)


def T(a, view=None):
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(view) if view else a).to(dev)


def _check_surface(S, xy, off, W, H, nd, nf, alpha, tol=2e-6):
    S = S.cpu().numpy()
    for b in range(len(off) - 1):
        ref = oracle.build_window(xy[off[b]:off[b + 1]], W, H, nd, nf, alpha, want=("S",))["S"]
        err = np.abs(S[b].astype(np.float64) - ref).max()
        assert err <= tol, (b, err)


def case_window_f32():
    """frame_kernel + window_kernel<19, float> (unpacked 1280-wide and packed 346-wide CTAs)."""
    for cfg, nd, nf, n in ((GEN4, 2, 3, 2), (DAVIS, 1, 4, 5)):
        xy, off = batch_events(cfg, 3, 0, n)
        with ieds.Builder(cfg.width, cfg.height, nd, nf, d_sat=6.0, device=0) as b:
            S = b.build_batch(T(xy, np.int32), T(off))
            b.sync()
        _check_surface(S, xy, off, cfg.width, cfg.height, nd, nf, oracle.alpha_from_dsat(6.0))


def case_window_variants():
    """window_kernel<8, uint8>, <10, uint16 (fp16)>, and a wide window (<40, float>, d_sat 12)."""
    xy, off = batch_events(DAVIS, 4, 0, 3)
    for kw in (dict(out="u8"), dict(out="f16"), dict(d_sat=12.0)):
        with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, device=0, **kw) as b:
            b.build_batch(T(xy, np.int32), T(off))
            b.sync()


def case_exact_edt():
    """frame_kernel (transposed T + column bitmap) + edt_kernel with every debug output."""
    xy, off = batch_events(DAVIS, 5, 0, 2)
    W, H = DAVIS.width, DAVIS.height
    nw = (W + 31) // 32
    B = len(off) - 1
    E, Ed, Edf = (torch.empty((B, H, nw), dtype=torch.int32, device=dev) for _ in range(3))
    D2 = torch.empty((B, H, W), dtype=torch.int32, device=dev)
    with ieds.Builder(W, H, 1, 4, d_sat=6.0, device=0) as b:
        S = b.build_batch(T(xy, np.int32), T(off), edge_bits=E, denoised_bits=Ed, filtered_bits=Edf, sqdist=D2)
        b.sync()
    _check_surface(S, xy, off, W, H, 1, 4, oracle.alpha_from_dsat(6.0))


def case_norm_u8():
    """edt_kernel (D2 scratch) + d2max_kernel + norm_u8_kernel."""
    xy, off = batch_events(DAVIS, 6, 0, 2)
    with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, device=0, out="u8", transfer="log") as b:
        b.build_batch(T(xy, np.int32), T(off))
        b.sync()


def case_bands_and_latency():
    """Banded frame kernel (forced 64-row bands) and the single-window latency mode (row bands of
    both kernels), on one 1280x720 window."""
    xy, off = batch_events(GEN4, 7, 0, 1)
    for kw in (dict(_test_bands=True), dict(chunk_windows=1)):
        with ieds.Builder(1280, 720, 2, 3, d_sat=6.0, device=0, **kw) as b:
            S = b.build_batch(T(xy, np.int32), T(off))
            b.sync()
        _check_surface(S, xy, off, 1280, 720, 2, 3, oracle.alpha_from_dsat(6.0))


def case_windowing_and_stream():
    """window_offsets_kernel and the streaming ingest (ieds_stream_*)."""
    xs, ts = [], []
    for k in range(4):
        xy, t, _ = window_events(DAVIS, 8, k, with_tp=True)
        xs.append(xy)
        ts.append(t)
    xy, t = np.concatenate(xs), np.concatenate(ts)
    with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, d_sat=6.0, device=0) as b:
        off = b.window_offsets(T(t), DAVIS.dt_us)
        S = b.build_batch(T(xy, np.int32), off)
        b.sync()
        with b.stream(DAVIS.dt_us) as st:
            parts = [st.push(t[:len(t) // 3], xy[:len(t) // 3]), st.push(t[len(t) // 3:], xy[len(t) // 3:]),
                     st.flush()]
    got = np.concatenate([p for p in parts if len(p)])
    assert np.array_equal(got, S.cpu().numpy())


def case_host_entry():
    """ieds_build_batch_host (internal streams, pipelined copies)."""
    xy, off = batch_events(DAVIS, 9, 0, 3)
    with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, d_sat=6.0, device=0) as b:
        b.build_batch_host(xy, off)


def case_fwl():
    """fwl_splat_kernel + fwl_finalize_kernel (row f3)."""
    from synth.flowscene import flow_batch

    fx, ft, fp, foff, flows, _fl, tref = flow_batch(DAVIS, 1, 0, 2)
    with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, device=0) as b:
        r = b.fwl_batch(T(fx, np.int32), T(ft), T(fp), T(foff), T(flows), T(tref), DAVIS.dt_us)
        b.sync()
    for k in range(2):
        sl = slice(foff[k], foff[k + 1])
        ref = oracle.fwl(fx[sl], ft[sl], fp[sl], DAVIS.width, DAVIS.height, flows[k], tref[k], DAVIS.dt_us)["fwl"]
        assert abs(r["fwl"][k].item() - ref) <= 1e-9 * abs(ref)


def case_flow():
    """Row f4: pyramid, prep, gradient, temporal-blocked and cooperative Jacobi kernels, output pass."""
    xy, off = batch_events(DAVIS, 10, 0, 3)
    W, H = DAVIS.width, DAVIS.height
    nw = (W + 31) // 32
    Ed = torch.empty((3, H, nw), dtype=torch.int32, device=dev)
    with ieds.Builder(W, H, 1, 4, d_sat=6.0, device=0) as b:
        S = b.build_batch(T(xy, np.int32), T(off), denoised_bits=Ed)
        b.sync()
    with ieds.FlowEstimator(W, H, device=0) as fe:
        for k in range(3):
            fe.step(S[k], Ed[k])
    torch.cuda.synchronize()


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        torch.cuda.synchronize()
        print(f"case {n}: ok", flush=True)
