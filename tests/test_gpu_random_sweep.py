"""Randomised parity sweep of the hot path (rows a1-a5) against the oracle.

Seeded random configurations cover:
- frame sizes 1x1 .. 600x400 (ragged widths, tiny heights);
- every N_d / N_f;
- d_sat 1 .. 12: the saturation-aware window kernel (C up to 31), and the exact kernel beyond
  K_sat = 1024;
- event densities from near-empty to 40 %, empty and single-event windows;
- batches small enough to take the row-band (latency) launch shape and large enough for the
  bulk one;
- unaligned event pointers.

Bars as in test_gpu_parity: frames and D2 bit-exact, surface within 2e-6 of the fp64 oracle,
and the surface-only path bit-identical to the exact path.
"""
import numpy as np
import pytest

import oracle
from synth.events import random_frame_events

from tests.test_gpu_parity import check_window, csr, run_gpu

pytestmark = pytest.mark.gpu


def _config(rng):
    W = int(rng.choice([1, 2, 31, 32, 33, 63, 64, 65, 100, 257, 346, 600]) if rng.random() < 0.5
            else rng.integers(1, 601))
    H = int(rng.choice([1, 2, 3, 17, 64, 100, 260, 400]) if rng.random() < 0.5 else rng.integers(1, 401))
    n_d = int(rng.integers(0, 5))
    n_f = int(rng.integers(1, 6))
    d_sat = float(rng.choice([1.0, 2.5, 4.0, 6.0, 8.0, 9.5, 12.0]))
    return W, H, n_d, n_f, d_sat


@pytest.mark.parametrize("seed", range(40))
def test_random_configs(seed):
    rng = np.random.default_rng(1000 + seed)
    W, H, n_d, n_f, d_sat = _config(rng)
    a = oracle.alpha_from_dsat(d_sat)
    nwin = int(rng.choice([1, 3, 7]))
    wins = []
    for k in range(nwin):
        r = rng.random()
        if r < 0.1:
            wins.append(np.zeros(0, np.uint32))                                    # empty
        elif r < 0.2:
            wins.append(random_frame_events(W, H, 1.0 / max(1, W * H), seed=seed * 10 + k))
        else:
            dens = float(rng.choice([0.001, 0.01, 0.05, 0.2, 0.4]))
            wins.append(random_frame_events(W, H, dens, seed=seed * 10 + k))
    xy, off = csr(wins)
    shift = int(rng.integers(0, 4))                                                # unaligned loads
    gpu = run_gpu(xy, off, W, H, n_d, n_f, a, xy_shift=shift)
    for b in range(nwin):
        check_window(gpu, b, xy[off[b]:off[b + 1]], W, H, n_d, n_f, a)


@pytest.mark.parametrize("seed", range(16))
def test_random_epilogue_variants(seed):
    """Row f1 over random transfer x output format x geometry x d_sat, against the oracle:
    fp32 within 2e-6 + one rounding, 8-bit codes exact (plain Eq. (1) or normalised ablation),
    fp16 bit-exact from the table and within one fp16 ulp beyond it (Id / ln)."""
    import torch

    import paper_2112_10591_b200 as ieds

    rng = np.random.default_rng(5000 + seed)
    W, H, n_d, n_f, d_sat = _config(rng)
    transfer = str(rng.choice(["invexp", "linear", "bounded", "log"]))
    out = str(rng.choice(["f32", "u8", "f16"]))
    bound = float(rng.choice([2.0, 6.0, 9.5]))
    a = oracle.alpha_from_dsat(d_sat)
    if out == "u8" and transfer == "invexp" and d_sat > 9.0:
        d_sat, a = 6.0, oracle.alpha_from_dsat(6.0)   # the 8-bit Eq. (1) table must saturate by D2 = 1024
    wins = [random_frame_events(W, H, float(rng.choice([0.002, 0.02, 0.1])), seed=seed * 7 + k) for k in range(3)]
    wins.append(np.zeros(0, np.uint32))
    xy, off = csr(wins)
    dev = torch.device("cuda", 0)
    with ieds.Builder(W, H, n_d, n_f, alpha=a, device=0, transfer=transfer, bound=bound, out=out) as bld:
        S = bld.build_batch(torch.from_numpy(np.ascontiguousarray(xy).view(np.int32)).to(dev),
                            torch.from_numpy(off).to(dev))
        bld.sync()
    S = S.cpu().numpy()
    for b in range(len(wins)):
        ref = oracle.build_window(xy[off[b]:off[b + 1]], W, H, n_d, n_f, a)
        v = oracle.transfer(ref["D2"], transfer, alpha=a, bound=bound)
        if out == "u8":
            q = oracle.quantize_u8(v) if transfer == "invexp" else oracle.quantize_norm_u8(ref["D2"], transfer, bound=bound)
            assert np.array_equal(S[b], q), (transfer, b)
        elif out == "f32":
            fin = np.isfinite(v)
            assert np.array_equal(np.isinf(S[b]), ~fin)
            err = np.abs(S[b][fin].astype(np.float64) - v[fin])
            assert np.all(err <= 2e-6 + np.abs(v[fin]) * 2.0 ** -23), (transfer, b, float(err.max()))
        else:
            e16 = v.astype(np.float16)
            same = S[b].view(np.uint16) == e16.view(np.uint16)
            if transfer in ("invexp", "bounded"):
                assert same.all(), (transfer, b)
            else:
                tab = (ref["D2"] >= 0) & (ref["D2"] < 1024)
                assert same[tab].all(), (transfer, b)
                fin = np.isfinite(e16)
                ulp = np.spacing(np.abs(e16[fin])).astype(np.float64)
                assert np.all(np.abs(S[b][fin].astype(np.float64) - e16[fin].astype(np.float64)) <= ulp)


@pytest.mark.parametrize("seed", range(8))
def test_random_sensor_width_configs(seed):
    """The 1280-wide sensor instantiations (compile-time row stride, immediate-offset stores; the
    8-bit / fp16 saturated-rotation path) on random heights, thresholds, densities, batch sizes
    (row-band latency shape and bulk shape) and output formats: bit-identical to the exact-EDT
    kernel's surfaces, and the fp32 ones within 2e-6 of the oracle on sampled windows."""
    import torch

    import paper_2112_10591_b200 as ieds

    rng = np.random.default_rng(7000 + seed)
    W = 1280
    H = int(rng.choice([1, 2, 37, 38, 39, 76, 200, 720]) if rng.random() < 0.5 else rng.integers(1, 721))
    n_d, n_f = int(rng.integers(0, 5)), int(rng.integers(1, 6))
    out = str(rng.choice(["f32", "u8", "f16"]))
    nwin = int(rng.choice([1, 3, 160]))
    dens = [0.0, 0.0003, 0.002, 0.01, 0.05, 0.3]
    distinct = [random_frame_events(W, H, float(rng.choice(dens)), 31 * seed + i) for i in range(4)]
    wins = [distinct[i % 4] for i in range(nwin)]
    xy, off = csr(wins)
    dev = torch.device("cuda", 0)
    txy = torch.from_numpy(np.ascontiguousarray(xy).view(np.int32)).to(dev)
    toff = torch.from_numpy(off).to(dev)
    res = {}
    for exact in (False, True):
        with ieds.Builder(W, H, n_d, n_f, d_sat=6.0, device=0, out=out, exact_edt=exact) as bld:
            res[exact] = bld.build_batch(txy, toff).cpu().numpy()
            bld.sync()
    assert np.array_equal(res[False].view(np.uint8), res[True].view(np.uint8)), (H, n_d, n_f, out, nwin)
    if out == "f32":
        a = oracle.alpha_from_dsat(6.0)
        for b in sorted({0, nwin - 1}):
            ref = oracle.build_window(wins[b], W, H, n_d, n_f, a, want=("S",))["S"]
            assert np.abs(res[False][b].astype(np.float64) - ref).max() <= 2e-6
