"""Out-of-bounds write checks of our own (compute-sanitizer is closed on this GPU pool: see
profiles/r02_sanitizer.md).  Every output buffer the library writes is embedded in a larger
allocation filled with a canary byte pattern; after each call the bytes before and after the
buffer must be intact, and every byte of the buffer must have been written (no canary left
where the path must produce output).  Covers the frame / window / exact / normalised-8-bit /
windowing / FWL / flow / streaming kernels on bulk, banded, ragged and packed launch shapes."""
import numpy as np
import pytest

from synth.events import DAVIS, GEN4, batch_events, random_frame_events, window_events

pytestmark = pytest.mark.gpu
CANARY = 0xA5
PAD = 4096   # bytes of canary on each side


def _guarded(shape, dtype):
    import torch

    n = int(np.prod(shape)) * torch.empty(0, dtype=dtype).element_size()
    raw = torch.full((n + 2 * PAD,), CANARY, dtype=torch.uint8, device="cuda")
    return raw, raw[PAD:PAD + n].view(dtype).view(shape)


def _intact(raw, must_write=True):
    a = raw.cpu().numpy()
    assert np.all(a[:PAD] == CANARY), "write before the buffer"
    assert np.all(a[-PAD:] == CANARY), "write after the buffer"
    if must_write:
        body = a[PAD:-PAD]
        # a fully written fp32/fp16/u8/int buffer cannot be all-canary in any 4-byte-aligned run of 64 B
        runs = body[: len(body) // 64 * 64].reshape(-1, 64)
        assert not np.any(np.all(runs == CANARY, axis=1)), "part of the buffer left unwritten"


def _csr(ws):
    off = np.zeros(len(ws) + 1, np.int64)
    off[1:] = np.cumsum([len(w) for w in ws])
    return np.concatenate(ws).astype(np.uint32), off


@pytest.mark.parametrize("W,H,nwin,out,extra", [
    (1280, 720, 3, "f32", {}), (1280, 720, 150, "f32", {}), (346, 260, 40, "f32", {}), (1000, 333, 9, "u8", {}),
    (1288, 97, 200, "f16", {}), (33, 17, 5, "f32", {}), (1280, 720, 2, "f32", {"exact_edt": True}),
    (346, 260, 3, "u8", {"transfer": "log"}), (1920, 1080, 2, "f32", {}), (208, 1013, 4, "u8", {"d_sat": 12.0}),
    # several launch chunks: the next chunk's frame kernel on the side stream, two E_df sets
    (346, 260, 40, "f32", {"chunk_windows": 7}), (1280, 720, 9, "u8", {"chunk_windows": 4})])
def test_outputs_stay_in_bounds(W, H, nwin, out, extra):
    import torch

    import paper_2112_10591_b200 as ieds

    base = [random_frame_events(W, H, d, 70 + i) for i, d in enumerate((0.01, 0.0, 0.05, 0.3))]
    xy, off = _csr([base[i % 4] for i in range(nwin)])
    odt = {"u8": torch.uint8, "f16": torch.float16}.get(out, torch.float32)
    nw = (W + 31) // 32
    extra = dict(extra)
    kw = dict(d_sat=extra.pop("d_sat", 6.0))
    with ieds.Builder(W, H, 1, 3, device=0, out=out, **kw, **extra) as bld:
        rS, S = _guarded((nwin, H, W), odt)
        bld.build_batch(torch.from_numpy(xy.view(np.int32)).cuda(), torch.from_numpy(off).cuda(), S)
        bld.sync()
        _intact(rS)
        if out == "f32" and not extra:
            rb = [_guarded((nwin, H, nw), torch.int32) for _ in range(3)]
            rd, D2 = _guarded((nwin, H, W), torch.int32)
            rS2, S2 = _guarded((nwin, H, W), odt)
            bld.build_batch(torch.from_numpy(xy.view(np.int32)).cuda(), torch.from_numpy(off).cuda(), S2,
                            edge_bits=rb[0][1], denoised_bits=rb[1][1], filtered_bits=rb[2][1], sqdist=D2)
            bld.sync()
            for r, _ in rb:
                _intact(r, must_write=False)   # bit frames of sparse windows are mostly zero words
            _intact(rd)
            _intact(rS2)
            assert torch.equal(S, S2)


def test_row_f_outputs_stay_in_bounds():
    import torch

    import paper_2112_10591_b200 as ieds
    from synth.flowscene import flow_batch

    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    # f2 windowing
    xs, ts = zip(*[window_events(DAVIS, 4, k, with_tp=True)[:2] for k in range(5)])
    t = np.concatenate(ts)
    with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, device=0) as bld:
        t0, K = bld.window_count(T(t), DAVIS.dt_us)
        ro, offs = _guarded((K + 1,), torch.int64)
        from paper_2112_10591_b200._lib import load
        import ctypes
        rc = load().ieds_window_offsets(bld._h, ctypes.c_void_p(T(t).data_ptr()), len(t), t0, DAVIS.dt_us, K,
                                        ctypes.c_void_p(offs.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0
        bld.sync()
        _intact(ro)
        # f3 FWL with the compensated image
        fx, ft, fp, foff, flows, _fl, tref = flow_batch(DAVIS, 1, 0, 3)
        r = bld.fwl_batch(T(fx.view(np.int32)), T(ft), T(fp), T(foff), T(flows), T(tref), DAVIS.dt_us,
                          variances=True, comp_image=True)
        bld.sync()
        assert torch.isfinite(r["fwl"]).all()
    # f4 flow into guarded outputs
    xy, off = batch_events(DAVIS, 2, 0, 3)
    with ieds.Builder(DAVIS.width, DAVIS.height, 1, 4, device=0) as bld:
        S = bld.build_batch(T(xy.view(np.int32)), T(off))
        bld.sync()
    with ieds.FlowEstimator(DAVIS.width, DAVIS.height, device=0) as fe:
        rf, F = _guarded((DAVIS.height, DAVIS.width, 2), torch.float32)
        for k in range(3):
            fe.step(S[k], out=F)
        torch.cuda.synchronize()
        _intact(rf, must_write=False)
