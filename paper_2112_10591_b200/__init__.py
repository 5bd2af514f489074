"""B200-native batched IEDS build (Brebion et al., arXiv 2112.10591).

Thin binding over the C ABI of include/ieds.h: it only marshals torch tensors (device
memory, streams) into the library's calls.  Every step of the path -- scatter, denoise
(Alg. 1), fill (Alg. 2), exact EDT and the Eq. (1) surface -- runs in the CUDA kernels of
libieds.so.  There is no CPU fallback: without the library or a CUDA device, calls raise.
"""
from __future__ import annotations

import ctypes
import dataclasses

from ._lib import (IedsFlowConfig, IEDS_FLAG_EXACT_EDT, IEDS_NO_EDGE, OUT_FORMATS, TRANSFERS, IedsConfig, IedsError, IedsOrderError, IedsRangeError, LIB_PATH,
                   check, load)

__all__ = ["Builder", "EventStream", "Pipeline", "alpha_from_dsat", "version", "IedsError", "IedsRangeError", "IedsOrderError",
           "IEDS_NO_EDGE", "LIB_PATH"]

load()   # fail loudly at import if libieds.so is missing


def _host_empty(shape, dtype):
    """Page-locked host array for the library's device-to-host copies (torch's caching pinned
    allocator, so repeated calls reuse blocks): copies into pageable memory go through the
    driver's staging buffers at a fraction of the PCIe rate."""
    import numpy as np
    import torch

    tdt = {np.dtype(np.float32): torch.float32, np.dtype(np.float16): torch.float16,
           np.dtype(np.uint8): torch.uint8}[np.dtype(dtype)]
    return torch.empty(tuple(shape), dtype=tdt, pin_memory=True).numpy()


def alpha_from_dsat(d_sat: float) -> float:
    """Eq. (2)-(3): alpha = d_sat / ln 255."""
    return load().ieds_alpha_from_dsat(float(d_sat))


def version() -> str:
    return load().ieds_version().decode()


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


@dataclasses.dataclass
class Params:
    width: int
    height: int
    n_d: int
    n_f: int
    alpha: float


class Builder:
    """One ieds_handle on one CUDA device.

    Builder(width, height, n_d, n_f, alpha=None, d_sat=6.0) -- alpha defaults to
    alpha_from_dsat(d_sat).  transfer selects Eq. (1) ("invexp") or a §IV-D ablation ("linear",
    "bounded" with `bound`, "log"); out="u8" gives the 8-bit coded surface (for the
    ablations, normalised by the frame maximum), out="f16" float16 surfaces.
    exact_edt=True forces the uncapped exact-EDT kernel even when only surfaces are requested
    (the default streaming kernel gives bit-identical surfaces).  chunk_windows = windows per
    launch pair, which sizes the handle's scratch; 0 = what a ~4 GB budget holds.  build_batch()
    enqueues on the current torch stream (or the given one) and does not synchronise; sync()
    reports latched device errors.
    """

    def __init__(self, width: int, height: int, n_d: int, n_f: int, alpha: float | None = None,
                 d_sat: float = 6.0, chunk_windows: int = 0, device=None, exact_edt: bool = False,
                 transfer: str = "invexp", bound: float = 6.0, out: str = "f32", _test_bands: bool = False):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_2112_10591_b200 needs a CUDA device (no CPU fallback)")
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", torch.device(device).index if not isinstance(device, int) else device)
        if alpha is None:
            alpha = alpha_from_dsat(d_sat)
        self.params = Params(width, height, n_d, n_f, float(alpha))
        if transfer not in TRANSFERS or out not in OUT_FORMATS:
            raise ValueError(f"transfer must be one of {list(TRANSFERS)}, out one of {list(OUT_FORMATS)}")
        cfg = IedsConfig(width, height, n_d, n_f, float(alpha), chunk_windows, self.device.index,
                         (IEDS_FLAG_EXACT_EDT if exact_edt else 0) | (2 if _test_bands else 0),
                         TRANSFERS[transfer], float(bound),
                         OUT_FORMATS[out])
        self.out = out
        self.transfer = transfer
        self.exact_edt = exact_edt
        h = ctypes.c_void_p()
        check(load().ieds_create(ctypes.byref(cfg), ctypes.byref(h)), "ieds_create")
        self._h = h
        self.width, self.height = width, height
        self.words = (width + 31) // 32

    # -- lifecycle -------------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            load().ieds_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- helpers ---------------------------------------------------------------------------
    def _stream(self, stream):
        import torch

        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(stream.cuda_stream)

    def _check_dev(self, t, name, dtypes):
        if t is None:
            return
        if not t.is_cuda or t.device != self.device:
            raise ValueError(f"{name} must be a tensor on {self.device}")
        if t.dtype not in dtypes:
            raise TypeError(f"{name} must have dtype in {dtypes}, got {t.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")

    def profile(self, on: bool = True):
        """Enable/disable per-kernel CUDA-event timing inside the library."""
        check(load().ieds_profile_enable(self._h, 1 if on else 0), "ieds_profile_enable")

    def profile_read(self) -> dict:
        """{'frame': (ms, launches), 'edt': (ms, launches)} since the last read."""
        fm, em = ctypes.c_double(), ctypes.c_double()
        fn, en = ctypes.c_int64(), ctypes.c_int64()
        check(load().ieds_profile_read(self._h, ctypes.byref(fm), ctypes.byref(fn), ctypes.byref(em),
                                       ctypes.byref(en)), "ieds_profile_read")
        return {"frame": (fm.value, fn.value), "edt": (em.value, en.value)}

    def launches_per_batch(self, num_windows: int) -> int:
        return int(load().ieds_launches_per_batch(self._h, int(num_windows)))

    # -- the path --------------------------------------------------------------------------
    def build_batch(self, events_xy, offsets, out=None, *, edge_bits=None, denoised_bits=None,
                    filtered_bits=None, sqdist=None, stream=None):
        """Surfaces [B, H, W] fp32 for the CSR batch (events_xy uint32/int32 [n], offsets int64 [B+1]).

        Optional outputs (pre-allocated, uint32/int32): edge_bits / denoised_bits /
        filtered_bits [B, H, ceil(W/32)] (E, E_d, E_df) and sqdist [B, H, W] (exact D2,
        0xFFFFFFFF when the window's E_df is empty).
        """
        import torch

        u32 = (torch.int32, getattr(torch, "uint32", torch.int32))
        self._check_dev(events_xy, "events_xy", u32)
        self._check_dev(offsets, "offsets", (torch.int64,))
        B = offsets.numel() - 1
        odt = {"u8": torch.uint8, "f16": torch.float16}.get(self.out, torch.float32)
        if out is None:
            out = torch.empty((B, self.height, self.width), dtype=odt, device=self.device)
        self._check_dev(out, "out", (odt,))
        if out.numel() < B * self.height * self.width:
            raise ValueError("out too small")
        for name, t, n in (("edge_bits", edge_bits, self.words), ("denoised_bits", denoised_bits, self.words),
                           ("filtered_bits", filtered_bits, self.words), ("sqdist", sqdist, self.width)):
            self._check_dev(t, name, u32)
            if t is not None and t.numel() < B * self.height * n:
                raise ValueError(f"{name} too small")
        check(load().ieds_build_batch(self._h, _ptr(events_xy), _ptr(offsets), events_xy.numel(), B,
                                      _ptr(out), _ptr(edge_bits), _ptr(denoised_bits), _ptr(filtered_bits),
                                      _ptr(sqdist), self._stream(stream)), "ieds_build_batch")
        return out

    def window_count(self, t_us, dt_us: int, stream=None):
        """Row f2 (ieds_window_count): (t0, K) of a time-ordered int64 timestamp tensor on this
        device -- t0 = t[0], K = floor((t[-1] - t0)/dt) + 1 windows (reading R16).  Synchronous."""
        import torch

        self._check_dev(t_us, "t_us", (torch.int64,))
        t0, K = ctypes.c_int64(), ctypes.c_int32()
        check(load().ieds_window_count(self._h, _ptr(t_us), t_us.numel(), int(dt_us), ctypes.byref(t0),
                                       ctypes.byref(K), self._stream(stream)), "ieds_window_count")
        return t0.value, K.value

    def stream(self, dt_us: int) -> "EventStream":
        """Row f2 streaming ingest (ieds_stream_*): an EventStream that takes host chunks of a
        time-ordered (t, xy) stream and returns each window's surface once it has closed."""
        return EventStream(self, dt_us)

    def window_offsets(self, t_us, dt_us: int, stream=None):
        """Row f2: CSR offsets [K+1] (int64, on the device) of the Delta-T windows of a
        time-ordered int64 timestamp tensor t_us (window k = floor((t - t0)/dt) == k, t0 = t[0]).
        Reads the first and last timestamps to size the output; ordering errors are latched
        and raised by sync()."""
        import torch

        self._check_dev(t_us, "t_us", (torch.int64,))
        n = t_us.numel()
        if dt_us <= 0:
            raise ValueError("dt_us must be > 0")
        if n == 0:
            return torch.zeros(1, dtype=torch.int64, device=self.device)
        try:
            t0, K = self.window_count(t_us, dt_us, stream)
        except IedsOrderError:
            # last timestamp before the first: one window; the kernel's order check latches
            # IEDS_EORDER for sync(), as for any other inversion
            t0, K = int(t_us[0].item()), 1
        off = torch.empty(K + 1, dtype=torch.int64, device=self.device)
        check(load().ieds_window_offsets(self._h, _ptr(t_us), n, t0, int(dt_us), K, _ptr(off),
                                         self._stream(stream)), "ieds_window_offsets")
        return off

    def fwl_batch(self, events_xy, events_t_us, events_p, offsets, flow, t_ref_us, dt_us: int, *,
                  variances: bool = False, comp_image: bool = False, stream=None) -> dict:
        """Row f3 (ieds_fwl_batch): Flow Warping Loss of each window.
        events_xy int32/uint32 [n], events_t_us int64 [n], events_p int8 [n], offsets int64
        [B+1], flow float32 [B, H, W, 2] (pixels per dt_us), t_ref_us int64 [B] -- all on this
        device.  Returns {"fwl": float64 [B]} plus "var_comp"/"var_uncomp" [B] and "comp_image"
        float64 [B, H, W] when asked.  Enqueued; call sync() to surface latched errors."""
        import torch

        self._check_dev(events_xy, "events_xy", (torch.int32, torch.uint32))
        self._check_dev(events_t_us, "events_t_us", (torch.int64,))
        self._check_dev(events_p, "events_p", (torch.int8,))
        self._check_dev(offsets, "offsets", (torch.int64,))
        self._check_dev(flow, "flow", (torch.float32,))
        self._check_dev(t_ref_us, "t_ref_us", (torch.int64,))
        B = offsets.numel() - 1
        n = events_xy.numel()
        if events_t_us.numel() != n or events_p.numel() != n:
            raise ValueError("events_xy, events_t_us and events_p must have the same length")
        if tuple(flow.shape) != (B, self.height, self.width, 2) or t_ref_us.numel() != B:
            raise ValueError("flow must be [B, H, W, 2] and t_ref_us [B]")
        dev = self.device
        out = {"fwl": torch.empty(B, dtype=torch.float64, device=dev)}
        if variances:
            out["var_comp"] = torch.empty(B, dtype=torch.float64, device=dev)
            out["var_uncomp"] = torch.empty(B, dtype=torch.float64, device=dev)
        if comp_image:
            out["comp_image"] = torch.empty((B, self.height, self.width), dtype=torch.float64, device=dev)
        check(load().ieds_fwl_batch(self._h, _ptr(events_xy), _ptr(events_t_us), _ptr(events_p), _ptr(offsets), n, B,
                                    _ptr(flow), _ptr(t_ref_us), int(dt_us), _ptr(out["fwl"]),
                                    _ptr(out.get("var_comp")), _ptr(out.get("var_uncomp")),
                                    _ptr(out.get("comp_image")), self._stream(stream)), "ieds_fwl_batch")
        return out

    def sync(self, stream=None):
        """Wait for the stream; raise IedsRangeError / IedsOrderError on latched data errors."""
        check(load().ieds_sync(self._h, self._stream(stream)), "ieds_sync")

    def build_batch_host(self, events_xy, offsets, out=None):
        """Host-buffer entry point (ieds_build_batch_host): numpy uint32 [n], int64 [B+1] ->
        float32 [B, H, W] host array; copies overlap the kernels inside the library."""
        import numpy as np

        xy = np.ascontiguousarray(events_xy).view(np.uint32)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        B = len(off) - 1
        odt = {"u8": np.uint8, "f16": np.float16}.get(self.out, np.float32)
        if out is None:
            out = _host_empty((B, self.height, self.width), odt)
        if out.dtype != odt or not out.flags.c_contiguous or out.size < B * self.height * self.width:
            raise ValueError(f"out must be a C-contiguous {np.dtype(odt).name} array of B*H*W")
        check(load().ieds_build_batch_host(self._h, xy.ctypes.data_as(ctypes.c_void_p),
                                           off.ctypes.data_as(ctypes.c_void_p), B,
                                           out.ctypes.data_as(ctypes.c_void_p)), "ieds_build_batch_host")
        return out


class EventStream:
    """Row f2: a live event stream, host chunks in, surfaces out as windows close (Fig. 1).

    push(t_us, xy) takes numpy int64 [n] timestamps (non-decreasing over the whole stream) and
    uint32 [n] packed x | y << 16; it returns the surfaces [k, H, W] (host numpy, the builder's
    output type) of the k windows that the chunk closed.  The open window's events stay on the
    device until a later event (or flush()) closes it.  Windows follow reading R16 (t0 = the first
    event; empty interior windows are emitted) and are bit-identical to the batched path."""

    def __init__(self, builder: Builder, dt_us: int):
        import numpy as np

        self.builder = builder
        self.dt_us = int(dt_us)
        self._odt = {"u8": np.uint8, "f16": np.float16}.get(builder.out, np.float32)
        self._s = ctypes.c_void_p()
        check(load().ieds_stream_create(builder._h, self.dt_us, ctypes.byref(self._s)), "ieds_stream_create")

    def closing(self, t_first_us: int, t_last_us: int) -> int:
        """Windows a push of a chunk spanning [t_first_us, t_last_us] would close."""
        return int(load().ieds_stream_closing(self._s, int(t_first_us), int(t_last_us)))

    def _out(self, k):
        import numpy as np

        return _host_empty((max(k, 0), self.builder.height, self.builder.width), self._odt)

    def push(self, t_us, events_xy):
        """t_us / events_xy: numpy arrays, or CPU torch tensors (pinned ones skip the library's
        host staging copy)."""
        import numpy as np

        if hasattr(t_us, "numpy"):      # CPU torch tensors: same memory, no copy
            t_us = t_us.numpy()
        if hasattr(events_xy, "numpy"):
            events_xy = events_xy.numpy()
        t = np.ascontiguousarray(t_us, dtype=np.int64)
        xy = np.ascontiguousarray(events_xy).view(np.uint32)
        if t.shape != xy.shape or t.ndim != 1:
            raise ValueError("t_us and events_xy must be 1-D arrays of the same length")
        n = len(t)
        out = self._out(self.closing(int(t[0]), int(t[-1])) if n else 0)
        got = ctypes.c_int32()
        check(load().ieds_stream_push(self._s, t.ctypes.data_as(ctypes.c_void_p), xy.ctypes.data_as(ctypes.c_void_p),
                                      n, out.ctypes.data_as(ctypes.c_void_p), len(out), ctypes.byref(got)),
              "ieds_stream_push")
        return out[:got.value]

    def flush(self):
        out = self._out(1)
        got = ctypes.c_int32()
        check(load().ieds_stream_flush(self._s, out.ctypes.data_as(ctypes.c_void_p), 1, ctypes.byref(got)),
              "ieds_stream_flush")
        return out[:got.value]

    def close(self):
        if getattr(self, "_s", None) is not None and self._s.value:
            load().ieds_stream_destroy(self._s)
            self._s = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class Pipeline:
    """The Fig. 1 pipeline (ieds_pipeline_*): host chunks of a live event stream in,
    per closed window its flow (and valid mask, optionally its surface) out, the surfaces of later
    windows built while earlier windows' flow runs.  push(t_us, xy) -> dict of host arrays
    {"flow": float32 [k, H, W, 2], "valid": uint8 [k, H, W], "surfaces": float32 [k, H, W] if
    asked}; flush() closes the last window and starts a new sequence (stream and estimator)."""

    def __init__(self, builder: "Builder", estimator: "FlowEstimator", dt_us: int, surfaces: bool = False):
        self.builder, self.estimator = builder, estimator
        self.want_surfaces = surfaces
        self._p = ctypes.c_void_p()
        check(load().ieds_pipeline_create(builder._h, estimator._h, int(dt_us), ctypes.byref(self._p)),
              "ieds_pipeline_create")

    def closing(self, t_first_us: int, t_last_us: int) -> int:
        return int(load().ieds_pipeline_closing(self._p, int(t_first_us), int(t_last_us)))

    def _outs(self, k):
        import numpy as np

        H, W = self.builder.height, self.builder.width
        o = {"flow": _host_empty((k, H, W, 2), np.float32), "valid": _host_empty((k, H, W), np.uint8)}
        if self.want_surfaces:
            o["surfaces"] = _host_empty((k, H, W), np.float32)
        return o

    @staticmethod
    def _ptrs(o):
        return [o[k].ctypes.data_as(ctypes.c_void_p) if k in o else None for k in ("flow", "valid", "surfaces")]

    def push(self, t_us, events_xy) -> dict:
        import numpy as np

        if hasattr(t_us, "numpy"):
            t_us = t_us.numpy()
        if hasattr(events_xy, "numpy"):
            events_xy = events_xy.numpy()
        t = np.ascontiguousarray(t_us, dtype=np.int64)
        xy = np.ascontiguousarray(events_xy).view(np.uint32)
        if t.shape != xy.shape or t.ndim != 1:
            raise ValueError("t_us and events_xy must be 1-D arrays of the same length")
        n = len(t)
        o = self._outs(self.closing(int(t[0]), int(t[-1])) if n else 0)
        got = ctypes.c_int32()
        check(load().ieds_pipeline_push(self._p, t.ctypes.data_as(ctypes.c_void_p), xy.ctypes.data_as(ctypes.c_void_p),
                                        n, *self._ptrs(o), len(o["flow"]), ctypes.byref(got)), "ieds_pipeline_push")
        return {k: v[:got.value] for k, v in o.items()}

    def flush(self) -> dict:
        o = self._outs(1)
        got = ctypes.c_int32()
        check(load().ieds_pipeline_flush(self._p, *self._ptrs(o), 1, ctypes.byref(got)), "ieds_pipeline_flush")
        return {k: v[:got.value] for k, v in o.items()}

    def close(self):
        if getattr(self, "_p", None) is not None and self._p.value:
            load().ieds_pipeline_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class FlowEstimator:
    """Row f4 (ieds_flow_*): the stateful flow consumer of the surfaces, DESIGN
    reading R21.  Defaults are the paper's HD settings (3 levels, weight 500, 20 sweeps
    each) with gamma = 0.5 and surfaces scaled by 255.  step(surface, edge_bits=None) takes a
    float32 [H, W] surface (and the uint32 [H, ceil(W/32)] denoised edge bits to restrict the
    output to) on this device and returns (flow float32 [H, W, 2], valid uint8 [H, W]),
    enqueued on the current stream; the first window of a sequence gives zero flow."""

    def __init__(self, width: int, height: int, levels: int = 3, lambdas=(500.0, 500.0, 500.0), iterations=(20, 20, 20),
                 gamma: float = 0.5, scale: float = 255.0, device=None):
        import torch

        self.width, self.height = int(width), int(height)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        cfg = IedsFlowConfig()
        cfg.width, cfg.height, cfg.levels = self.width, self.height, int(levels)
        for l in range(min(int(levels), 8)):
            cfg.iterations[l] = int(iterations[l])
            cfg.lambda_[l] = float(lambdas[l])
        cfg.gamma, cfg.scale, cfg.device = float(gamma), float(scale), self.device.index
        self._h = ctypes.c_void_p()
        check(load().ieds_flow_create(ctypes.byref(cfg), ctypes.byref(self._h)), "ieds_flow_create")

    def step(self, surface, edge_bits=None, out=None, stream=None):
        import torch

        H, W = self.height, self.width
        if surface.dtype != torch.float32 or surface.device != self.device or not surface.is_contiguous():
            raise TypeError("surface must be a contiguous float32 tensor on the estimator's device")
        if tuple(surface.shape[-2:]) != (H, W) or surface.numel() != H * W:
            raise ValueError(f"surface must hold one {H}x{W} frame, got shape {tuple(surface.shape)}")
        if edge_bits is not None:
            if edge_bits.device != self.device or not edge_bits.is_contiguous():
                raise TypeError("edge_bits must be a contiguous tensor on the estimator's device")
            if edge_bits.dtype not in (torch.int32, torch.uint32) or edge_bits.numel() < H * ((W + 31) // 32):
                raise ValueError(f"edge_bits must be int32/uint32 with >= {H}*ceil({W}/32) words")
        if out is not None:
            if (out.dtype != torch.float32 or out.device != self.device or not out.is_contiguous()
                    or tuple(out.shape) != (H, W, 2)):
                raise ValueError(f"out must be a contiguous float32 [{H}, {W}, 2] tensor on {self.device}")
            flow = out
        else:
            flow = torch.empty((H, W, 2), dtype=torch.float32, device=self.device)
        valid = torch.empty((H, W), dtype=torch.uint8, device=self.device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        st = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        check(load().ieds_flow_step(self._h, _ptr(surface), _ptr(edge_bits), _ptr(flow), _ptr(valid),
                                    ctypes.c_void_p(st)), "ieds_flow_step")
        return flow, valid

    def reset(self):
        check(load().ieds_flow_reset(self._h), "ieds_flow_reset")

    def launches_per_step(self) -> int:
        return int(load().ieds_flow_launches_per_step(self._h))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load().ieds_flow_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
