"""CPU oracle of the IEDS surface build (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  It shares no code with the CUDA path and the CUDA path never
calls it.  The arithmetic lives in ieds_oracle.c (plain C, fp64 / int64), each function
citing the PAPER.md passage it follows; this module only marshals numpy arrays.

Outputs use the oracle's own representation: byte images [H][W] of 0/1 and int64
squared distances with NO_EDGE = -1 for "no edge pixel in the frame".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

NO_EDGE = -1
_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ieds_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            i64, i32, f64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double
            lib.oracle_accumulate.argtypes = [P, i64, i32, i32, P]
            lib.oracle_accumulate.restype = i32
            lib.oracle_denoise.argtypes = [P, i32, i32, i32, P]
            lib.oracle_fill.argtypes = [P, i32, i32, i32, P]
            lib.oracle_edt_separable.argtypes = [P, i32, i32, P]
            lib.oracle_edt_bruteforce.argtypes = [P, i32, i32, P]
            lib.oracle_surface.argtypes = [P, i64, f64, P]
            lib.oracle_transfer.argtypes = [P, i64, i32, f64, f64, P]
            lib.oracle_quantize_u8.argtypes = [P, i64, P]
            lib.oracle_quantize_norm_u8.argtypes = [P, i64, i32, f64, P]
            lib.oracle_quantize_norm_u8.restype = i32
            lib.oracle_window_offsets.argtypes = [P, i64, i64, P, i64]
            lib.oracle_window_offsets.restype = i64
            lib.oracle_fwl.argtypes = [P, P, P, i64, i32, i32, P, i64, i64, P, P, P]
            lib.oracle_fwl.restype = i32
            lib.oracle_downsample.argtypes = [P, i32, i32, P]
            lib.oracle_upsample_flow.argtypes = [P, i32, i32, i32, i32, P]
            lib.oracle_warp.argtypes = [P, i32, i32, P, P]
            lib.oracle_gradients.argtypes = [P, i32, i32, P, P]
            lib.oracle_hs_jacobi.argtypes = [P, P, P, P, i32, i32, f64, i32, P]
            lib.oracle_advect_flow.argtypes = [P, i32, i32, P]
            lib.oracle_flow_levels.argtypes = [i32, i32, i32, P, P]
            lib.oracle_flow_levels.restype = i64
            lib.oracle_flow_step.argtypes = [i32, i32, i32, P, P, f64, f64, i32, P, P, P, P]
            lib.oracle_flow_step.restype = i32
            lib.oracle_mask_flow.argtypes = [P, P, i64, P, P]
            lib.oracle_alpha_from_dsat.argtypes = [f64]
            lib.oracle_alpha_from_dsat.restype = f64
            lib.oracle_build_window.argtypes = [P, i64, i32, i32, i32, i32, f64, P, P, P, P, P]
            lib.oracle_build_window.restype = i32
            _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _img(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint8)


class OracleRangeError(ValueError):
    """An event lies outside the W x H frame."""


def accumulate(xy, width: int, height: int) -> np.ndarray:
    xy = np.ascontiguousarray(xy, dtype=np.uint32)
    E = np.zeros((height, width), np.uint8)
    st = _load().oracle_accumulate(_ptr(xy), len(xy), width, height, _ptr(E))
    if st != 0:
        raise OracleRangeError("event outside the frame")
    return E


def denoise(E, n_d: int) -> np.ndarray:
    E = _img(E)
    out = np.empty_like(E)
    _load().oracle_denoise(_ptr(E), E.shape[1], E.shape[0], n_d, _ptr(out))
    return out


def fill(E_d, n_f: int) -> np.ndarray:
    E_d = _img(E_d)
    out = np.empty_like(E_d)
    _load().oracle_fill(_ptr(E_d), E_d.shape[1], E_d.shape[0], n_f, _ptr(out))
    return out


def edt(E_df) -> np.ndarray:
    """Exact squared EDT (separable, FH lower envelope); NO_EDGE if the frame is empty."""
    E_df = _img(E_df)
    out = np.empty(E_df.shape, np.int64)
    _load().oracle_edt_separable(_ptr(E_df), E_df.shape[1], E_df.shape[0], _ptr(out))
    return out


def edt_bruteforce(E_df) -> np.ndarray:
    E_df = _img(E_df)
    out = np.empty(E_df.shape, np.int64)
    _load().oracle_edt_bruteforce(_ptr(E_df), E_df.shape[1], E_df.shape[0], _ptr(out))
    return out


def surface(D2, alpha: float) -> np.ndarray:
    D2 = np.ascontiguousarray(D2, dtype=np.int64)
    out = np.empty(D2.shape, np.float64)
    _load().oracle_surface(_ptr(D2), D2.size, float(alpha), _ptr(out))
    return out


def window_offsets(t_us, dt_us: int, max_windows: int = 1 << 24) -> np.ndarray:
    """CSR offsets of the Delta-T windows of a time-ordered stream (row f2, §III-A)."""
    t = np.ascontiguousarray(t_us, dtype=np.int64)
    n = len(t)
    est = 1 if n == 0 else min(max_windows, (int(t[-1]) - int(t[0])) // max(1, int(dt_us)) + 2) if n else 1
    out = np.zeros(max(est, 1) + 1, np.int64)
    k = _load().oracle_window_offsets(_ptr(t), n, int(dt_us), _ptr(out), len(out) - 1)
    if k == -1:
        raise ValueError("dt must be > 0")
    if k == -3:
        raise ValueError("timestamps not ordered")
    if k == -4:
        raise ValueError("too many windows")
    return out[:k + 1]


TRANSFERS = {"invexp": 0, "linear": 1, "bounded": 2, "log": 3}


def transfer(D2, kind: str, alpha: float = 1.0, bound: float = 6.0) -> np.ndarray:
    """Ablation transfers of §IV-D: invexp (Eq. (1)), linear, bounded, log."""
    D2 = np.ascontiguousarray(D2, dtype=np.int64)
    out = np.empty(D2.shape, np.float64)
    _load().oracle_transfer(_ptr(D2), D2.size, TRANSFERS[kind], float(alpha), float(bound), _ptr(out))
    return out


def quantize_u8(S) -> np.ndarray:
    """8-bit coding q = round(255 * d_exp), half away from zero."""
    S = np.ascontiguousarray(S, dtype=np.float64)
    q = np.empty(S.shape, np.uint8)
    _load().oracle_quantize_u8(_ptr(S), S.size, _ptr(q))
    return q


def quantize_norm_u8(D2, kind: str, bound: float = 6.0) -> np.ndarray:
    """8-bit view of Id / min(d, bound) / ln(d+1) normalised by the frame maximum:
    q = round(255 * v / max v); empty frame -> 255, max v = 0 -> 0 (reading R17)."""
    D2 = np.ascontiguousarray(D2, dtype=np.int64)
    q = np.empty(D2.shape, np.uint8)
    rc = _load().oracle_quantize_norm_u8(_ptr(D2), D2.size, TRANSFERS[kind], float(bound), _ptr(q))
    if rc == -1:
        raise ValueError("Eq. (1) is coded without normalisation (quantize_u8)")
    if rc != 0:
        raise MemoryError("oracle_quantize_norm_u8")
    return q


def fwl(xy, t_us, p, width: int, height: int, flow, t_ref_us: int, dt_us: int, images: bool = False) -> dict:
    """Row f3: flow-compensated event image and the Flow Warping
    Loss of one window.  flow is float32 [H][W][2] (dx, dy) in pixels per dt_us.  Returns
    {"var_comp", "var_uncomp", "fwl"} (+ "I_comp", "I_uncomp" fp64 [H][W] if images)."""
    xy = np.ascontiguousarray(xy, dtype=np.uint32)
    t = np.ascontiguousarray(t_us, dtype=np.int64)
    pp = np.ascontiguousarray(p, dtype=np.int8)
    F = np.ascontiguousarray(flow, dtype=np.float32)
    assert F.shape == (height, width, 2) and len(t) == len(xy) == len(pp)
    out3 = np.empty(3, np.float64)
    ic = np.empty((height, width), np.float64) if images else None
    iu = np.empty((height, width), np.float64) if images else None
    st = _load().oracle_fwl(_ptr(xy), _ptr(t), _ptr(pp), len(xy), width, height, _ptr(F), int(t_ref_us),
                            int(dt_us), _ptr(ic) if images else None, _ptr(iu) if images else None, _ptr(out3))
    if st == -1:
        raise ValueError("invalid parameters")
    if st == -2:
        raise OracleRangeError("event outside the frame")
    r = {"var_comp": float(out3[0]), "var_uncomp": float(out3[1]), "fwl": float(out3[2])}
    if images:
        r["I_comp"], r["I_uncomp"] = ic, iu
    return r


# ------------------------------------------------------------------ row f4: flow consumer

def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def downsample(I) -> np.ndarray:
    """2x2 mean pyramid step (reading R21): [H][W] -> [H//2][W//2]."""
    I = _f64(I)
    H, W = I.shape
    out = np.empty((H // 2, W // 2), np.float64)
    _load().oracle_downsample(_ptr(I), W, H, _ptr(out))
    return out


def upsample_flow(Fc, W: int, H: int) -> np.ndarray:
    """Half-pixel-centred bilinear upsampling of a [h][w][2] flow to [H][W][2], vectors x2."""
    Fc = _f64(Fc)
    h, w = Fc.shape[:2]
    out = np.empty((H, W, 2), np.float64)
    _load().oracle_upsample_flow(_ptr(Fc), w, h, W, H, _ptr(out))
    return out


def warp(I, F) -> np.ndarray:
    """out(p) = bilinear sample of I at p + F(p), coordinates clamped to the frame."""
    I, F = _f64(I), _f64(F)
    H, W = I.shape
    out = np.empty_like(I)
    _load().oracle_warp(_ptr(I), W, H, _ptr(F), _ptr(out))
    return out


def gradients(J):
    """Central differences, one-sided on the border: (Ix, Iy)."""
    J = _f64(J)
    H, W = J.shape
    Ix, Iy = np.empty_like(J), np.empty_like(J)
    _load().oracle_gradients(_ptr(J), W, H, _ptr(Ix), _ptr(Iy))
    return Ix, Iy


def hs_jacobi(Ix, Iy, It, lam: float, K: int, init=None) -> np.ndarray:
    """K Jacobi sweeps of Horn-Schunck on the total flow from w^0 = init (default 0): [H][W][2]."""
    Ix, Iy, It = _f64(Ix), _f64(Iy), _f64(It)
    H, W = Ix.shape
    ini = _f64(init) if init is not None else None
    w = np.empty((H, W, 2), np.float64)
    _load().oracle_hs_jacobi(_ptr(Ix), _ptr(Iy), _ptr(It), _ptr(ini) if ini is not None else None, W, H,
                             float(lam), int(K), _ptr(w))
    return w


def advect_flow(P) -> np.ndarray:
    """Pt(p) = P(p - P(p)): a [H][W][2] flow transported by itself (bilinear, border-clamped)."""
    P = _f64(P)
    H, W = P.shape[:2]
    out = np.empty_like(P)
    _load().oracle_advect_flow(_ptr(P), W, H, _ptr(out))
    return out


def mask_flow(F, E_d):
    """keep the flow on denoised edge pixels; (masked flow, valid bytes)."""
    F = _f64(F)
    E = np.ascontiguousarray(E_d, dtype=np.uint8)
    out = np.empty_like(F)
    valid = np.empty(E.shape, np.uint8)
    _load().oracle_mask_flow(_ptr(F), _ptr(E), E.size, _ptr(out), _ptr(valid))
    return out, valid


class FlowOracle:
    """Stateful row-f4 estimator (reading R21): feed surfaces window by window with step()."""

    def __init__(self, width: int, height: int, levels=3, lambdas=(500.0, 500.0, 500.0), iters=(20, 20, 20),
                 gamma: float = 0.5, scale: float = 255.0):
        self.W, self.H, self.L = width, height, int(levels)
        self.lam = np.ascontiguousarray(lambdas[:self.L], dtype=np.float64)
        self.it = np.ascontiguousarray(iters[:self.L], dtype=np.int32)
        self.gamma, self.scale = float(gamma), float(scale)
        Ws = np.zeros(16, np.int32)
        Hs = np.zeros(16, np.int32)
        tot = _load().oracle_flow_levels(width, height, self.L, _ptr(Ws), _ptr(Hs))
        if tot < 0:
            raise ValueError("pyramid level smaller than 2x2")
        self.sizes = [(int(Ws[l]), int(Hs[l])) for l in range(self.L)]
        self.prev = np.zeros(tot, np.float64)
        self.P = np.zeros(2 * tot, np.float64)
        self.fresh = True

    def reset(self):
        self.fresh = True

    def step(self, S) -> np.ndarray:
        S = _f64(S)
        assert S.shape == (self.H, self.W)
        F0 = np.empty((self.H, self.W, 2), np.float64)
        rc = _load().oracle_flow_step(self.W, self.H, self.L, _ptr(self.lam), _ptr(self.it), self.gamma, self.scale,
                                      1 if self.fresh else 0, _ptr(S), _ptr(self.prev), _ptr(self.P), _ptr(F0))
        if rc != 0:
            raise ValueError("oracle_flow_step")
        self.fresh = False
        return F0


def alpha_from_dsat(d_sat: float) -> float:
    return _load().oracle_alpha_from_dsat(float(d_sat))


def build_window(xy, width: int, height: int, n_d: int, n_f: int, alpha: float,
                 want=("E", "E_d", "E_df", "D2", "S")) -> dict:
    """accumulate -> Alg. 1 -> Alg. 2 -> EDT -> Eq. (1) for one window."""
    xy = np.ascontiguousarray(xy, dtype=np.uint32)
    shp = (height, width)
    out = {}
    bufs = {}
    for k, dt in (("E", np.uint8), ("E_d", np.uint8), ("E_df", np.uint8), ("D2", np.int64), ("S", np.float64)):
        bufs[k] = np.empty(shp, dt) if k in want else None
    st = _load().oracle_build_window(
        _ptr(xy), len(xy), width, height, n_d, n_f, float(alpha),
        *[(_ptr(bufs[k]) if bufs[k] is not None else None) for k in ("E", "E_d", "E_df", "D2", "S")])
    if st == -1:
        raise ValueError("invalid parameters")
    if st == -2:
        raise OracleRangeError("event outside the frame")
    for k in want:
        out[k] = bufs[k]
    return out


def build_batch(xy, offsets, width: int, height: int, n_d: int, n_f: int, alpha: float,
                windows=None, threads: int | None = None, want=("S",)) -> list:
    """Run build_window over windows (list of indices) of a CSR batch on a thread pool.

    ctypes releases the GIL during the C call, so `threads` host cores run concurrently.
    """
    xy = np.ascontiguousarray(xy, dtype=np.uint32)
    offsets = np.asarray(offsets, dtype=np.int64)
    idx = range(len(offsets) - 1) if windows is None else windows
    threads = threads or len(os.sched_getaffinity(0))

    def one(i):
        return build_window(xy[offsets[i]:offsets[i + 1]], width, height, n_d, n_f, alpha, want=want)

    if threads <= 1:
        return [one(i) for i in idx]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(one, idx))
