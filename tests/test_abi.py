"""CPU-side checks of the C ABI: the in-tree library builds/loads and exports every symbol that
include/ieds.h declares; host-only entry points behave (no compute calls without a GPU)."""
import ctypes
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2112_10591_b200 import _lib

    return _lib.load()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ieds.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ieds_[a-z_]+)\s*\(", src)))


def test_header_declarations_match_binding():
    from paper_2112_10591_b200 import _lib

    assert declared_functions() == sorted(_lib.EXPORTS)


def test_every_declared_symbol_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_host_only_entry_points(lib):
    assert lib.ieds_version().decode().startswith("ieds-b200")
    assert lib.ieds_strerror(0) == b"ok"
    assert lib.ieds_strerror(-2) == b"event outside the frame"
    # Eq. (2)-(3): alpha = d_sat / ln 255 ~ d_sat / 5.541, 1.08 for 6 px
    a6 = lib.ieds_alpha_from_dsat(6.0)
    assert abs(a6 - 1.08) < 5e-3 and abs(6.0 / a6 - 5.541) < 5e-4
    assert abs(lib.ieds_alpha_from_dsat(math.log(255.0)) - 1.0) < 1e-15
    assert math.isnan(lib.ieds_alpha_from_dsat(0.0)) and math.isnan(lib.ieds_alpha_from_dsat(-3.0))


def test_create_rejects_bad_config_before_touching_cuda(lib):
    from paper_2112_10591_b200._lib import IEDS_EINVAL, IedsConfig

    h = ctypes.c_void_p()
    def cfg_(w=10, h_=10, nd=1, nf=4, a=1.0, flags=0, transfer=0, bound=6.0, fmt=0):
        return IedsConfig(w, h_, nd, nf, a, 0, 0, flags, transfer, bound, fmt)

    bad = [cfg_(w=0), cfg_(nd=5), cfg_(nf=0), cfg_(a=float("nan")), cfg_(a=-2.0), cfg_(h_=3000),
           cfg_(flags=8), cfg_(transfer=4), cfg_(transfer=2, bound=0.0), cfg_(fmt=3), cfg_(fmt=-1),
           cfg_(a=50.0, fmt=1)]              # 8-bit Eq. (1) saturation beyond the 1024-entry table
    for cfg in bad:
        assert lib.ieds_create(ctypes.byref(cfg), ctypes.byref(h)) == IEDS_EINVAL
        assert not h.value
    assert lib.ieds_create(None, ctypes.byref(h)) == IEDS_EINVAL
    lib.ieds_destroy(None)   # NULL-safe


def test_build_batch_argument_errors_without_handle(lib):
    from paper_2112_10591_b200._lib import IEDS_EINVAL

    assert lib.ieds_build_batch(None, None, None, 0, 1, None, None, None, None, None, None) == IEDS_EINVAL
    assert lib.ieds_sync(None, None) == IEDS_EINVAL
    assert lib.ieds_launches_per_batch(None, 10) == 0


def test_sass_is_sm100a(lib):
    """The library carries sm_100a SASS (cuobjdump), built with nvcc here."""
    import shutil
    import subprocess

    from paper_2112_10591_b200._lib import LIB_PATH

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_row_f_entry_points_reject_bad_arguments_without_cuda(lib):
    """Rows f2-f4: argument and configuration errors are returned synchronously, before any CUDA
    call (include/ieds.h), so they are checkable on a host without a GPU."""
    from paper_2112_10591_b200._lib import IEDS_EINVAL, IedsFlowConfig

    # f2 windowing and f3 FWL without a handle
    assert lib.ieds_window_offsets(None, None, 0, 0, 1000, 1, None, None) == IEDS_EINVAL
    assert lib.ieds_fwl_batch(None, None, None, None, None, 0, 1, None, None, 1000, None, None, None, None,
                              None) == IEDS_EINVAL
    # f4: every invalid flow configuration is rejected by ieds_flow_create
    def fcfg(**kw):
        c = IedsFlowConfig()
        c.width, c.height, c.levels = kw.get("w", 64), kw.get("h", 48), kw.get("levels", 3)
        for l in range(8):
            c.iterations[l] = kw.get("it", 20)
            c.lambda_[l] = kw.get("lam", 500.0)
        c.gamma, c.scale, c.device = kw.get("gamma", 0.5), kw.get("scale", 255.0), -1
        return c

    h = ctypes.c_void_p()
    bad = [dict(levels=0), dict(levels=9), dict(w=1), dict(h=1),
           dict(w=6, h=6, levels=3),   # level 2 would be 1 x 1
           dict(gamma=-0.1), dict(gamma=1.5), dict(scale=0.0), dict(scale=float("inf")), dict(it=-1),
           dict(lam=-1.0), dict(lam=float("nan"))]
    for kw in bad:
        c = fcfg(**kw)
        assert lib.ieds_flow_create(ctypes.byref(c), ctypes.byref(h)) == IEDS_EINVAL, kw
        assert not h.value
    assert lib.ieds_flow_create(None, ctypes.byref(h)) == IEDS_EINVAL
    assert lib.ieds_flow_step(None, None, None, None, None, None) == IEDS_EINVAL
    assert lib.ieds_flow_reset(None) == IEDS_EINVAL
    assert lib.ieds_flow_launches_per_step(None) == 0
    lib.ieds_flow_destroy(None)   # NULL-safe


def test_stream_entry_points_reject_bad_arguments_without_cuda(lib):
    """Row f2 (streaming ingest, window count): argument errors are returned before any CUDA call."""
    from paper_2112_10591_b200._lib import IEDS_EINVAL

    s = ctypes.c_void_p()
    assert lib.ieds_stream_create(None, 1000, ctypes.byref(s)) == IEDS_EINVAL and not s.value
    assert lib.ieds_stream_create(None, 1000, None) == IEDS_EINVAL
    n = ctypes.c_int32()
    assert lib.ieds_stream_push(None, None, None, 0, None, 0, ctypes.byref(n)) == IEDS_EINVAL
    assert lib.ieds_stream_flush(None, None, 0, ctypes.byref(n)) == IEDS_EINVAL
    assert lib.ieds_stream_closing(None, 0, 5) == 0
    lib.ieds_stream_destroy(None)   # NULL-safe
    t0, k = ctypes.c_int64(), ctypes.c_int32()
    assert lib.ieds_window_count(None, None, 0, 1000, ctypes.byref(t0), ctypes.byref(k), None) == IEDS_EINVAL


def test_pipeline_entry_points_reject_bad_arguments_without_cuda(lib):
    from paper_2112_10591_b200._lib import IEDS_EINVAL

    p = ctypes.c_void_p()
    n = ctypes.c_int32()
    assert lib.ieds_pipeline_create(None, None, 1000, ctypes.byref(p)) == IEDS_EINVAL and not p.value
    assert lib.ieds_pipeline_create(None, None, 1000, None) == IEDS_EINVAL
    assert lib.ieds_pipeline_push(None, None, None, 0, None, None, None, 0, ctypes.byref(n)) == IEDS_EINVAL
    assert lib.ieds_pipeline_flush(None, None, None, None, 0, ctypes.byref(n)) == IEDS_EINVAL
    assert lib.ieds_pipeline_closing(None, 0, 5) == 0
    lib.ieds_pipeline_destroy(None)   # NULL-safe
