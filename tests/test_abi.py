"""The C-ABI library: loads without a GPU, exports every symbol that
include/rangefit_b200.h declares, and validates arguments (reference
ValueError conventions) before touching the device.  No compute calls."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2103_06644_b200 import _native as N

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "rangefit_b200.h"


def header_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:rf_status|int32_t|int64_t|const char\*)\s+(rf_\w+)\(", text, re.M)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(N.EXPORTED_SYMBOLS)


def test_library_exports_every_symbol():
    lib = N.load()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.rf_abi_version() == N.RF_ABI_VERSION


def test_launch_count():
    # one tile kernel per call for one space (implicit and explicit fits share it)
    lib = N.load()
    f32 = N.RF_DEPTH_F32_M
    assert lib.rf_launches_per_call(N.RF_IMPLICIT_STANDARD, 5, f32, 64, 480, 640) == 1
    assert lib.rf_launches_per_call(N.RF_IMPLICIT_RGBD, 5, f32, 1, 480, 640) == 1
    assert lib.rf_launches_per_call(N.RF_IMPLICIT_STANDARD | N.RF_EXPLICIT_STANDARD, 31, f32, 1, 480, 640) == 1


@pytest.mark.gpu
def test_launch_count_fused():
    # small batches: both spaces in one launch wherever two CTAs fit per SM; large: one per space
    lib = N.load()
    f32, u16 = N.RF_DEPTH_F32_M, N.RF_DEPTH_U16_MM
    both = N.RF_IMPLICIT_STANDARD | N.RF_IMPLICIT_RGBD
    for window in (9, 11):  # fused at one frame
        assert lib.rf_launches_per_call(both, window, f32, 1, 480, 640) == 1, window
    for window in (3, 5, 7):  # one wave of tiles at small radii: a launch per space at three CTAs per SM
        assert lib.rf_launches_per_call(both, window, f32, 1, 480, 640) == 2, window
    for window in (3, 5, 7, 9, 11, 15, 31):
        assert lib.rf_launches_per_call(both, window, f32, 64, 480, 640) == 2, window
    assert lib.rf_launches_per_call(both, 15, u16, 1, 480, 640) == 1  # fused


@pytest.mark.parametrize("fx,fy,cx,cy,w,h,msg", [
    (0.0, 1.0, 0.5, 0.5, 4, 4, "focal"),           # camera.py:55-56
    (1.0, -1.0, 0.5, 0.5, 4, 4, "focal"),
    (1.0, 1.0, 0.5, 0.5, 0, 4, "size"),            # camera.py:57-58
    (1.0, 1.0, 4.0, 0.5, 4, 4, "principal"),       # camera.py:59-63
    (1.0, 1.0, 0.5, -0.1, 4, 4, "principal"),
])
def test_tables_create_validation(fx, fy, cx, cy, w, h, msg):
    lib = N.load()
    intr = N.RfIntrinsics(fx, fy, cx, cy, w, h)
    out = ctypes.c_void_p()
    st = lib.rf_tables_create(ctypes.byref(intr), None, None, 0, ctypes.byref(out))
    assert st == N.RF_ERR_ARGUMENT
    assert msg in N.last_error()
    assert not out


def test_fit_pixels_null_arguments():
    lib = N.load()
    st = lib.rf_fit_pixels(None, None, 0, 1, 4, 4, 4, None, 5, 3, None, None)
    assert st == N.RF_ERR_ARGUMENT
    with pytest.raises(ValueError):
        N.check(st, "fit_pixels")


def test_check_maps_status_to_exceptions():
    N.check(N.RF_OK, "x")
    with pytest.raises(ValueError):
        N.check(N.RF_ERR_SHAPE, "x")
    with pytest.raises(RuntimeError):
        N.check(N.RF_ERR_CUDA, "x")


def test_new_entry_points_validate_before_the_device():
    """The integral / scatter / rect / render entry points reject bad arguments without any
    CUDA call (so these run on a CPU-only host)."""
    lib = N.load()
    vp = ctypes.c_void_p
    # rf_box_sums: counts and pointers
    assert lib.rf_box_sums(None, 0, 4, 4, None, 0, None, None) == N.RF_OK  # nothing to do
    assert lib.rf_box_sums(None, -1, 4, 4, None, 1, None, None) == N.RF_ERR_ARGUMENT
    ptrs = (vp * 40)()
    assert lib.rf_box_sums(ptrs, 40, 4, 4, vp(1), 1, vp(1), None) == N.RF_ERR_ARGUMENT  # > 32 tables
    assert lib.rf_box_sums(ptrs, 1, 0, 4, vp(1), 1, vp(1), None) == N.RF_ERR_SHAPE
    # rf_fit_scatters: count, formulation, explicit systems need a right-hand side
    assert lib.rf_fit_scatters(None, None, None, None, -1, 0, None, None) == N.RF_ERR_ARGUMENT
    assert lib.rf_fit_scatters(None, None, None, None, 1, 7, None, None) == N.RF_ERR_ARGUMENT
    assert lib.rf_fit_scatters(vp(1), None, None, vp(1), 1, N.RF_FORM_EXPLICIT_RGBD, vp(1), None) \
        == N.RF_ERR_ARGUMENT
    assert lib.rf_fit_scatters(None, None, None, None, 0, 0, None, None) == N.RF_OK
    # rf_integral: shape and pointers
    assert lib.rf_integral(None, 4, None, 4, 4, None, None) == N.RF_ERR_ARGUMENT
    assert lib.rf_integral(vp(1), 2, None, 4, 4, vp(1), None) == N.RF_ERR_SHAPE  # pitch < width
    # entry points that need camera tables reject a null handle
    assert lib.rf_build_channel(None, None, 0, 4, None, 0, vp(1), None) == N.RF_ERR_ARGUMENT
    assert lib.rf_fit_rects(None, None, 0, 1, 4, 4, 4, None, None, 1, 0, None, None) == N.RF_ERR_ARGUMENT
    assert lib.rf_max_residuals(None, None, 0, 1, 4, 4, 4, None, None, 1, 0, None, None, None) \
        == N.RF_ERR_ARGUMENT
    assert lib.rf_render_planes(None, None, None, 1, None, None, 0.0, 0.0, None, None, None, None) \
        == N.RF_ERR_ARGUMENT
    assert "rf_render_planes" in N.last_error()
