"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper around the CPU restatement in
``oracle/rf_oracle.c`` (the parity checker and the timed CPU baseline).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module.  The
product path (``paper_2103_06644_b200``) never does.

The host-side helpers restate the reference's input conventions so the oracle
and the GPU read the same bits:

* :func:`tan_maps` -- ``compute_tan_maps`` (reference ``camera.py:124-135``):
  ``tan_x = (cols + delta_x - cx) / fx``, ``tan_y = (rows + delta_y - cy) / fy``.
* :func:`depth_from_meters` -- ``DepthImage.__post_init__`` (``synth.py:80-94``):
  values cast to float64, ``valid = mask & isfinite & > 0``.
* :func:`depth_from_millimeters` -- ``DepthImage.from_millimeters``
  (``synth.py:111-114``): ``mm.astype(float64) / 1000.0``, ``valid = mm > 0``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "librf_oracle.so"

STANDARD = 0  # reference "implicit-standard"
RGBD = 1  # reference "implicit-rgbd" (disparity form)
EXPLICIT_STANDARD = 2  # reference "explicit-standard"
EXPLICIT_RGBD = 3  # reference "explicit-rgbd"
NAIVE = 0
INTEGRAL = 1

FORMULATION_CODES = {"implicit-standard": STANDARD, "implicit-rgbd": RGBD,
                     "explicit-standard": EXPLICIT_STANDARD, "explicit-rgbd": EXPLICIT_RGBD}

_lib = None


def build() -> Path:
    """Compile the oracle with its Makefile (plain gcc, no reference build system)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.POINTER(ctypes.c_float)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        i64p = ctypes.POINTER(ctypes.c_int64)
        L.rfo_fit_pixels.argtypes = [
            dp, u8p, dp, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            i64p, ctypes.c_int64, fp, fp, fp, fp, u8p, dp, dp, dp, dp, ctypes.c_int,
        ]
        L.rfo_fit_pixels.restype = ctypes.c_int
        L.rfo_fit_scatter.argtypes = [
            dp, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, ctypes.POINTER(ctypes.c_int),
        ]
        L.rfo_fit_scatter.restype = ctypes.c_int
        L.rfo_jacobi_eigh.argtypes = [ctypes.c_int, dp, dp, dp]
        L.rfo_jacobi_eigh.restype = ctypes.c_int
        L.rfo_max_threads.restype = ctypes.c_int
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.rfo_fit_rects.argtypes = [dp, u8p, dp, dp, ctypes.c_int, ctypes.c_int, i32p, ctypes.c_int64,
                                    ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, i32p, i32p]
        L.rfo_fit_rects.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def tan_maps(fx, fy, cx, cy, width, height, delta_x=None, delta_y=None):
    """compute_tan_maps restated (reference camera.py:124-135)."""
    if delta_x is None:
        delta_x = np.zeros((height, width))
    if delta_y is None:
        delta_y = np.zeros((height, width))
    cols = np.arange(width, dtype=np.float64)
    rows = np.arange(height, dtype=np.float64)
    tan_x = (cols[None, :] + np.asarray(delta_x, np.float64) - cx) / fx
    tan_y = (rows[:, None] + np.asarray(delta_y, np.float64) - cy) / fy
    return np.ascontiguousarray(tan_x), np.ascontiguousarray(tan_y)


def depth_from_meters(values, mask=None):
    """DepthImage(values, valid=mask) restated (reference synth.py:80-94)."""
    v = np.asarray(values, dtype=np.float64)
    positive = np.isfinite(v) & (v > 0)
    valid = positive if mask is None else (np.asarray(mask, dtype=bool) & positive)
    return v, valid


def depth_from_millimeters(mm):
    """DepthImage.from_millimeters restated (reference synth.py:111-114)."""
    mm = np.asarray(mm)
    return depth_from_meters(mm.astype(np.float64) / 1000.0, mm > 0)


def max_threads() -> int:
    return int(lib().rfo_max_threads())


def fit_pixels(values, valid, tan_x, tan_y, window, formulation, backend=NAIVE, pixels=None,
               nthreads=0, want_coef=False):
    """Per-pixel windowed implicit fit on one (H, W) frame.

    Returns a dict with ``normal`` (P,3) f32, ``offset``/``residual``/``curvature`` (P,) f32
    and ``status`` (P,) u8, where P = H*W (or len(pixels)), ``scale`` = ||S||_F / n (P,)
    f64 (the rounding floor of lambda), ``curv_cond`` = sum of the uncentred monomial
    diagonal / trace of the centred scatter (the rounding amplification of the curvature); optionally the canonical
    fp64 coefficient vector ``coef`` (P,4) and smallest eigenvalue ``lam`` (for the explicit
    formulations ``coef`` is explicit_to_implicit of the fit and ``lam`` the residual sum
    of squares sum(b^2) - alpha.rhs).
    """
    if isinstance(formulation, str):
        formulation = FORMULATION_CODES[formulation]
    values = np.ascontiguousarray(values, dtype=np.float64)
    valid = np.ascontiguousarray(valid, dtype=np.uint8)
    tan_x = np.ascontiguousarray(np.broadcast_to(tan_x, values.shape), dtype=np.float64)
    tan_y = np.ascontiguousarray(np.broadcast_to(tan_y, values.shape), dtype=np.float64)
    H, W = values.shape
    if pixels is None:
        pix_arr = None
        P = H * W
    else:
        pix_arr = np.ascontiguousarray(pixels, dtype=np.int64)
        P = pix_arr.size
    out = {
        "normal": np.empty((P, 3), np.float32),
        "offset": np.empty(P, np.float32),
        "residual": np.empty(P, np.float32),
        "curvature": np.empty(P, np.float32),
        "status": np.empty(P, np.uint8),
    }
    coef = np.empty((P, 4), np.float64) if want_coef else None
    lam = np.empty(P, np.float64) if want_coef else None
    scale = np.empty(P, np.float64)
    curv_cond = np.empty(P, np.float64)
    rc = lib().rfo_fit_pixels(
        _ptr(values, ctypes.c_double), _ptr(valid, ctypes.c_uint8), _ptr(tan_x, ctypes.c_double),
        _ptr(tan_y, ctypes.c_double), H, W, int(window), int(formulation), int(backend),
        None if pix_arr is None else _ptr(pix_arr, ctypes.c_int64), P,
        _ptr(out["normal"], ctypes.c_float), _ptr(out["offset"], ctypes.c_float),
        _ptr(out["residual"], ctypes.c_float), _ptr(out["curvature"], ctypes.c_float),
        _ptr(out["status"], ctypes.c_uint8),
        None if coef is None else _ptr(coef, ctypes.c_double),
        None if lam is None else _ptr(lam, ctypes.c_double), _ptr(scale, ctypes.c_double),
        _ptr(curv_cond, ctypes.c_double), int(nthreads),
    )
    if rc != 0:
        raise ValueError(f"oracle rfo_fit_pixels failed with code {rc}")
    out["scale"] = scale
    out["curv_cond"] = curv_cond
    if want_coef:
        out["coef"] = coef
        out["lam"] = lam
    return out


def fit_scatter(matrix, n, formulation):
    """_fit_implicit on a given 4x4 scatter (reference fitting.py:546-559)."""
    if isinstance(formulation, str):
        formulation = FORMULATION_CODES[formulation]
    S = np.ascontiguousarray(matrix, dtype=np.float64)
    coef = np.empty(4)
    lam = ctypes.c_double()
    rms = ctypes.c_double()
    curv = ctypes.c_double()
    deg = ctypes.c_int()
    rc = lib().rfo_fit_scatter(_ptr(S, ctypes.c_double), int(n), int(formulation),
                               _ptr(coef, ctypes.c_double), ctypes.byref(lam), ctypes.byref(rms),
                               ctypes.byref(curv), ctypes.byref(deg))
    return {"coef": coef, "lam": lam.value, "rms": rms.value, "curvature": curv.value,
            "degenerate": bool(deg.value), "converged": rc == 0}


def jacobi_eigh(matrix):
    """jacobi_eigh restated (reference fitting.py:193-253)."""
    m = np.ascontiguousarray(matrix, dtype=np.float64)
    n = m.shape[0]
    vals = np.empty(n)
    vecs = np.empty((n, n))
    rc = lib().rfo_jacobi_eigh(n, _ptr(m, ctypes.c_double), _ptr(vals, ctypes.c_double),
                               _ptr(vecs, ctypes.c_double))
    return vals, vecs, rc == 0


def fit_rects(values, valid, tan_x, tan_y, rects, formulation, backend=NAIVE):
    """fit_rect for a list of (x0, y0, x1, y1) rects of one frame (reference fitting.py:757-786).
    Returns coef (R,4) canonical implicit, lam, rms, curvature, n (R,), status (R,) with bit1
    fitted, bit2 degenerate, bit4 out of bounds."""
    if isinstance(formulation, str):
        formulation = FORMULATION_CODES[formulation]
    values = np.ascontiguousarray(values, dtype=np.float64)
    valid = np.ascontiguousarray(valid, dtype=np.uint8)
    H, W = values.shape
    tan_x = np.ascontiguousarray(np.broadcast_to(tan_x, values.shape), dtype=np.float64)
    tan_y = np.ascontiguousarray(np.broadcast_to(tan_y, values.shape), dtype=np.float64)
    r = np.ascontiguousarray(np.asarray(rects, dtype=np.int32).reshape(-1, 4))
    R = r.shape[0]
    out = {"coef": np.empty((R, 4)), "lam": np.empty(R), "rms": np.empty(R), "curvature": np.empty(R),
           "n": np.empty(R, np.int32), "status": np.empty(R, np.int32)}
    rc = lib().rfo_fit_rects(
        _ptr(values, ctypes.c_double), _ptr(valid, ctypes.c_uint8), _ptr(tan_x, ctypes.c_double),
        _ptr(tan_y, ctypes.c_double), H, W, _ptr(r, ctypes.c_int32), R, int(formulation), int(backend),
        _ptr(out["coef"], ctypes.c_double), _ptr(out["lam"], ctypes.c_double), _ptr(out["rms"], ctypes.c_double),
        _ptr(out["curvature"], ctypes.c_double), _ptr(out["n"], ctypes.c_int32), _ptr(out["status"], ctypes.c_int32))
    if rc != 0:
        raise ValueError(f"oracle rfo_fit_rects failed with code {rc}")
    return out
