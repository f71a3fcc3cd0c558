"""ctypes binding of the C ABI in ``include/rangefit_b200.h``.

The shared library ``librangefit_b200.so`` is built in-tree by
``paper_2103_06644_b200.build`` (``__graft_entry__.build()``).  There is no
fallback: if the library is missing every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_NAME = "librangefit_b200.so"
LIB_PATH = Path(os.environ["RF_LIB_PATH"]) if os.environ.get("RF_LIB_PATH") else PKG_DIR / LIB_NAME

RF_OK = 0
RF_ERR_ARGUMENT = 1
RF_ERR_SHAPE = 2
RF_ERR_CUDA = 3
RF_ERR_UNSUPPORTED = 4

RF_DEPTH_F32_M = 0
RF_DEPTH_U16_MM = 1
RF_DEPTH_F64_M = 2

RF_FORM_IMPLICIT_STANDARD = 0
RF_FORM_IMPLICIT_RGBD = 1
RF_FORM_EXPLICIT_STANDARD = 2
RF_FORM_EXPLICIT_RGBD = 3
RF_NUM_FORMULATIONS = 4
RF_IMPLICIT_STANDARD = 1 << RF_FORM_IMPLICIT_STANDARD
RF_IMPLICIT_RGBD = 1 << RF_FORM_IMPLICIT_RGBD
RF_EXPLICIT_STANDARD = 1 << RF_FORM_EXPLICIT_STANDARD
RF_EXPLICIT_RGBD = 1 << RF_FORM_EXPLICIT_RGBD
RF_ABI_VERSION = 4

RF_PIX_INPUT_VALID = 1
RF_PIX_FIT = 2
RF_PIX_DEGENERATE = 4

RF_RECT_JACOBI_FAILED = 8

# rf_channel ids (integral.py channel names)
RF_CHANNELS = {
    "count": 0, "ones": 1,
    "x2": 2, "xy": 3, "xz": 4, "x": 5, "y2": 6, "yz": 7, "y": 8, "z2": 9, "z": 10,
    "tx_over_z": 11, "ty_over_z": 12, "inv_z": 13, "inv_z2": 14,
    "tx2": 15, "txty": 16, "ty2": 17, "tx": 18, "ty": 19,
    "m_tx2": 20, "m_txty": 21, "m_ty2": 22, "m_tx": 23, "m_ty": 24,
}
RF_MAX_BOX_CHANNELS = 32

# every symbol include/rangefit_b200.h declares
EXPORTED_SYMBOLS = (
    "rf_tables_create",
    "rf_tables_destroy",
    "rf_fit_pixels",
    "rf_fit_rects",
    "rf_build_channel",
    "rf_integral",
    "rf_box_sums",
    "rf_fit_scatters",
    "rf_render_planes",
    "rf_max_residuals",
    "rf_launches_per_call",
    "rf_last_error",
    "rf_abi_version",
)


class RfIntrinsics(ctypes.Structure):
    _fields_ = [
        ("fx", ctypes.c_double),
        ("fy", ctypes.c_double),
        ("cx", ctypes.c_double),
        ("cy", ctypes.c_double),
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
    ]


class RfPixelOut(ctypes.Structure):
    _fields_ = [
        ("normal", ctypes.c_void_p),
        ("offset", ctypes.c_void_p),
        ("residual", ctypes.c_void_p),
        ("curvature", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
    ]


class NativeLibraryMissing(RuntimeError):
    """The sm_100a extension is not built; there is no CPU fallback."""


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryMissing(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the sm_100a path has no CPU fallback)"
        )
    L = ctypes.CDLL(str(LIB_PATH))
    vp = ctypes.c_void_p
    L.rf_tables_create.argtypes = [ctypes.POINTER(RfIntrinsics), vp, vp, ctypes.c_int, ctypes.POINTER(vp)]
    L.rf_tables_create.restype = ctypes.c_int
    L.rf_tables_destroy.argtypes = [vp]
    L.rf_tables_destroy.restype = ctypes.c_int
    L.rf_fit_pixels.argtypes = [
        vp, vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, vp,
        ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(RfPixelOut), vp,
    ]
    L.rf_fit_pixels.restype = ctypes.c_int
    L.rf_fit_rects.argtypes = [
        vp, vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, vp,
        vp, ctypes.c_int64, ctypes.c_int32, vp, vp,
    ]
    L.rf_fit_rects.restype = ctypes.c_int
    L.rf_build_channel.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int64, vp, ctypes.c_int32, vp, vp]
    L.rf_build_channel.restype = ctypes.c_int
    L.rf_integral.argtypes = [vp, ctypes.c_int64, vp, ctypes.c_int32, ctypes.c_int32, vp, vp]
    L.rf_integral.restype = ctypes.c_int
    L.rf_box_sums.argtypes = [ctypes.POINTER(vp), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, vp,
                              ctypes.c_int64, vp, vp]
    L.rf_box_sums.restype = ctypes.c_int
    L.rf_fit_scatters.argtypes = [vp, vp, vp, vp, ctypes.c_int64, ctypes.c_int32, vp, vp]
    L.rf_fit_scatters.restype = ctypes.c_int
    L.rf_render_planes.argtypes = [vp, vp, vp, ctypes.c_int32, vp, vp, ctypes.c_double, ctypes.c_double, vp, vp,
                                   vp, vp]
    L.rf_render_planes.restype = ctypes.c_int
    L.rf_max_residuals.argtypes = [
        vp, vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, vp,
        vp, ctypes.c_int64, ctypes.c_int32, vp, vp, vp,
    ]
    L.rf_max_residuals.restype = ctypes.c_int
    L.rf_launches_per_call.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                        ctypes.c_int32, ctypes.c_int32]
    L.rf_launches_per_call.restype = ctypes.c_int32
    L.rf_last_error.argtypes = []
    L.rf_last_error.restype = ctypes.c_char_p
    L.rf_abi_version.argtypes = []
    L.rf_abi_version.restype = ctypes.c_int32
    if L.rf_abi_version() != RF_ABI_VERSION:
        raise NativeLibraryMissing(f"{LIB_PATH} has ABI {L.rf_abi_version()}, expected {RF_ABI_VERSION}: rebuild")
    _lib = L
    return L


def last_error() -> str:
    return load().rf_last_error().decode(errors="replace")


def check(status: int, what: str) -> None:
    """Map an rf_status onto the reference's exception conventions."""
    if status == RF_OK:
        return
    msg = f"{what}: {last_error()}"
    if status in (RF_ERR_ARGUMENT, RF_ERR_SHAPE):
        raise ValueError(msg)
    if status == RF_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)
