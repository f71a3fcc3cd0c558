"""Reference-compatible fitting API on the sm_100a path (drop-in for ``rangefit.fitting``).

Names, signatures and error behaviour follow ``/root/reference/pkg/src/rangefit``:

* constants ``IMPLICIT_STANDARD`` ... ``FORMULATIONS``, ``MIN_SAMPLES`` (``fitting.py:45-60``);
* ``InsufficientSamplesError``, ``DegenerateFitError`` (``errors.py:4-10``);
* ``Rect`` (``integral.py:50-66``), ``canonicalize_implicit``, ``ImplicitPlane``,
  ``ExplicitPlane``, ``FitResult``, ``explicit_to_implicit``, ``normal_angle``
  (``fitting.py:76-174, 729-754``) -- small host-side value types;
* ``fit_rect(depth, maps, rect, formulation, backend="b200", ...)`` (``fitting.py:757-786``)
  with a new ``"b200"`` backend (the reference's plugin point), and the batched
  ``fit_rects`` it is built on (``rf_fit_rects``, one CTA per rect, direct sums).

The fits themselves always run on the GPU through ``librangefit_b200.so``.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import torch

from . import _native as N
from .pixels import (
    EXPLICIT_RGBD,
    EXPLICIT_STANDARD,
    FORMULATIONS,
    IMPLICIT_RGBD,
    IMPLICIT_STANDARD,
    MIN_SAMPLES,
    TanAngleMaps,
    _FORM_ID,
    _depth_dtype,
)

SPACE_STANDARD = "standard"
SPACE_RGBD = "rgbd"
_CANONICAL_EPS = 1e-9
BACKENDS = ("b200",)


class InsufficientSamplesError(ValueError):
    """A window holds fewer valid samples than the formulation needs (errors.py:4-6)."""


class DegenerateFitError(ValueError):
    """The scatter system is ill-posed (errors.py:9-10)."""


class Rect(NamedTuple):
    """Half-open pixel rectangle: x in [x0, x1), y in [y0, y1) (integral.py:50-66)."""

    x0: int
    y0: int
    x1: int
    y1: int

    @property
    def area(self) -> int:
        return (self.x1 - self.x0) * (self.y1 - self.y0)

    def contains(self, other: "Rect") -> bool:
        return self.x0 <= other.x0 <= other.x1 <= self.x1 and self.y0 <= other.y0 <= other.y1 <= self.y1


def canonicalize_implicit(coefficients) -> np.ndarray:
    """Unit-normalize; make the first of (c, b, a, d) above 1e-9 positive (fitting.py:76-94)."""
    coef = np.asarray(coefficients, dtype=np.float64)
    if coef.shape != (4,):
        raise ValueError(f"expected 4 coefficients, got shape {coef.shape}")
    norm = float(np.linalg.norm(coef))
    if norm == 0 or not np.isfinite(norm):
        raise ValueError("cannot canonicalize a zero or non-finite coefficient vector")
    unit = coef / norm
    for idx in (2, 1, 0, 3):
        if abs(unit[idx]) > _CANONICAL_EPS:
            return unit if unit[idx] > 0 else -unit
    return unit


@dataclass(frozen=True)
class ImplicitPlane:
    """a*X + b*Y + c*Z + d = 0, unit norm, canonical sign (fitting.py:97-112)."""

    coefficients: np.ndarray

    def __post_init__(self) -> None:
        object.__setattr__(self, "coefficients", canonicalize_implicit(self.coefficients))

    @property
    def normal(self) -> np.ndarray:
        return self.coefficients[:3]

    @property
    def offset(self) -> float:
        return float(self.coefficients[3])


@dataclass(frozen=True)
class ExplicitPlane:
    """Z = aX + bY + c (standard) or 1/Z = a tan_x + b tan_y + c (rgbd) (fitting.py:115-132)."""

    coefficients: np.ndarray
    space: str

    def __post_init__(self) -> None:
        coef = np.asarray(self.coefficients, dtype=np.float64)
        if coef.shape != (3,):
            raise ValueError(f"expected 3 coefficients, got shape {coef.shape}")
        if self.space not in (SPACE_STANDARD, SPACE_RGBD):
            raise ValueError(f"unknown plane space {self.space!r}")
        object.__setattr__(self, "coefficients", coef)


@dataclass(frozen=True)
class FitResult:
    """A fitted plane plus diagnostics (fitting.py:158-174)."""

    plane: ImplicitPlane | ExplicitPlane
    n_points: int
    rms_residual: float | None
    eigenvalue: float | None = None
    degenerate: bool = False
    curvature: float | None = None  # SURVEY.md A17 extension (not in the reference)


def explicit_to_implicit(plane: ExplicitPlane) -> ImplicitPlane:
    """(a, b, -1, c) standard, (a, b, c, -1) rgbd (fitting.py:729-739)."""
    a, b, c = (float(v) for v in plane.coefficients)
    if plane.space == SPACE_STANDARD:
        return ImplicitPlane(np.array([a, b, -1.0, c]))
    return ImplicitPlane(np.array([a, b, c, -1.0]))


def normal_angle(p: ImplicitPlane, q: ImplicitPlane) -> float:
    """Orientation-blind angle between plane normals, atan2(|n x m|, |n.m|) (fitting.py:742-754)."""
    np_, nq = p.normal, q.normal
    denom = float(np.linalg.norm(np_) * np.linalg.norm(nq))
    if denom == 0:
        raise ValueError("degenerate normal")
    return math.atan2(float(np.linalg.norm(np.cross(np_, nq))), abs(float(np_ @ nq)))


# rf_rect_fit (include/rangefit_b200.h) as a numpy structured dtype
RECT_FIT_DTYPE = np.dtype([("coef", "<f8", 4), ("explicit_coef", "<f8", 3), ("eigenvalue", "<f8"),
                           ("rms", "<f8"), ("curvature", "<f8"), ("n_points", "<i4"), ("status", "<i4")])
RECT_FIT = N.RF_PIX_FIT
RECT_DEGENERATE = N.RF_PIX_DEGENERATE
RECT_OUT_OF_BOUNDS = 16


def _as_depth_tensor(depth, device) -> torch.Tensor:
    """Accept a CUDA tensor [B,H,W]/[H,W] or a reference-style object with ``.values``/``.valid``."""
    if isinstance(depth, torch.Tensor):
        d = depth
    elif hasattr(depth, "values"):
        vals = np.asarray(depth.values)
        valid = np.asarray(getattr(depth, "valid", np.isfinite(vals) & (vals > 0)), dtype=bool)
        d = torch.from_numpy(np.where(valid, vals, 0.0).astype(np.float32))
    else:
        d = torch.as_tensor(np.asarray(depth))
    if not d.is_cuda:
        d = d.to(device)
    return d.unsqueeze(0) if d.dim() == 2 else d


def fit_rects(depth, maps: TanAngleMaps, rects, formulation: str, frames=None, mask=None,
              stream: torch.cuda.Stream | None = None) -> np.ndarray:
    """Fit every rect (x0, y0, x1, y1) of ``frames`` (default frame 0) on the GPU.

    Returns a structured numpy array of ``RECT_FIT_DTYPE`` (one row per rect)."""
    if formulation not in _FORM_ID:
        raise ValueError(f"unknown formulation {formulation!r}; expected one of {FORMULATIONS}")
    dev = torch.device("cuda", maps.device)
    d = _as_depth_tensor(depth, dev)
    if d.stride(-1) != 1 or (d.shape[0] > 1 and d.stride(0) != d.stride(1) * d.shape[1]):
        d = d.contiguous()
    B, H, W = d.shape
    if (H, W) != (maps.height, maps.width):
        raise ValueError(f"depth {W}x{H} does not match maps {maps.width}x{maps.height}")
    r = np.asarray(rects, dtype=np.int64).reshape(-1, 4)
    f = np.zeros(len(r), np.int64) if frames is None else np.broadcast_to(np.asarray(frames, np.int64), (len(r),))
    rr = torch.from_numpy(np.column_stack([f, r]).astype(np.int32)).to(dev)
    out = torch.empty((len(r), RECT_FIT_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    mptr = None
    if mask is not None:
        m = mask.unsqueeze(0) if mask.dim() == 2 else mask
        m = m.to(device=dev, dtype=torch.uint8).contiguous()
        mptr = m.data_ptr()
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    lib = N.load()
    st = lib.rf_fit_rects(maps.handle, d.data_ptr(), _depth_dtype(d), B, H, W, d.stride(-2), mptr,
                          rr.data_ptr(), len(r), _FORM_ID[formulation], out.data_ptr(),
                          ctypes.c_void_p(stream.cuda_stream))
    N.check(st, "fit_rects")
    return out.cpu().numpy().view(RECT_FIT_DTYPE).reshape(-1)


def _result(row, formulation: str) -> FitResult:
    if row["status"] & RECT_OUT_OF_BOUNDS:
        raise ValueError("rect out of bounds")
    n = int(row["n_points"])
    if not row["status"] & RECT_FIT:
        raise InsufficientSamplesError(
            f"window holds {n} valid samples; {formulation} needs {MIN_SAMPLES[formulation]}")
    degenerate = bool(row["status"] & RECT_DEGENERATE)
    if formulation in (IMPLICIT_STANDARD, IMPLICIT_RGBD):
        return FitResult(ImplicitPlane(row["coef"]), n, float(row["rms"]), float(row["eigenvalue"]),
                         degenerate, float(row["curvature"]))
    space = SPACE_STANDARD if formulation == EXPLICIT_STANDARD else SPACE_RGBD
    return FitResult(ExplicitPlane(np.array(row["explicit_coef"]), space), n, float(row["rms"]), None,
                     degenerate, float(row["curvature"]))


def fit_rect(depth, maps: TanAngleMaps, rect: Rect, formulation: str, backend: str = "b200",
             stack=None, constant=None, rgbd_fitter=None) -> FitResult:
    """One window, reference signature (fitting.py:757-766).  ``backend`` must be ``"b200"``;
    ``stack``/``constant``/``rgbd_fitter`` are accepted for signature compatibility and unused
    (the device path sums each rect directly)."""
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}; expected one of {BACKENDS}")
    if formulation not in _FORM_ID:
        raise ValueError(f"unknown formulation {formulation!r}; expected one of {FORMULATIONS}")
    x0, y0, x1, y1 = (int(v) for v in rect)
    if not (0 <= x0 <= x1 <= maps.width and 0 <= y0 <= y1 <= maps.height):
        raise ValueError(f"rect {tuple(rect)} out of bounds for {maps.width}x{maps.height} image")
    row = fit_rects(depth, maps, [(x0, y0, x1, y1)], formulation)[0]
    return _result(row, formulation)
