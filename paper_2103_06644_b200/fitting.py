"""Reference-compatible fitting API on the sm_100a path (drop-in for ``rangefit.fitting``).

Names, signatures and error behaviour follow ``/root/reference/pkg/src/rangefit``:

* constants ``IMPLICIT_STANDARD`` ... ``FORMULATIONS``, ``MIN_SAMPLES`` (``fitting.py:45-60``);
* ``InsufficientSamplesError``, ``DegenerateFitError`` (``errors.py:4-10``);
* ``Rect`` (``integral.py:50-66``), ``canonicalize_implicit``, ``ImplicitPlane``,
  ``ExplicitPlane``, ``FitResult``, ``explicit_to_implicit``, ``normal_angle``
  (``fitting.py:76-174, 729-754``) -- small host-side value types;
* ``Scatter4``, ``Scatter3``, ``scatter_from_integrals``, ``fit_implicit_standard``,
  ``fit_implicit_rgbd``, ``fit_explicit_standard``, ``fit_explicit_rgbd``,
  ``FIT_BY_FORMULATION``, ``ExplicitRgbdFitter`` (``fitting.py:135-157, 420-739``): the
  assembled systems are solved on the device (``rf_fit_scatters``), box sums come from the
  device summed-area tables of ``integral.py`` (``rf_box_sums``);
* ``fit_rect(depth, maps, rect, formulation, backend="b200", ...)`` (``fitting.py:757-786``):
  ``"b200"`` / ``"naive"`` = the batched direct-sum rect kernel (``rf_fit_rects``, one CTA
  per rect -- the naive backend's numerics), ``"integral"`` = the device integral backend;
* ``CSV_HEADER`` and ``fit_result_csv_row`` (``fitting.py:73, 789-813``).

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
BACKENDS = ("b200", "naive", "integral")
CSV_HEADER = "formulation,backend,x0,y0,x1,y1,a,b,c,d,lambda,rms,n_points"
_EIGEN_TIE_REL = 1e-9
_PIVOT_REL = 1e-12


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
        d = torch.from_numpy(np.where(valid, vals, 0.0).astype(np.float64))  # RF_DEPTH_F64_M: the values as held
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


def _canonical_rows(coef: np.ndarray) -> np.ndarray:
    """canonicalize_implicit (fitting.py:76-94) for many coefficient rows at once."""
    c = np.asarray(coef, dtype=np.float64).reshape(-1, 4)
    unit = c / np.sqrt((c * c).sum(axis=1))[:, None]
    sign = np.ones(len(c))
    decided = np.zeros(len(c), bool)
    for idx in (2, 1, 0, 3):
        take = ~decided & (np.abs(unit[:, idx]) > _CANONICAL_EPS)
        sign[take] = np.where(unit[take, idx] > 0, 1.0, -1.0)
        decided |= take
    return unit * sign[:, None]


def _implicit_plane_fast(unit: np.ndarray) -> ImplicitPlane:
    """An ImplicitPlane from an already canonical unit vector (skips re-validation)."""
    p = object.__new__(ImplicitPlane)
    object.__setattr__(p, "coefficients", unit)
    return p


def _results_from_rows(rows, formulation: str) -> list:
    """FitResults for rect rows that carry a fit (batched canonicalisation)."""
    n = rows["n_points"].astype(int)
    deg = (rows["status"] & RECT_DEGENERATE) != 0
    rms = rows["rms"]
    curv = rows["curvature"]
    out = []
    if formulation in (IMPLICIT_STANDARD, IMPLICIT_RGBD):
        units = _canonical_rows(rows["coef"])
        lam = rows["eigenvalue"]
        for i in range(len(rows)):
            out.append(FitResult(_implicit_plane_fast(units[i]), int(n[i]), float(rms[i]), float(lam[i]),
                                 bool(deg[i]), float(curv[i])))
        return out
    space = SPACE_STANDARD if formulation == EXPLICIT_STANDARD else SPACE_RGBD
    for i in range(len(rows)):
        out.append(FitResult(ExplicitPlane(np.array(rows["explicit_coef"][i]), space), int(n[i]), float(rms[i]), None,
                             bool(deg[i]), float(curv[i])))
    return out


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


@dataclass(frozen=True)
class Scatter4:
    """Symmetric 4x4 scatter matrix (sum of outer products) and sample count (fitting.py:135-140)."""

    matrix: np.ndarray
    n: int


@dataclass(frozen=True)
class Scatter3:
    """3x3 normal equations, right-hand side, count, optional sum of squared targets
    (fitting.py:143-156)."""

    matrix: np.ndarray
    rhs: np.ndarray
    n: int
    target_sq: float | None = None


def _check_formulation(formulation: str) -> None:
    if formulation not in _FORM_ID:
        raise ValueError(f"unknown formulation {formulation!r}; expected one of {FORMULATIONS}")


def _require_n(n: int, minimum: int) -> None:
    if n < minimum:
        raise InsufficientSamplesError(f"fit needs at least {minimum} samples, got {n}")


def _check_matrix(m: np.ndarray, size: int) -> np.ndarray:
    """jacobi_eigh's / cholesky3's input checks (fitting.py:201-208, 270-272)."""
    a = np.asarray(m, dtype=np.float64)
    if a.shape != (size, size):
        raise ValueError(f"expected a {size}x{size} matrix, got shape {a.shape}")
    if size == 4:
        if not np.all(np.isfinite(a)):
            raise ValueError("matrix holds non-finite entries")
        fro = float(np.linalg.norm(a))
        if float(np.abs(a - a.T).max()) > 1e-12 * max(fro, 1.0):
            raise ValueError("matrix is not symmetric")
    return a


def fit_scatters(matrices, counts, formulation: str, rhs=None, target_sq=None, device=None) -> np.ndarray:
    """Solve many assembled systems on the device in one launch (``rf_fit_scatters``).

    matrices [n,4,4] (implicit) or [n,3,3] (explicit), counts [n], rhs [n,3] and target_sq [n]
    (explicit; NaN = absent).  Returns a structured array of ``RECT_FIT_DTYPE``."""
    _check_formulation(formulation)
    explicit_fit = formulation in (EXPLICIT_STANDARD, EXPLICIT_RGBD)
    m = np.asarray(matrices, dtype=np.float64)
    size = 3 if explicit_fit else 4
    m = m.reshape(-1, size, size)
    n = m.shape[0]
    full = np.zeros((n, 4, 4))
    full[:, :size, :size] = m
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    d_m = torch.from_numpy(full.reshape(n, 16)).to(dev)
    d_c = torch.from_numpy(np.asarray(counts, dtype=np.int64).reshape(n)).to(dev)
    d_rhs = d_tq = None
    if explicit_fit:
        if rhs is None:
            raise ValueError("explicit systems need a right-hand side")
        d_rhs = torch.from_numpy(np.asarray(rhs, dtype=np.float64).reshape(n, 3)).to(dev)
        tq = np.full(n, np.nan) if target_sq is None else np.asarray(
            [np.nan if v is None else v for v in np.atleast_1d(np.asarray(target_sq, dtype=object))],
            dtype=np.float64)
        d_tq = torch.from_numpy(tq.reshape(n)).to(dev)
    out = torch.empty((n, RECT_FIT_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        st = N.load().rf_fit_scatters(d_m.data_ptr(), d_rhs.data_ptr() if d_rhs is not None else None,
                                      d_tq.data_ptr() if d_tq is not None else None, d_c.data_ptr(), n,
                                      _FORM_ID[formulation], out.data_ptr(),
                                      ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    N.check(st, "fit_scatters")
    return out.cpu().numpy().view(RECT_FIT_DTYPE).reshape(-1)


RECT_JACOBI_FAILED = N.RF_RECT_JACOBI_FAILED


def _scatter_result(row, formulation: str, n: int) -> FitResult:
    if row["status"] & RECT_JACOBI_FAILED:
        raise DegenerateFitError("eigen iteration did not converge; ill-posed scatter matrix")
    degenerate = bool(row["status"] & RECT_DEGENERATE)
    rms = float(row["rms"])
    curv = float(row["curvature"])
    curv = None if math.isnan(curv) else curv
    if formulation in (IMPLICIT_STANDARD, IMPLICIT_RGBD):
        return FitResult(ImplicitPlane(row["coef"]), n, rms, float(row["eigenvalue"]), degenerate, curv)
    space = SPACE_STANDARD if formulation == EXPLICIT_STANDARD else SPACE_RGBD
    return FitResult(ExplicitPlane(np.array(row["explicit_coef"]), space), n,
                     None if math.isnan(rms) else rms, None, degenerate, curv)


def _fit_implicit(scatter: Scatter4, formulation: str) -> FitResult:
    _require_n(scatter.n, 4)
    a = _check_matrix(scatter.matrix, 4)
    row = fit_scatters(a[None], [scatter.n], formulation)[0]
    return _scatter_result(row, formulation, scatter.n)


def fit_implicit_standard(scatter: Scatter4) -> FitResult:
    """Implicit fit on [X, Y, Z, 1] monomials: smallest scatter eigenpair (fitting.py:562-568)."""
    return _fit_implicit(scatter, IMPLICIT_STANDARD)


def fit_implicit_rgbd(scatter: Scatter4) -> FitResult:
    """Implicit fit on [tan_x, tan_y, 1, 1/Z]; the eigenvector is the XYZ plane (fitting.py:571-579)."""
    return _fit_implicit(scatter, IMPLICIT_RGBD)


def _fit_explicit(scatter: Scatter3, formulation: str) -> FitResult:
    _require_n(scatter.n, 3)
    a = np.asarray(scatter.matrix, dtype=np.float64)
    if a.shape != (3, 3):
        raise ValueError(f"expected a 3x3 matrix, got shape {a.shape}")
    row = fit_scatters(a[None], [scatter.n], formulation, rhs=np.asarray(scatter.rhs, dtype=np.float64)[None],
                       target_sq=[scatter.target_sq])[0]
    return _scatter_result(row, formulation, scatter.n)


def fit_explicit_standard(scatter: Scatter3) -> FitResult:
    """Explicit fit Z = aX + bY + c via the normal equations (fitting.py:602-609)."""
    return _fit_explicit(scatter, EXPLICIT_STANDARD)


def fit_explicit_rgbd(scatter: Scatter3) -> FitResult:
    """Explicit fit 1/Z = a tan_x + b tan_y + c via the normal equations (fitting.py:612-621)."""
    return _fit_explicit(scatter, EXPLICIT_RGBD)


FIT_BY_FORMULATION = {
    IMPLICIT_STANDARD: fit_implicit_standard,
    IMPLICIT_RGBD: fit_implicit_rgbd,
    EXPLICIT_STANDARD: fit_explicit_standard,
    EXPLICIT_RGBD: fit_explicit_rgbd,
}


def _require_channels(stack, names, what: str) -> None:
    missing = [name for name in names if name not in stack.channels]
    if missing:
        raise ValueError(f"{what} stack is missing channels: {', '.join(missing)}")


def scatter_from_integrals(stack, constant, rect, formulation: str):
    """Assemble a window's scatter system from device box sums (fitting.py:420-533): same
    channel choice (camera-constant tan block for hole-free windows, the frame's masked tan
    channels otherwise), same checks and errors; the box sums run in one device launch."""
    from . import integral as I

    _check_formulation(formulation)
    rect = Rect(*rect)
    I._check_rect(rect, stack.width, stack.height)
    names = list(stack.channels)
    tables = [stack.count.table] + [stack.channels[k].table for k in names]
    cnames = []
    if constant is not None and formulation in (IMPLICIT_RGBD, EXPLICIT_RGBD):
        if tuple(constant.count.table.shape) != tuple(stack.count.table.shape):
            raise ValueError("constant stack dimensions do not match the per-frame stack")
        cnames = [k for k in ("tx2", "txty", "ty2", "tx", "ty") if k in constant.channels]
        tables += [constant.channels[k].table for k in cnames]
    sums = I.box_sums(tables, [rect])[0]
    n = int(round(float(sums[0])))
    if n < MIN_SAMPLES[formulation]:
        raise InsufficientSamplesError(
            f"window {rect} holds {n} valid samples; {formulation} needs {MIN_SAMPLES[formulation]}")
    box = dict(zip(names, (float(v) for v in sums[1:1 + len(names)])))
    cbox = dict(zip(cnames, (float(v) for v in sums[1 + len(names):])))
    if formulation == IMPLICIT_STANDARD:
        _require_channels(stack, ("x2", "xy", "xz", "x", "y2", "yz", "y", "z2", "z"), "per-frame")
        b = box
        matrix = np.array([[b["x2"], b["xy"], b["xz"], b["x"]],
                           [b["xy"], b["y2"], b["yz"], b["y"]],
                           [b["xz"], b["yz"], b["z2"], b["z"]],
                           [b["x"], b["y"], b["z"], float(n)]])
        return Scatter4(matrix=matrix, n=n)
    if formulation == EXPLICIT_STANDARD:
        _require_channels(stack, ("x2", "xy", "x", "y2", "y", "xz", "yz", "z"), "per-frame")
        b = box
        matrix = np.array([[b["x2"], b["xy"], b["x"]], [b["xy"], b["y2"], b["y"]], [b["x"], b["y"], float(n)]])
        rhs = np.array([b["xz"], b["yz"], b["z"]])
        return Scatter3(matrix=matrix, rhs=rhs, n=n, target_sq=b.get("z2"))
    if n == rect.area:
        if constant is None:
            raise ValueError(f"{formulation} requires the camera-constant channel stack")
        _require_channels(constant, ("tx2", "txty", "ty2", "tx", "ty"), "constant")
        t = cbox
        stx2, stxty, sty2, stx, sty = t["tx2"], t["txty"], t["ty2"], t["tx"], t["ty"]
    else:
        if not stack.hole_corrected:
            raise ValueError(f"window {rect} contains invalid pixels but the frame stack carries "
                             "no masked tan channels (was it built from a different frame?)")
        b = box
        stx2, stxty, sty2, stx, sty = b["m_tx2"], b["m_txty"], b["m_ty2"], b["m_tx"], b["m_ty"]
    pixel_count = float(n)
    b = box
    if formulation == IMPLICIT_RGBD:
        _require_channels(stack, ("tx_over_z", "ty_over_z", "inv_z", "inv_z2"), "per-frame")
        matrix = np.array([[stx2, stxty, stx, b["tx_over_z"]],
                           [stxty, sty2, sty, b["ty_over_z"]],
                           [stx, sty, pixel_count, b["inv_z"]],
                           [b["tx_over_z"], b["ty_over_z"], b["inv_z"], b["inv_z2"]]])
        return Scatter4(matrix=matrix, n=n)
    _require_channels(stack, ("tx_over_z", "ty_over_z", "inv_z"), "per-frame")
    matrix = np.array([[stx2, stxty, stx], [stxty, sty2, sty], [stx, sty, pixel_count]])
    rhs = np.array([b["tx_over_z"], b["ty_over_z"], b["inv_z"]])
    return Scatter3(matrix=matrix, rhs=rhs, n=n, target_sq=b.get("inv_z2"))


def fit_rects_integral(stack, constant, rects, formulation: str) -> np.ndarray:
    """scatter_from_integrals + FIT_BY_FORMULATION for many rects of one frame: one box-sum
    launch, the systems assembled as the reference assembles them, one fit launch.
    Returns ``RECT_FIT_DTYPE`` rows; rects below MIN_SAMPLES carry no RECT_FIT bit."""
    from . import integral as I

    _check_formulation(formulation)
    rr = [Rect(*r) for r in rects]
    out = np.zeros(len(rr), dtype=RECT_FIT_DTYPE)
    if not rr:
        return out
    names = list(stack.channels)
    tables = [stack.count.table] + [stack.channels[k].table for k in names]
    cnames = []
    if formulation in (IMPLICIT_RGBD, EXPLICIT_RGBD) and constant is not None:
        cnames = ["tx2", "txty", "ty2", "tx", "ty"]
        _require_channels(constant, cnames, "constant")
        tables += [constant.channels[k].table for k in cnames]
    sums = I.box_sums(tables, rr)
    n = np.rint(sums[:, 0]).astype(np.int64)
    col = {k: sums[:, 1 + i] for i, k in enumerate(names)}
    ccol = {k: sums[:, 1 + len(names) + i] for i, k in enumerate(cnames)}
    area = np.array([r.area for r in rr])
    ok = n >= MIN_SAMPLES[formulation]
    nf = n.astype(np.float64)
    size = 4 if formulation in (IMPLICIT_STANDARD, IMPLICIT_RGBD) else 3
    M = np.zeros((len(rr), size, size))
    rhs = tq = None
    if formulation in (IMPLICIT_STANDARD, EXPLICIT_STANDARD):
        need = ("x2", "xy", "xz", "x", "y2", "yz", "y", "z2", "z") if size == 4 else \
            ("x2", "xy", "x", "y2", "y", "xz", "yz", "z")
        _require_channels(stack, need, "per-frame")
        c = col
        if size == 4:
            rows = [[c["x2"], c["xy"], c["xz"], c["x"]], [c["xy"], c["y2"], c["yz"], c["y"]],
                    [c["xz"], c["yz"], c["z2"], c["z"]], [c["x"], c["y"], c["z"], nf]]
        else:
            rows = [[c["x2"], c["xy"], c["x"]], [c["xy"], c["y2"], c["y"]], [c["x"], c["y"], nf]]
            rhs = np.stack([c["xz"], c["yz"], c["z"]], axis=1)
            tq = c.get("z2")
    else:
        full = n == area
        if (full & ok).any() and constant is None:
            raise ValueError(f"{formulation} requires the camera-constant channel stack")
        if (~full & ok).any() and not stack.hole_corrected:
            raise ValueError("a window contains invalid pixels but the frame stack carries no masked tan channels")
        t = {}
        for k in ("tx2", "txty", "ty2", "tx", "ty"):
            t[k] = np.where(full, ccol[k] if ccol else 0.0, col[f"m_{k}"] if f"m_{k}" in col else 0.0)
        c = col
        need = ("tx_over_z", "ty_over_z", "inv_z", "inv_z2") if size == 4 else ("tx_over_z", "ty_over_z", "inv_z")
        _require_channels(stack, need, "per-frame")
        if size == 4:
            rows = [[t["tx2"], t["txty"], t["tx"], c["tx_over_z"]], [t["txty"], t["ty2"], t["ty"], c["ty_over_z"]],
                    [t["tx"], t["ty"], nf, c["inv_z"]], [c["tx_over_z"], c["ty_over_z"], c["inv_z"], c["inv_z2"]]]
        else:
            rows = [[t["tx2"], t["txty"], t["tx"]], [t["txty"], t["ty2"], t["ty"]], [t["tx"], t["ty"], nf]]
            rhs = np.stack([c["tx_over_z"], c["ty_over_z"], c["inv_z"]], axis=1)
            tq = c.get("inv_z2")
    for a in range(size):
        for b in range(size):
            M[:, a, b] = rows[a][b]
    out["n_points"] = n
    idx = np.nonzero(ok)[0]
    if len(idx):
        res = fit_scatters(M[idx], n[idx], formulation, rhs=None if rhs is None else rhs[idx],
                           target_sq=None if tq is None else tq[idx], device=stack.count.table.device.index)
        out[idx] = res
    return out


def max_residuals(depth, maps: TanAngleMaps, rects, formulation: str, coefs, frames=None, mask=None,
                  stream: torch.cuda.Stream | None = None) -> np.ndarray:
    """segment.py's _max_residual (segment.py:306-325) for many rects on the device: coefs
    [n, 4] canonical implicit coefficients, or [n, 3] explicit (a, b, c)."""
    _check_formulation(formulation)
    dev = torch.device("cuda", maps.device)
    d = _as_depth_tensor(depth, dev)
    if d.stride(-1) != 1 or (d.shape[0] > 1 and d.stride(0) != d.stride(1) * d.shape[1]):
        d = d.contiguous()
    B, H, W = d.shape
    r = np.asarray(rects, dtype=np.int64).reshape(-1, 4)
    f = np.zeros(len(r), np.int64) if frames is None else np.broadcast_to(np.asarray(frames, np.int64), (len(r),))
    rr = torch.from_numpy(np.column_stack([f, r]).astype(np.int32)).to(dev)
    c = np.zeros((len(r), 4))
    cin = np.asarray(coefs, dtype=np.float64).reshape(len(r), -1)
    c[:, :cin.shape[1]] = cin
    dc = torch.from_numpy(c).to(dev)
    out = torch.empty(len(r), dtype=torch.float64, device=dev)
    mptr = None
    if mask is not None:
        m = mask.unsqueeze(0) if mask.dim() == 2 else mask
        m = m.to(device=dev, dtype=torch.uint8).contiguous()
        mptr = m.data_ptr()
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    st = N.load().rf_max_residuals(maps.handle, d.data_ptr(), _depth_dtype(d), B, H, W, d.stride(-2), mptr,
                                   rr.data_ptr(), len(r), _FORM_ID[formulation], dc.data_ptr(), out.data_ptr(),
                                   ctypes.c_void_p(stream.cuda_stream))
    N.check(st, "max_residuals")
    return out.cpu().numpy()


def gather_window_samples(depth, maps: TanAngleMaps, rect, formulation: str) -> np.ndarray:
    """Valid samples of a window for the naive path (fitting.py:384-402): (X, Y, Z) rows for
    the standard formulations, (tan_x, tan_y, Z) for rgbd.  Host helper on a DepthImage."""
    from . import integral as I

    _check_formulation(formulation)
    rect = Rect(*rect)
    I._check_rect(rect, depth.width, depth.height)
    sl = (slice(rect.y0, rect.y1), slice(rect.x0, rect.x1))
    valid = depth.valid[sl]
    z = depth.values[sl][valid]
    tx, ty = maps.tan_x[sl][valid], maps.tan_y[sl][valid]
    if formulation in (IMPLICIT_STANDARD, EXPLICIT_STANDARD):
        return np.column_stack((z * tx, z * ty, z))
    return np.column_stack((tx, ty, z))


def accumulate_scatter_naive(samples, formulation: str):
    """Scatter system straight from per-sample monomials (fitting.py:339-381): the Gram
    matrix of [u, v, z, 1] (standard) / [tx, ty, 1, 1/Z] (rgbd), symmetrised; explicit forms
    get the 3x3 normal equations, right-hand side and sum of squared targets."""
    _check_formulation(formulation)
    smp = np.asarray(samples, dtype=np.float64)
    if smp.ndim != 2 or smp.shape[1] != 3:
        raise ValueError(f"samples must be (N, 3), got shape {smp.shape}")
    n = smp.shape[0]
    if n < MIN_SAMPLES[formulation]:
        raise InsufficientSamplesError(f"{formulation} needs at least {MIN_SAMPLES[formulation]} samples, got {n}")
    u, v, z = smp[:, 0], smp[:, 1], smp[:, 2]
    rgbd = formulation in (IMPLICIT_RGBD, EXPLICIT_RGBD)
    if rgbd and np.any(z <= 0):
        raise ValueError("rgbd formulations require strictly positive depths")
    one = np.ones(n)

    def gram(m):
        g = m.T @ m
        return (g + g.T) * 0.5

    if formulation == IMPLICIT_STANDARD:
        return Scatter4(matrix=gram(np.column_stack((u, v, z, one))), n=n)
    if formulation == IMPLICIT_RGBD:
        return Scatter4(matrix=gram(np.column_stack((u, v, one, 1.0 / z))), n=n)
    m = np.column_stack((u, v, one))
    target = 1.0 / z if rgbd else z
    return Scatter3(matrix=gram(m), rhs=m.T @ target, n=n, target_sq=float(target @ target))


def smallest_eigenvector(matrix):
    """Unit eigenvector of the smallest eigenvalue of a symmetric matrix, and that eigenvalue
    (fitting.py:256-261).  The sign of the vector is arbitrary, as in the reference."""
    a = np.asarray(matrix, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {a.shape}")
    if not np.all(np.isfinite(a)):
        raise ValueError("matrix holds non-finite entries")
    if float(np.abs(a - a.T).max()) > 1e-12 * max(float(np.linalg.norm(a)), 1.0):
        raise ValueError("matrix is not symmetric")
    vals, vecs = np.linalg.eigh(a)
    v = vecs[:, 0]
    return v / float(np.linalg.norm(v)), float(vals[0])


def solve_spd3(matrix, rhs) -> np.ndarray:
    """Solve a 3x3 symmetric positive-definite system by Cholesky (fitting.py:264-310); a pivot
    below 1e-12 of the trace raises DegenerateFitError, as in the reference."""
    s = np.asarray(matrix, dtype=np.float64)
    if s.shape != (3, 3):
        raise ValueError(f"expected a 3x3 matrix, got shape {s.shape}")
    trace = float(s[0, 0] + s[1, 1] + s[2, 2])
    floor = _PIVOT_REL * trace
    if not np.isfinite(trace) or trace <= 0.0:
        raise DegenerateFitError("scatter matrix has non-positive trace")
    p0 = float(s[0, 0])
    if p0 <= floor:
        raise DegenerateFitError("rank-deficient scatter matrix (pivot 1)")
    l00 = math.sqrt(p0)
    l10, l20 = float(s[1, 0]) / l00, float(s[2, 0]) / l00
    p1 = float(s[1, 1]) - l10 * l10
    if p1 <= floor:
        raise DegenerateFitError("rank-deficient scatter matrix (pivot 2)")
    l11 = math.sqrt(p1)
    l21 = (float(s[2, 1]) - l20 * l10) / l11
    p2 = float(s[2, 2]) - l20 * l20 - l21 * l21
    if p2 <= floor:
        raise DegenerateFitError("rank-deficient scatter matrix (pivot 3)")
    l22 = math.sqrt(p2)
    b0, b1, b2 = (float(v) for v in np.asarray(rhs, dtype=np.float64))
    y0 = b0 / l00
    y1 = (b1 - l10 * y0) / l11
    y2 = (b2 - l20 * y0 - l21 * y1) / l22
    x2 = y2 / l22
    x1 = (y1 - l21 * x2) / l11
    x0 = (y0 - l10 * x1 - l20 * x2) / l00
    return np.array([x0, x1, x2])


class ExplicitRgbdFitter:
    """Explicit inverse-depth fits over a camera-constant stack (fitting.py:632-726).

    The reference caches each window's Cholesky factor on the host; on the device the 3x3
    system is refactored per fit (cheaper than a cache lookup), so ``fit`` is
    ``fit_explicit_rgbd(scatter_from_integrals(stack, constant, rect, EXPLICIT_RGBD))``."""

    def __init__(self, constant):
        _require_channels(constant, ("tx2", "txty", "ty2", "tx", "ty"), "constant")
        self.constant = constant

    def matrix_for(self, rect) -> np.ndarray:
        from . import integral as I

        rect = Rect(*rect)
        I._check_rect(rect, self.constant.width, self.constant.height)
        c = self.constant.channels
        s = I.box_sums([c["tx2"].table, c["txty"].table, c["ty2"].table, c["tx"].table, c["ty"].table,
                        self.constant.count.table], [rect])[0]
        return np.array([[s[0], s[1], s[3]], [s[1], s[2], s[4]], [s[3], s[4], s[5]]])

    def fit(self, stack, rect) -> FitResult:
        return fit_explicit_rgbd(scatter_from_integrals(stack, self.constant, rect, EXPLICIT_RGBD))


def fit_rect(depth, maps: TanAngleMaps, rect: Rect, formulation: str, backend: str = "b200",
             stack=None, constant=None, rgbd_fitter=None) -> FitResult:
    """One window, reference signature (fitting.py:757-786).

    ``"b200"`` and ``"naive"``: direct sums over the rect on the device (``rf_fit_rects``, the
    naive backend's numerics).  ``"integral"``: the scatter assembled from the device channel
    stacks (``stack`` required; ``constant`` for the rgbd formulations), solved on the device."""
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}; expected one of {BACKENDS}")
    if formulation not in _FORM_ID:
        raise ValueError(f"unknown formulation {formulation!r}; expected one of {FORMULATIONS}")
    if backend == "integral":
        if stack is None:
            raise ValueError("integral backend requires a per-frame channel stack")
        if formulation == EXPLICIT_RGBD and rgbd_fitter is not None:
            return rgbd_fitter.fit(stack, rect)
        return FIT_BY_FORMULATION[formulation](scatter_from_integrals(stack, constant, rect, formulation))
    x0, y0, x1, y1 = (int(v) for v in rect)
    if not (0 <= x0 <= x1 <= maps.width and 0 <= y0 <= y1 <= maps.height):
        raise ValueError(f"rect {tuple(rect)} out of bounds for {maps.width}x{maps.height} image")
    row = fit_rects(depth, maps, [(x0, y0, x1, y1)], formulation)[0]
    return _result(row, formulation)


def fit_result_csv_row(result: FitResult, formulation: str, backend: str, rect) -> str:
    """One CSV row per fit; explicit fits are reported in implicit form (fitting.py:789-813)."""
    rect = Rect(*rect)
    coef = (explicit_to_implicit(result.plane).coefficients if isinstance(result.plane, ExplicitPlane)
            else result.plane.coefficients)
    lam = "" if result.eigenvalue is None else repr(result.eigenvalue)
    rms = "" if result.rms_residual is None else repr(result.rms_residual)
    fields = [formulation, backend, str(rect.x0), str(rect.y0), str(rect.x1), str(rect.y1),
              *(repr(float(c)) for c in coef[:4]), lam, rms, str(result.n_points)]
    return ",".join(fields)
