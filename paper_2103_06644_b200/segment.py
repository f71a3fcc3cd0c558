"""Quadtree planar segmentation on the batched GPU rect fits.

Same behaviour as the reference's ``segment()`` (``segment.py:327-431``): the frame is
cut into a square grid, each tile is fitted, tiles whose fit is degenerate or whose
rms residual exceeds the threshold split into four children up to ``max_depth``,
tiles with too few valid pixels are rejected, and k-means over the fitted tiles'
plane features groups coplanar tiles.

B200 design: the quadtree is evaluated **level-synchronously** -- every pending tile
of a level is fitted in ONE launch instead of one Python ``fit_rect`` per tile:
``rf_fit_rects`` (one CTA per tile, direct sums) for the ``"b200"`` / ``"naive"``
backends, or one ``rf_box_sums`` + one ``rf_fit_scatters`` launch over the frame's device
channel stack for ``"integral"``; ``error_metric="max"`` adds one ``rf_max_residuals``
launch per level (``_max_residual``, segment.py:306-325).  Each tile's decision depends only on
its own fit, so the leaf set equals the reference's; the leaves are then listed in
the reference's LIFO traversal order so that k-means (which seeds by sample index)
sees the same sequence.  k-means runs on the host: it clusters a few hundred
4-vectors and must reproduce the reference's numpy ``default_rng`` seeding.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from . import fitting as F
from .pixels import EXPLICIT_RGBD, EXPLICIT_STANDARD, FORMULATIONS, IMPLICIT_RGBD, IMPLICIT_STANDARD, TanAngleMaps

UNLABELED = -1
MIN_TILE_EDGE = 2  # segment.py:62-64: a 2x2 tile still holds 4 samples
DEFAULT_THRESHOLDS = {IMPLICIT_STANDARD: 8e-3, IMPLICIT_RGBD: 8e-3, EXPLICIT_STANDARD: 0.02, EXPLICIT_RGBD: 8e-3}


class TileStatus(enum.Enum):
    FITTED = "fitted"
    TOO_INVALID = "too_invalid"
    HIGH_ERROR = "high_error_leaf"


@dataclass(frozen=True)
class SegConfig:
    """Segmentation knobs (reference segment.py:81-130).  Every backend runs on the device:
    ``"b200"``/``"naive"`` direct sums per tile, ``"integral"`` the frame's channel stack."""

    formulation: str = IMPLICIT_RGBD
    backend: str = "b200"
    initial_tile: int = 64
    max_depth: int = 3
    rms_threshold: float | None = None
    min_valid_fraction: float = 0.5
    k: int = 8
    seed: int = 0
    d_scale: float = 5.0
    error_metric: str = "rms"

    def __post_init__(self) -> None:
        if self.formulation not in FORMULATIONS:
            raise ValueError(f"unknown formulation {self.formulation!r}")
        if self.backend not in F.BACKENDS:
            raise ValueError(f"unknown backend {self.backend!r}")
        if self.max_depth < 0:
            raise ValueError("max_depth must be non-negative")
        if self.initial_tile < (1 << self.max_depth) * MIN_TILE_EDGE:
            raise ValueError(f"initial_tile {self.initial_tile} cannot survive {self.max_depth} subdivisions")
        if self.threshold <= 0:
            raise ValueError("rms_threshold must be positive")
        if not 0.0 <= self.min_valid_fraction <= 1.0:
            raise ValueError("min_valid_fraction must be in [0, 1]")
        if self.k < 1:
            raise ValueError("k must be at least 1")
        if self.d_scale <= 0:
            raise ValueError("d_scale must be positive")
        if self.error_metric not in ("rms", "max"):
            raise ValueError(f"unknown error metric {self.error_metric!r}")

    @property
    def threshold(self) -> float:
        return self.rms_threshold if self.rms_threshold is not None else DEFAULT_THRESHOLDS[self.formulation]


@dataclass
class Tile:
    rect: F.Rect
    status: TileStatus
    level: int
    result: F.FitResult | None = None
    cluster: int = UNLABELED


@dataclass
class Segmentation:
    tiles: list
    labels: torch.Tensor
    centroids: np.ndarray
    n_fitted: int
    n_too_invalid: int
    n_high_error: int
    warnings: list = field(default_factory=list)


def tile_features(result: F.FitResult, d_scale: float = 5.0) -> np.ndarray:
    """Plane scaled to a unit normal with offset >= 0, offset / d_scale (segment.py:199-214)."""
    coef = (F.explicit_to_implicit(result.plane).coefficients if isinstance(result.plane, F.ExplicitPlane)
            else result.plane.coefficients).copy()
    norm = float(np.linalg.norm(coef[:3]))
    if norm == 0:
        raise ValueError("fit has a degenerate normal")
    coef /= norm
    flip = coef[3] < 0
    if coef[3] == 0:
        for v in (coef[2], coef[1], coef[0]):
            if abs(v) > 1e-12:
                flip = v < 0
                break
    if flip:
        coef = -coef
    return np.array([coef[0], coef[1], coef[2], coef[3] / d_scale])


def _features(tiles, d_scale: float) -> np.ndarray:
    """tile_features for many fitted tiles at once (same arithmetic, vectorised)."""
    rows = []
    for t in tiles:
        pl = t.result.plane
        rows.append(F.explicit_to_implicit(pl).coefficients if isinstance(pl, F.ExplicitPlane) else pl.coefficients)
    coef = np.array(rows, dtype=np.float64)
    norm = np.sqrt((coef[:, :3] * coef[:, :3]).sum(axis=1))
    if np.any(norm == 0):
        raise ValueError("fit has a degenerate normal")
    coef = coef / norm[:, None]
    flip = coef[:, 3] < 0
    zero = coef[:, 3] == 0
    if zero.any():
        for i in np.nonzero(zero)[0]:
            for v in (coef[i, 2], coef[i, 1], coef[i, 0]):
                if abs(v) > 1e-12:
                    flip[i] = v < 0
                    break
    coef[flip] = -coef[flip]
    coef[:, 3] /= d_scale
    return coef


def kmeans(features: np.ndarray, k: int, seed: int = 0, max_iter: int = 100):
    """Lloyd's k-means, k-means++ seeding from numpy default_rng(seed) (segment.py:224-269)."""
    x = np.asarray(features, dtype=np.float64)
    if x.ndim != 2 or x.shape[0] == 0:
        raise ValueError(f"features must be a non-empty (n, d) array, got {x.shape}")
    n = x.shape[0]
    if k < 1:
        raise ValueError("k must be at least 1")
    k = min(k, n)
    rng = np.random.default_rng(seed)
    cent = np.empty((k, x.shape[1]))
    cent[0] = x[rng.integers(n)]
    for i in range(1, k):
        d2 = ((x[:, None, :] - cent[None, :i, :]) ** 2).sum(axis=2).min(axis=1)
        tot = float(d2.sum())
        if tot == 0.0:
            cent[i:] = x[rng.integers(n, size=k - i)]
            break
        cent[i] = x[rng.choice(n, p=d2 / tot)]
    labels = np.full(n, -1)
    for _ in range(max_iter):
        dist = ((x[:, None, :] - cent[None, :, :]) ** 2).sum(axis=2)
        new = dist.argmin(axis=1)
        if np.array_equal(new, labels):
            break
        labels = new
        for j in range(k):
            members = x[labels == j]
            cent[j] = members.mean(axis=0) if len(members) else x[int(dist.min(axis=1).argmax())]
    return labels, cent


def _grid(width: int, height: int, tile: int):
    return [F.Rect(x, y, min(x + tile, width), min(y + tile, height))
            for y in range(0, height, tile) for x in range(0, width, tile)]


def _children(r: F.Rect):
    xm, ym = r.x0 + (r.x1 - r.x0) // 2, r.y0 + (r.y1 - r.y0) // 2
    return [F.Rect(r.x0, r.y0, xm, ym), F.Rect(xm, r.y0, r.x1, ym),
            F.Rect(r.x0, ym, xm, r.y1), F.Rect(xm, ym, r.x1, r.y1)]


def build_frame_stack(depth, maps: TanAngleMaps, formulation: str):
    """The per-frame channel stack a formulation needs, with residuals (segment.py:272-285)."""
    from . import integral as I

    if formulation == IMPLICIT_STANDARD:
        return I.build_standard_implicit_channels(depth, maps)
    if formulation == IMPLICIT_RGBD:
        return I.build_rgbd_implicit_channels(depth, maps)
    if formulation == EXPLICIT_STANDARD:
        return I.build_standard_explicit_channels(depth, maps, include_residual=True)
    if formulation == EXPLICIT_RGBD:
        return I.build_rgbd_explicit_channels(depth, maps, include_residual=True)
    raise ValueError(f"unknown formulation {formulation!r}")


def segment(depth, maps: TanAngleMaps, config: SegConfig, constant=None, frame: int = 0,
            mask=None) -> Segmentation:
    """Segment one frame (reference signature segment.py:327-333; ``depth`` a DepthImage or a
    device tensor [H,W] / [B,H,W] with ``frame`` selecting the frame)."""
    from . import integral as I

    d = F._as_depth_tensor(depth, torch.device("cuda", maps.device))
    H, W = d.shape[-2:]
    if W < 1 or H < 1:
        raise ValueError("empty depth image")
    if W < MIN_TILE_EDGE or H < MIN_TILE_EDGE:
        raise ValueError(f"image {W}x{H} is smaller than one fittable tile")
    stack = None
    if config.backend == "integral":
        if config.formulation in (IMPLICIT_RGBD, EXPLICIT_RGBD) and constant is None:
            constant = I.build_constant_channels(maps)
        fd = d[frame]
        if mask is not None:
            m = (mask[frame] if mask.dim() == 3 else mask).to(fd.device).bool()
            fd = torch.where(m, fd, torch.zeros((), dtype=fd.dtype, device=fd.device))
        stack = build_frame_stack(fd, maps, config.formulation)
    implicit = config.formulation in (IMPLICIT_STANDARD, IMPLICIT_RGBD)
    decided = {}   # rect -> (kind, result); kind in {"fit", "invalid", "split", "high"}
    level_rects = [(r, 0) for r in _grid(W, H, config.initial_tile)]
    while level_rects:
        rects = [tuple(r) for r, _ in level_rects]
        if stack is not None:
            rows = F.fit_rects_integral(stack, constant, rects, config.formulation)
        else:
            rows = F.fit_rects(d, maps, rects, config.formulation, frames=frame, mask=mask)
        area = np.array([r.area for r, _ in level_rects])
        n_valid = rows["n_points"].astype(np.int64)
        fitted = (n_valid >= config.min_valid_fraction * area) & (n_valid > 0) & ((rows["status"] & F.RECT_FIT) != 0)
        degenerate = (rows["status"] & F.RECT_DEGENERATE) != 0
        fidx = np.nonzero(fitted)[0]
        if config.error_metric == "max":
            err = np.full(len(rows), np.inf)
            if len(fidx):
                coefs = F._canonical_rows(rows["coef"][fidx]) if implicit else rows["explicit_coef"][fidx]
                err[fidx] = F.max_residuals(d, maps, [rects[i] for i in fidx], config.formulation, coefs,
                                            frames=frame, mask=mask)
        else:
            err = np.where(np.isnan(rows["rms"]), np.inf, rows["rms"])
        accept = fitted & ~degenerate & (err <= config.threshold)
        nxt = []
        leaves = []
        for i, (r, lev) in enumerate(level_rects):
            if not fitted[i]:
                decided[r] = ("invalid", None)
            elif accept[i]:
                decided[r] = ("fit", i)
                leaves.append(i)
            elif lev < config.max_depth and r.x1 - r.x0 >= 2 * MIN_TILE_EDGE and r.y1 - r.y0 >= 2 * MIN_TILE_EDGE:
                decided[r] = ("split", None)
                nxt.extend((c, lev + 1) for c in _children(r))
            else:
                decided[r] = ("high", i)
                leaves.append(i)
        # result objects only for the leaves that keep one (batched canonicalisation)
        if leaves:
            res = F._results_from_rows(rows[np.array(leaves)], config.formulation)
            by_row = dict(zip(leaves, res))
            for r, _ in level_rects:
                kind, payload = decided[r]
                if kind in ("fit", "high") and isinstance(payload, (int, np.integer)):
                    decided[r] = (kind, by_row[int(payload)])
        level_rects = nxt
    # leaves in the reference's LIFO order (pending.pop() / pending.extend(children))
    tiles = []
    pending = [(r, 0) for r in _grid(W, H, config.initial_tile)]
    while pending:
        r, lev = pending.pop()
        kind, res = decided[r]
        if kind == "split":
            pending.extend((c, lev + 1) for c in _children(r))
        elif kind == "fit":
            tiles.append(Tile(r, TileStatus.FITTED, lev, res))
        elif kind == "high":
            tiles.append(Tile(r, TileStatus.HIGH_ERROR, lev, res))
        else:
            tiles.append(Tile(r, TileStatus.TOO_INVALID, lev))
    warnings = []
    fitted = [t for t in tiles if t.status is TileStatus.FITTED]
    if fitted:
        feats = _features(fitted, config.d_scale)
        k = config.k
        if k > len(fitted):
            warnings.append(f"k={k} exceeds {len(fitted)} fitted tiles; clamped")
            k = len(fitted)
        labels, centroids = kmeans(feats, k, seed=config.seed)
        for t, lab in zip(fitted, labels):
            t.cluster = int(lab)
    else:
        centroids = np.zeros((0, 4))
        warnings.append("no tiles were fitted")
    host = np.full((H, W), UNLABELED, dtype=np.int16)
    for t in fitted:
        host[t.rect.y0:t.rect.y1, t.rect.x0:t.rect.x1] = t.cluster
    lab = torch.from_numpy(host).to(d.device)  # one upload: the label lattice lives with the depth
    return Segmentation(tiles, lab, centroids, len(fitted),
                        sum(t.status is TileStatus.TOO_INVALID for t in tiles),
                        sum(t.status is TileStatus.HIGH_ERROR for t in tiles), warnings)
