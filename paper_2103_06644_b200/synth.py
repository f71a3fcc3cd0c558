"""The reference's virtual depth sensor with the nearest-hit render on the device
(drop-in for ``rangefit.synth``).

``GroundTruthPlane``, ``SyntheticScene``, ``NoiseModel``, ``render_scene``, ``parse_scene``,
``load_scene``, ``write_depth``, ``read_depth`` and ``INVALID_LABEL`` follow
``synth.py:24-246`` / ``camera.py:99-114``.  ``render_scene`` runs ``rf_render_planes``
(``csrc/rf_render.cu``): every plane's ray intersection, nearest positive hit, quadratic
depth noise and dropout, per pixel on the device.

Random draws: ``rng="reference"`` (default) draws them exactly as the reference does -- one
``numpy.random.default_rng`` per image row from ``SeedSequence(seed).spawn(H)``, normals
then uniforms -- on the host, so the rendered frame is the reference's bit for bit;
``rng="device"`` draws them on the device with a seeded ``torch.Generator`` (same
distributions, not the reference's stream) for large synthetic batches.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from . import imageio
from .depth import DepthImage
from .pixels import TanAngleMaps

INVALID_LABEL = 255
DEPTH_NOISE_COEFFICIENT = 1.425e-3  # camera.py:29


@dataclass(frozen=True)
class NoiseModel:
    """sigma_Z = slope_coefficient * Z^2 (camera.py:99-114)."""

    slope_coefficient: float = DEPTH_NOISE_COEFFICIENT

    def __post_init__(self) -> None:
        if self.slope_coefficient <= 0:
            raise ValueError(f"slope_coefficient must be positive, got {self.slope_coefficient}")

    def sigma_z(self, depth):
        return self.slope_coefficient * depth * depth


@dataclass(frozen=True)
class GroundTruthPlane:
    """a X + b Y + c Z + d = 0 with a unit normal; optional half-open mask rect (synth.py:27-55)."""

    coefficients: np.ndarray
    mask_rect: tuple | None = None

    def __post_init__(self) -> None:
        coef = np.asarray(self.coefficients, dtype=np.float64)
        if coef.shape != (4,):
            raise ValueError(f"plane needs 4 coefficients, got shape {coef.shape}")
        norm = float(np.linalg.norm(coef[:3]))
        if norm == 0:
            raise ValueError("plane normal must be nonzero")
        object.__setattr__(self, "coefficients", coef / norm)

    @property
    def normal(self) -> np.ndarray:
        return self.coefficients[:3]

    @property
    def offset(self) -> float:
        return float(self.coefficients[3])


@dataclass(frozen=True)
class SyntheticScene:
    """An ordered set of ground-truth planes; nearest intersection wins (synth.py:57-66)."""

    planes: tuple

    def __post_init__(self) -> None:
        if not self.planes:
            raise ValueError("scene must contain at least one plane")
        object.__setattr__(self, "planes", tuple(self.planes))


def ray_for_pixel(maps: TanAngleMaps, pixel) -> np.ndarray:
    """Unnormalised viewing ray (tan_x, tan_y, 1) of one pixel (synth.py:117-122)."""
    x, y = pixel
    if not (0 <= x < maps.width and 0 <= y < maps.height):
        raise ValueError(f"pixel ({x}, {y}) outside {maps.width}x{maps.height} image")
    return np.array([maps.tan_x[y, x], maps.tan_y[y, x], 1.0])


def intersect_plane(ray: np.ndarray, plane: GroundTruthPlane):
    """Depth of a ray-plane intersection, None if behind or parallel (synth.py:125-134)."""
    a, b, c, d = plane.coefficients
    denom = a * ray[0] + b * ray[1] + c * ray[2]
    if denom == 0.0:
        return None
    z = -d / denom
    if z <= 0 or not np.isfinite(z):
        return None
    return float(z)


def _plane_rects(scene: SyntheticScene, width: int, height: int) -> np.ndarray:
    """Mask rects as the reference's numpy slices select them (masked[y0:y1, x0:x1])."""
    out = np.empty((len(scene.planes), 4), np.int32)
    for i, p in enumerate(scene.planes):
        if p.mask_rect is None:
            out[i] = (0, 0, width, height)
            continue
        x0, y0, x1, y1 = p.mask_rect
        xs, ys = slice(x0, x1).indices(width), slice(y0, y1).indices(height)
        out[i] = (xs[0], ys[0], max(xs[0], xs[1]), max(ys[0], ys[1]))
    return out


def _reference_draws(height: int, width: int, seed: int, noise: bool, dropout: float):
    """The reference's random stream: one generator per row, normals then uniforms."""
    eps = np.empty((height, width)) if noise else None
    uni = np.empty((height, width)) if dropout > 0.0 else None
    for y, ss in enumerate(np.random.SeedSequence(seed).spawn(height)):
        rng = np.random.default_rng(ss)
        if noise:
            eps[y] = rng.standard_normal(width)
        if dropout > 0.0:
            uni[y] = rng.random(width)
    return eps, uni


def render_depth(scene: SyntheticScene, maps: TanAngleMaps, noise: NoiseModel | None = None, seed: int = 0,
                 dropout: float = 0.0, rng: str = "reference"):
    """Render on the device -> (depth float64 [H, W], valid uint8, labels uint8), device tensors."""
    if not (0.0 <= dropout < 1.0):
        raise ValueError(f"dropout must be in [0, 1), got {dropout}")
    if rng not in ("reference", "device"):
        raise ValueError(f"rng must be 'reference' or 'device', got {rng!r}")
    H, W = maps.height, maps.width
    dev = torch.device("cuda", maps.device)
    planes = torch.from_numpy(np.stack([p.coefficients for p in scene.planes])).to(dev)
    rects = torch.from_numpy(_plane_rects(scene, W, H)).to(dev)
    eps = uni = None
    if noise is not None or dropout > 0.0:
        if rng == "reference":
            e, u = _reference_draws(H, W, seed, noise is not None, dropout)
            eps = None if e is None else torch.from_numpy(e).to(dev)
            uni = None if u is None else torch.from_numpy(u).to(dev)
        else:
            g = torch.Generator(device=dev)
            g.manual_seed(seed)
            if noise is not None:
                eps = torch.randn((H, W), generator=g, device=dev, dtype=torch.float64)
            if dropout > 0.0:
                uni = torch.rand((H, W), generator=g, device=dev, dtype=torch.float64)
    depth = torch.empty((H, W), dtype=torch.float64, device=dev)
    valid = torch.empty((H, W), dtype=torch.uint8, device=dev)
    labels = torch.empty((H, W), dtype=torch.uint8, device=dev)
    st = N.load().rf_render_planes(maps.handle, planes.data_ptr(), rects.data_ptr(), len(scene.planes),
                                   eps.data_ptr() if eps is not None else None,
                                   uni.data_ptr() if uni is not None else None,
                                   float(noise.slope_coefficient) if noise is not None else 0.0, float(dropout),
                                   depth.data_ptr(), valid.data_ptr(), labels.data_ptr(),
                                   ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    N.check(st, "render_scene")
    return depth, valid, labels


def render_scene(scene: SyntheticScene, maps: TanAngleMaps, noise: NoiseModel | None = None, seed: int = 0,
                 dropout: float = 0.0, rng: str = "reference"):
    """Reference signature and return types (synth.py:152-194): (DepthImage, labels uint8)."""
    depth, valid, labels = render_depth(scene, maps, noise, seed, dropout, rng)
    return (DepthImage(values=depth.cpu().numpy(), valid=valid.cpu().numpy().astype(bool)),
            labels.cpu().numpy())


def parse_scene(text: str) -> SyntheticScene:
    """One plane per line, ``a b c d [x0 y0 x1 y1]``; '#' comments (synth.py:197-217)."""
    planes = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        parts = line.split()
        if len(parts) not in (4, 8):
            raise ValueError(f"scene line {lineno}: expected 'a b c d' or 'a b c d x0 y0 x1 y1', got {raw!r}")
        mask = tuple(int(v) for v in parts[4:]) if len(parts) == 8 else None
        planes.append(GroundTruthPlane(coefficients=np.array([float(v) for v in parts[:4]]), mask_rect=mask))
    if not planes:
        raise ValueError("scene file holds no planes")
    return SyntheticScene(planes=tuple(planes))


def load_scene(path) -> SyntheticScene:
    return parse_scene(Path(path).read_text())


def write_depth(path, depth: DepthImage) -> None:
    """``.pgm`` -> millimetre PGM (invalid = 0), else RF64 raw with NaN holes (synth.py:224-236)."""
    path = Path(path)
    if path.suffix.lower() == ".pgm":
        imageio.write_pgm16(path, depth.to_millimeters())
    else:
        imageio.write_raw_float(path, np.where(depth.valid, depth.values, np.nan))


def read_depth(path) -> DepthImage:
    path = Path(path)
    if path.suffix.lower() == ".pgm":
        return DepthImage.from_millimeters(imageio.read_pgm16(path))
    values = imageio.read_raw_float(path)
    return DepthImage(values=values, valid=np.isfinite(values) & (values > 0))
