"""Pinhole-camera helpers of the reference (``camera.py``) around the device tan tables.

``back_project``, ``back_project_image``, ``project_point``, ``noise_sigma``,
``load_intrinsics``, ``Point3`` and the noise constants follow ``camera.py:29-267``.  They are
small geometry utilities on either side of the fitting path; ``back_project_image`` keeps a
device tensor on the device.
"""

from __future__ import annotations

from pathlib import Path
from typing import NamedTuple

import numpy as np
import torch

from .pixels import CameraIntrinsics, TanAngleMaps
from .synth import DEPTH_NOISE_COEFFICIENT, NoiseModel

DISPARITY_SLOPE_M_OVER_FB = -2.85e-3
MM_PER_METER = 1000.0

__all__ = ["DEPTH_NOISE_COEFFICIENT", "DISPARITY_SLOPE_M_OVER_FB", "MM_PER_METER", "Point3", "back_project",
           "back_project_image", "project_point", "noise_sigma", "load_intrinsics"]


class Point3(NamedTuple):
    """A 3D point in the camera frame (metres, Z along the optical axis)."""

    x: float
    y: float
    z: float


def _check_pixel(maps: TanAngleMaps, x: int, y: int) -> None:
    if not (0 <= x < maps.width and 0 <= y < maps.height):
        raise ValueError(f"pixel ({x}, {y}) outside {maps.width}x{maps.height} image")


def back_project(pixel, depth: float, maps: TanAngleMaps) -> Point3:
    """(Z tan_x, Z tan_y, Z) of one pixel (camera.py:141-155)."""
    x, y = pixel
    _check_pixel(maps, x, y)
    if depth <= 0:
        raise ValueError(f"depth must be positive, got {depth}")
    return Point3(depth * float(maps.tan_x[y, x]), depth * float(maps.tan_y[y, x]), float(depth))


def back_project_image(depth, maps: TanAngleMaps):
    """(H, W, 3) camera-frame coordinates of a depth lattice (camera.py:158-166).  A CUDA tensor
    stays on its device (one fused elementwise pass); numpy input returns numpy."""
    if isinstance(depth, torch.Tensor):
        d = depth.to(torch.float64)
        tx = torch.from_numpy(np.ascontiguousarray(maps.tan_x)).to(d.device)
        ty = torch.from_numpy(np.ascontiguousarray(maps.tan_y)).to(d.device)
        return torch.stack((d * tx, d * ty, d), dim=-1)
    d = np.asarray(depth, dtype=np.float64)
    return np.stack((d * maps.tan_x, d * maps.tan_y, d), axis=-1)


def project_point(point: Point3, intrinsics: CameraIntrinsics, distortion_pixel=None):
    """Forward pinhole projection x = fx X / Z + cx - delta_x (camera.py:169-195)."""
    if point.z <= 0:
        raise ValueError(f"cannot project point with Z={point.z}")
    if distortion_pixel is None:
        dx = dy = 0.0
        if np.any(intrinsics.delta_x) or np.any(intrinsics.delta_y):
            raise ValueError("distorted camera: pass distortion_pixel to project_point")
    else:
        px, py = distortion_pixel
        dx = float(intrinsics.delta_x[py, px])
        dy = float(intrinsics.delta_y[py, px])
    return (intrinsics.fx * point.x / point.z + intrinsics.cx - dx,
            intrinsics.fy * point.y / point.z + intrinsics.cy - dy)


def noise_sigma(depth: float, pixel, maps: TanAngleMaps, model: NoiseModel):
    """Per-axis measurement sigmas (tan_x sz, tan_y sz, sz) at one pixel (camera.py:198-214)."""
    x, y = pixel
    _check_pixel(maps, x, y)
    if depth <= 0:
        raise ValueError(f"depth must be positive, got {depth}")
    sz = float(model.sigma_z(depth))
    return (float(maps.tan_x[y, x]) * sz, float(maps.tan_y[y, x]) * sz, sz)


def load_intrinsics(path) -> CameraIntrinsics:
    """key=value intrinsics file, optional ``distortion=<raw float64 delta_x then delta_y>``
    (camera.py:217-267)."""
    path = Path(path)
    values = {}
    for lineno, raw in enumerate(path.read_text().splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ValueError(f"{path}:{lineno}: expected key=value, got {raw!r}")
        key, _, value = line.partition("=")
        values[key.strip()] = value.strip()
    missing = [k for k in ("fx", "fy", "cx", "cy", "width", "height") if k not in values]
    if missing:
        raise ValueError(f"{path}: missing intrinsics keys: {', '.join(missing)}")
    width, height = int(values["width"]), int(values["height"])
    delta_x = delta_y = None
    if "distortion" in values:
        dist = Path(values["distortion"])
        if not dist.is_absolute():
            dist = path.parent / dist
        flat = np.fromfile(dist, dtype="<f8")
        if flat.size != 2 * width * height:
            raise ValueError(f"{dist}: expected {2 * width * height} float64 values, got {flat.size}")
        delta_x = flat[:width * height].reshape(height, width)
        delta_y = flat[width * height:].reshape(height, width)
    return CameraIntrinsics(fx=float(values["fx"]), fy=float(values["fy"]), cx=float(values["cx"]),
                            cy=float(values["cy"]), width=width, height=height, delta_x=delta_x, delta_y=delta_y)
