"""Test helpers: run the oracle and the sm_100a path on the same stored bits."""

from __future__ import annotations

import numpy as np
import torch

from oracle import oracle as O
from oracle.compare import compare

FORM_CODE = {"implicit-standard": O.STANDARD, "implicit-rgbd": O.RGBD}


def oracle_frame(depth: torch.Tensor, cam, window: int, formulation: str, pixels=None, mask=None,
                 backend=O.NAIVE):
    """Oracle outputs for one [H, W] frame (CPU tensor or numpy), flat arrays."""
    d = depth.cpu().numpy() if isinstance(depth, torch.Tensor) else np.asarray(depth)
    if d.dtype == np.uint16:
        values, valid = O.depth_from_millimeters(d)
    else:
        values, valid = O.depth_from_meters(d)
    if mask is not None:
        m = mask.cpu().numpy() if isinstance(mask, torch.Tensor) else np.asarray(mask)
        valid = valid & m.astype(bool)
    tx, ty = O.tan_maps(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    return O.fit_pixels(values, valid, tx, ty, window, FORM_CODE[formulation], backend=backend,
                        pixels=pixels)


def gpu_flat(fits, frame: int = 0, pixels=None):
    """PixelFits of one frame -> dict of flat numpy arrays (optionally a pixel subset)."""
    out = {}
    for k in ("normal", "offset", "residual", "curvature", "status"):
        t = getattr(fits, k)
        t = t[frame] if t.dim() >= (4 if k == "normal" else 3) else t
        a = t.cpu().numpy()
        a = a.reshape(-1, 3) if k == "normal" else a.reshape(-1)
        out[k] = a if pixels is None else a[pixels]
    return out


def check_frame(depth_gpu, fits, cam, window, formulation, frame=0, pixels=None, mask=None):
    ref = oracle_frame(depth_gpu[frame] if depth_gpu.dim() == 3 else depth_gpu, cam, window,
                       formulation, pixels=pixels,
                       mask=None if mask is None else (mask[frame] if mask.dim() == 3 else mask))
    got = gpu_flat(fits, frame, pixels)
    return compare(got, ref), got, ref
