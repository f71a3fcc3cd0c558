"""Test helpers: run the oracle and the sm_100a path on the same stored bits."""

from __future__ import annotations

import numpy as np
import torch

from oracle import oracle as O
from oracle.compare import compare

FORM_CODE = {"implicit-standard": O.STANDARD, "implicit-rgbd": O.RGBD,
             "explicit-standard": O.EXPLICIT_STANDARD, "explicit-rgbd": O.EXPLICIT_RGBD}


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
    tx, ty = O.tan_maps(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height,
                        getattr(cam, "delta_x", None), getattr(cam, "delta_y", None))
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
    return compare(got, ref, explicit_fit=formulation.startswith("explicit")), got, ref


# ------------------------------------------------------------ golden fixtures
GOLDEN_DIR = __import__("pathlib").Path(__file__).resolve().parent / "golden"
GOLDEN_CASES = ("planes_f32_w3", "planes_f32_w5", "planes_f32_mask_w5", "planes_u16_w5",
                "frontal_z3_w5", "half_invalid_w3", "near_far_w7", "distorted_f32_w5", "planes_u16_mask_w9",
                "near_far_w15", "near_far_w31", "planes_f32_w11")


class Cam:
    def __init__(self, fx, fy, cx, cy, width, height, delta_x=None, delta_y=None):
        self.fx, self.fy, self.cx, self.cy, self.width, self.height = fx, fy, cx, cy, width, height
        self.delta_x, self.delta_y = delta_x, delta_y

    def intrinsics(self):
        """The package's CameraIntrinsics (distortion lattices included)."""
        import paper_2103_06644_b200 as rf
        return rf.CameraIntrinsics(self.fx, self.fy, self.cx, self.cy, self.width, self.height,
                                   self.delta_x, self.delta_y)


def load_golden(name: str) -> dict:
    """Golden case written by tests/golden/make_golden.py (reference outputs, per pixel)."""
    z = np.load(GOLDEN_DIR / f"{name}.npz")
    depth = z["depth"]
    H, W = depth.shape
    cam = Cam(float(z["fx"]), float(z["fy"]), float(z["cx"]), float(z["cy"]), W, H,
              z["delta_x"] if "delta_x" in z.files else None, z["delta_y"] if "delta_y" in z.files else None)
    g = {"depth": depth, "cam": cam, "window": int(z["window"]), "dtype": str(z["dtype"]),
         "valid": z["valid"].astype(bool) if "valid" in z.files else None}
    for key, form in (("rgbd", "implicit-rgbd"), ("std", "implicit-standard"),
                      ("xrgbd", "explicit-rgbd"), ("xstd", "explicit-standard")):
        coef = z[f"{key}_coef"]
        nrm = np.linalg.norm(coef[:, :3], axis=1)
        with np.errstate(invalid="ignore", divide="ignore"):
            normal = coef[:, :3] / nrm[:, None]
            offset = coef[:, 3] / nrm
        g[form] = {"normal": normal, "offset": offset, "residual": z[f"{key}_rms"],
                   "curvature": z[f"{key}_curv"], "status": z[f"{key}_status"],
                   "scale": z[f"{key}_scale"], "coef": coef, "lam": z[f"{key}_lam"],
                   "n": z[f"{key}_n"]}
    return g


def golden_mask(g: dict):
    """Explicit validity mask of a golden case (None when derived from the depth values)."""
    d = g["depth"]
    derived = (d > 0) if d.dtype == np.uint16 else (np.isfinite(d) & (d > 0))
    if g["valid"] is None or np.array_equal(g["valid"], derived):
        return None
    return g["valid"]


def load_golden_rects(name: str = "rects_planes_f32") -> dict:
    """Reference fit_rect results on random rects (tests/golden/make_golden.py:run_rects)."""
    z = np.load(GOLDEN_DIR / f"{name}.npz")
    depth = z["depth"]
    H, W = depth.shape
    g = {"depth": depth, "cam": Cam(float(z["fx"]), float(z["fy"]), float(z["cx"]), float(z["cy"]), W, H),
         "rects": z["rects"], "dtype": str(z["dtype"])}
    for key, form in (("rgbd", "implicit-rgbd"), ("std", "implicit-standard"),
                      ("xrgbd", "explicit-rgbd"), ("xstd", "explicit-standard")):
        g[form] = {k: z[f"{key}_{k}"] for k in ("coef", "xcoef", "rms", "lam", "curv", "n", "status", "scale")}
    return g
