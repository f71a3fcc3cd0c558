"""Randomised parity sweep (seeded, deterministic): frame sizes from 1 pixel to a few tiles
with ragged edges, every odd window up to 25, the three depth element types, optional
masks, holes, and hostile values (NaN, +/-inf, negative depths, 1 mm depths among metres)
-- all four formulations against the oracle, plus the batched-rect kernel on random rects.
(Subnormal depths are valid input but not a parity case: 1/Z ~ 1e39 puts the disparity
scatter's entries 80 orders of magnitude apart, where the reference's fp64 Jacobi and any
other solver return rounding noise.)"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2103_06644_b200 as rf
from oracle.compare import compare, normal_angles
from tests.helpers import Cam, gpu_flat, oracle_frame

pytestmark = pytest.mark.gpu


def _frame(rng, W, H, dtype):
    """Planes + noise + holes + hostile values, stored in the requested element type."""
    fx = float(rng.uniform(0.5, 2.0) * max(W, H))
    cx, cy = (W - 1) / 2.0, (H - 1) / 2.0
    tx = (np.arange(W) - cx) / fx
    ty = (np.arange(H) - cy) / fx
    n = rng.standard_normal(3)
    n[2] = -abs(n[2]) - 0.5
    d0 = rng.uniform(0.4, 6.0)
    denom = n[0] * tx[None, :] + n[1] * ty[:, None] + n[2]
    z = -d0 * n[2] / denom
    z = np.where((z > 0.05) & (z < 30), z, 0.0)
    z = z + 1.425e-3 * z * z * rng.standard_normal(z.shape)
    z[rng.random(z.shape) < rng.uniform(0.0, 0.3)] = 0.0
    if dtype == "u16":
        mm = np.clip(np.round(z * 1000.0), 0, 65535).astype(np.uint16)
        return mm, Cam(fx, fx, cx, cy, W, H)
    hostile = rng.random(z.shape)
    z = np.where(hostile < 0.01, np.nan, z)
    z = np.where((hostile >= 0.01) & (hostile < 0.015), np.inf, z)
    z = np.where((hostile >= 0.015) & (hostile < 0.02), -z - 1.0, z)
    z = np.where((hostile >= 0.02) & (hostile < 0.022), 1e-3, z)
    return (z.astype(np.float32) if dtype == "f32" else z.astype(np.float64)), Cam(fx, fx, cx, cy, W, H)


CASES = []
_rng = np.random.default_rng(2103)
for i in range(48):
    W = int(_rng.choice([1, 2, 5, 17, 63, 64, 65, 100, 130]))
    H = int(_rng.choice([1, 3, 15, 16, 17, 40, 71]))
    window = int(_rng.choice([1, 3, 5, 7, 9, 11, 13, 15, 17, 25]))
    CASES.append((i, W, H, window, ["f32", "u16", "f64"][i % 3], bool(i % 4 == 1)))


@pytest.mark.parametrize("case,W,H,window,dtype,use_mask", CASES)
def test_random_frames(case, W, H, window, dtype, use_mask):
    rng = np.random.default_rng(1000 + case)
    z, cam = _frame(rng, W, H, dtype)
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(cam.fx, cam.fy, cam.cx, cam.cy, W, H))
    depth = torch.from_numpy(z).cuda()
    mask = torch.from_numpy(rng.random((H, W)) > 0.15).cuda() if use_mask else None
    out = rf.fit_pixels(depth, maps, window, rf.FORMULATIONS, mask=mask)
    torch.cuda.synchronize()
    for form in rf.FORMULATIONS:
        ref = oracle_frame(torch.from_numpy(z), cam, window, form, mask=None if mask is None else mask.cpu())
        m = compare(gpu_flat(out[form]), ref, explicit_fit=form.startswith("explicit"))
        assert m["ok"], (case, form, {k: m[k] for k in ("status_mismatch", "max_normal_rad", "max_residual_rel",
                                                         "max_curvature_rel", "nonfit_is_nan")})


@pytest.mark.parametrize("case", range(6))
def test_random_rects(case):
    rng = np.random.default_rng(500 + case)
    W, H = int(rng.integers(8, 90)), int(rng.integers(8, 60))
    dtype = ["f32", "u16", "f64"][case % 3]
    z, cam = _frame(rng, W, H, dtype)
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(cam.fx, cam.fy, cam.cx, cam.cy, W, H))
    rects = []
    for _ in range(40):
        x0, y0 = int(rng.integers(0, W)), int(rng.integers(0, H))
        rects.append((x0, y0, int(rng.integers(x0, W + 1)), int(rng.integers(y0, H + 1))))
    depth = torch.from_numpy(z).cuda()
    from oracle import oracle as O
    values, valid = (O.depth_from_millimeters(z) if dtype == "u16" else O.depth_from_meters(z))
    tx, ty = O.tan_maps(cam.fx, cam.fy, cam.cx, cam.cy, W, H)
    for form, code in (("implicit-standard", O.STANDARD), ("implicit-rgbd", O.RGBD),
                       ("explicit-standard", O.EXPLICIT_STANDARD), ("explicit-rgbd", O.EXPLICIT_RGBD)):
        got = rf.fit_rects(depth, maps, rects, form)
        ref = O.fit_rects(values, valid, tx, ty, rects, code)
        np.testing.assert_array_equal(got["n_points"], ref["n"])
        np.testing.assert_array_equal(got["status"] & 2, ref["status"] & 2)
        ok = ((ref["status"] & 2) != 0) & ((ref["status"] & 4) == 0) & ((got["status"] & 4) == 0)
        if ok.any():
            assert normal_angles(got["coef"][ok, :3], ref["coef"][ok, :3]).max() <= 1e-4, (case, form)


def _adversarial(kind, W=96, H=48):
    """Hand-made hard windows: stripes of validity (collinear samples), checkerboards, depth
    steps through window centres, noiseless oblique planes (lambda ~ 0), near-grazing planes."""
    fx = 80.0
    cx, cy = (W - 1) / 2.0, (H - 1) / 2.0
    tx = (np.arange(W) - cx) / fx
    ty = (np.arange(H) - cy) / fx
    TX, TY = np.meshgrid(tx, ty)
    if kind == "stripes":
        z = 2.0 + 0.3 * TX - 0.2 * TY
        z[np.arange(H) % 3 != 0, :] = 0.0           # only every third row valid
    elif kind == "checker":
        z = 1.5 - 0.4 * TY + 1e-3 * np.sin(7 * TX)
        z[(np.arange(H)[:, None] + np.arange(W)[None, :]) % 2 == 1] = 0.0
    elif kind == "steps":
        z = np.where(TX < 0, 1.0, 3.0) + np.where(TY < 0, 0.0, 0.5)
    elif kind == "oblique":
        n = np.array([0.6, -0.3, -0.74])            # noiseless plane n.X + 2 = 0
        z = -2.0 / (n[0] * TX + n[1] * TY + n[2])
    else:  # grazing: plane nearly parallel to the viewing rays
        n = np.array([0.995, 0.0, -0.0999])
        z = -0.2 / (n[0] * TX + n[1] * TY + n[2])
        z = np.where((z > 0) & (z < 50), z, 0.0)
    return z.astype(np.float32), Cam(fx, fx, cx, cy, W, H)


@pytest.mark.parametrize("kind", ["stripes", "checker", "steps", "oblique", "grazing"])
@pytest.mark.parametrize("window", [3, 5, 9])
def test_adversarial_windows(kind, window):
    z, cam = _adversarial(kind)
    H, W = z.shape
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(cam.fx, cam.fy, cam.cx, cam.cy, W, H))
    out = rf.fit_pixels(torch.from_numpy(z).cuda(), maps, window, rf.FORMULATIONS)
    torch.cuda.synchronize()
    for form in rf.FORMULATIONS:
        ref = oracle_frame(torch.from_numpy(z), cam, window, form)
        m = compare(gpu_flat(out[form]), ref, explicit_fit=form.startswith("explicit"))
        assert m["ok"], (kind, window, form, {k: m[k] for k in ("status_mismatch", "max_normal_rad",
                                                                 "max_residual_rel", "max_curvature_rel")})


@pytest.mark.parametrize("window,dtype,use_mask,direct", [(3, "f32", False, False), (5, "u16", True, False),
                                                           (9, "f64", False, False), (15, "f32", True, False),
                                                           (31, "f32", False, False), (5, "f32", True, True),
                                                           (11, "u16", False, True)])
def test_distortion_lattices(window, dtype, use_mask, direct, monkeypatch):
    """Cameras with per-pixel distortion offsets: the tiled lattice kernel (and the direct
    per-pixel fallback) against the oracle with the same lattices."""
    if direct:
        monkeypatch.setenv("RF_LATTICE_DIRECT", "1")
    rng = np.random.default_rng(window * 7 + len(dtype))
    W, H = 100, 70
    z, cam = _frame(rng, W, H, dtype)
    dx, dy = rng.uniform(-0.45, 0.45, (H, W)), rng.uniform(-0.45, 0.45, (H, W))
    cam = Cam(cam.fx, cam.fy, cam.cx, cam.cy, W, H, dx, dy)
    maps = rf.compute_tan_maps(cam.intrinsics())
    mask = torch.from_numpy(rng.random((H, W)) > 0.1).cuda() if use_mask else None
    out = rf.fit_pixels(torch.from_numpy(z).cuda(), maps, window, rf.FORMULATIONS, mask=mask)
    torch.cuda.synchronize()
    for form in rf.FORMULATIONS:
        ref = oracle_frame(torch.from_numpy(z), cam, window, form, mask=None if mask is None else mask.cpu())
        m = compare(gpu_flat(out[form]), ref, explicit_fit=form.startswith("explicit"))
        assert m["ok"], (window, dtype, form, {k: m[k] for k in ("status_mismatch", "max_normal_rad",
                                                                  "max_residual_rel", "max_curvature_rel")})


@pytest.mark.parametrize("seed", [9372, 9405])
def test_sweep_three_sample_explicit_windows(seed):
    """Frames of the long sweep (tests/diagnostics/stress_sweep.py, seeds 9000+) whose
    explicit-standard fits include 3-sample windows -- one 1 mm sample and two ~30 m samples
    at nearly collinear X-Y positions: an exact fit (residual 0) that the centred 2x2 solve
    used to return as 1e-3 m of cancellation."""
    rng = np.random.default_rng(seed)
    W, H = int(rng.integers(1, 150)), int(rng.integers(1, 90))
    window = int(rng.choice([1, 3, 5, 7, 9, 11, 13, 15, 17, 21, 25, 31]))
    dtype = ["f32", "u16", "f64"][int(rng.integers(3))]
    z, cam = _frame(rng, W, H, dtype)
    if rng.random() < 0.2:
        cam = Cam(cam.fx, cam.fy, cam.cx, cam.cy, W, H, rng.uniform(-0.4, 0.4, (H, W)),
                  rng.uniform(-0.4, 0.4, (H, W)))
    mask = torch.from_numpy(rng.random((H, W)) > 0.2).cuda() if rng.random() < 0.3 else None
    maps = rf.compute_tan_maps(cam.intrinsics())
    out = rf.fit_pixels(torch.from_numpy(z).cuda(), maps, window, rf.FORMULATIONS, mask=mask)
    torch.cuda.synchronize()
    for form in rf.FORMULATIONS:
        ref = oracle_frame(torch.from_numpy(z), cam, window, form, mask=None if mask is None else mask.cpu())
        m = compare(gpu_flat(out[form]), ref, explicit_fit=form.startswith("explicit"))
        assert m["ok"], (seed, form, m["max_residual_rel"])


@pytest.mark.parametrize("kind,window", [("stripes", 3), ("stripes", 5), ("checker", 3)])
def test_degenerate_explicit_windows(kind, window):
    """Rank-deficient explicit systems (every valid sample of a window in one row: collinear in
    tan_y): the reference's Cholesky fails and _pinv_solve returns the minimum-norm plane and
    its true residual (fitting.py:313-322, 584-597).  The per-pixel kernel queues such windows
    for the slow pass, which solves them that way; degenerate pixels are compared too."""
    z, cam = _adversarial(kind)
    H, W = z.shape
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(cam.fx, cam.fy, cam.cx, cam.cy, W, H))
    out = rf.fit_pixels(torch.from_numpy(z).cuda(), maps, window, rf.FORMULATIONS)
    torch.cuda.synchronize()
    for form in (rf.EXPLICIT_STANDARD, rf.EXPLICIT_RGBD):
        ref = oracle_frame(torch.from_numpy(z), cam, window, form)
        got = gpu_flat(out[form])
        rdeg = (ref["status"] & 6) == 6
        if kind == "stripes" and window == 3:
            assert rdeg.sum() > 100  # the case exercises the minimum-norm path
        assert np.array_equal((got["status"] & 6) == 6, rdeg), form
        m = compare(got, ref, explicit_fit=True, include_degenerate=True)
        assert m["ok"], (kind, window, form, {k: m[k] for k in ("compared", "status_mismatch", "max_normal_rad",
                                                                 "max_residual_rel", "max_curvature_rel")})
