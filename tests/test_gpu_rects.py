"""Batched rect fits on the GPU (rf_fit_rects) and the reference-signature
fit_rect(..., backend="b200") against the reference's own fit_rect results."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2103_06644_b200 as rf
from oracle.compare import normal_angles
from tests.helpers import load_golden_rects

pytestmark = pytest.mark.gpu


def _maps(cam):
    return rf.compute_tan_maps(rf.CameraIntrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height))


@pytest.mark.parametrize("form", list(rf.FORMULATIONS))
def test_rects_match_reference(form):
    g = load_golden_rects()
    maps = _maps(g["cam"])
    depth = torch.from_numpy(g["depth"]).cuda()
    got = rf.fit_rects(depth, maps, g["rects"], form)
    ref = g[form]
    np.testing.assert_array_equal(got["n_points"], ref["n"])
    np.testing.assert_array_equal(got["status"] & 3, ref["status"] & 3)
    ok = ((ref["status"] & 2) != 0) & ((ref["status"] & 4) == 0)
    ang = normal_angles(got["coef"][ok, :3], ref["coef"][ok, :3])
    assert ang.max() <= 1e-5, ang.max()
    assert np.abs(got["coef"][ok] - ref["coef"][ok]).max() <= 1e-5
    floor = np.sqrt((1e-10 if form.startswith("explicit") else 1e-11) * ref["scale"][ok])
    res_err = np.abs(got["rms"][ok] - ref["rms"][ok]) / (1e-4 * np.abs(ref["rms"][ok]) + floor)
    assert res_err.max() <= 1.0
    cur_err = np.abs(got["curvature"][ok] - ref["curv"][ok]) / (1e-4 * np.abs(ref["curv"][ok]) + 1e-8)
    assert cur_err.max() <= 1.0
    if form.startswith("explicit"):
        np.testing.assert_allclose(got["explicit_coef"][ok], ref["xcoef"][ok], rtol=1e-6, atol=1e-9)


def test_fit_rect_dropin_semantics():
    g = load_golden_rects()
    maps = _maps(g["cam"])
    depth = torch.from_numpy(g["depth"]).cuda()
    res = rf.fit_rect(depth, maps, rf.Rect(0, 0, g["cam"].width, g["cam"].height), rf.IMPLICIT_RGBD)
    assert isinstance(res, rf.FitResult) and isinstance(res.plane, rf.ImplicitPlane)
    ref = g[rf.IMPLICIT_RGBD]
    assert res.n_points == ref["n"][0]
    assert rf.normal_angle(res.plane, rf.ImplicitPlane(ref["coef"][0])) <= 1e-6
    ex = rf.fit_rect(depth, maps, rf.Rect(0, 0, 10, 10), rf.EXPLICIT_STANDARD)
    assert isinstance(ex.plane, rf.ExplicitPlane) and ex.eigenvalue is None
    with pytest.raises(rf.InsufficientSamplesError):
        rf.fit_rect(depth, maps, rf.Rect(0, 0, 1, 1), rf.IMPLICIT_STANDARD)
    with pytest.raises(ValueError):
        rf.fit_rect(depth, maps, rf.Rect(0, 0, g["cam"].width + 1, 4), rf.IMPLICIT_STANDARD)
    with pytest.raises(ValueError):
        rf.fit_rect(depth, maps, rf.Rect(0, 0, 4, 4), rf.IMPLICIT_STANDARD, backend="integral")


def test_rects_out_of_bounds_and_frames():
    g = load_golden_rects()
    maps = _maps(g["cam"])
    d = torch.from_numpy(g["depth"]).cuda()
    batch = torch.stack([d, d])
    out = rf.fit_rects(batch, maps, [(0, 0, 8, 8), (0, 0, 8, 8), (-1, 0, 4, 4)], rf.IMPLICIT_RGBD, frames=[0, 1, 0])
    assert out["status"][2] & rf.fitting.RECT_OUT_OF_BOUNDS
    np.testing.assert_array_equal(out["coef"][0], out["coef"][1])


@pytest.mark.parametrize("window", [3, 7, 15])
def test_pixel_and_rect_kernels_agree(window):
    """Two independent device paths, one semantics: the per-pixel tile kernel at pixel (x, y)
    and the rect kernel on that pixel's clipped window (A9) give the same fit."""
    from paper_2103_06644_b200 import scenes
    cfg = scenes.small_config("C2", 128, 80)
    depth = scenes.render_frame(cfg, 9).cuda()
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height))
    out = rf.fit_pixels(depth, maps, window, rf.FORMULATIONS)
    rng = np.random.default_rng(window)
    H, W = depth.shape
    r = window // 2
    pix = rng.choice(H * W, 300, replace=False)
    rects = [(max(p % W - r, 0), max(p // W - r, 0), min(p % W + r + 1, W), min(p // W + r + 1, H)) for p in pix]
    for form in rf.FORMULATIONS:
        rows = rf.fit_rects(depth, maps, rects, form)
        st = out[form].status.reshape(-1)[torch.from_numpy(pix).cuda()].cpu().numpy()
        center_valid = (st & 1) != 0
        # the rect fit ignores the centre pixel's own validity (a rect has no centre rule)
        np.testing.assert_array_equal((st & 2) != 0, center_valid & ((rows["status"] & 2) != 0))
        ok = ((st & 6) == 2) & ((rows["status"] & 4) == 0)
        gn = out[form].normal.reshape(-1, 3)[torch.from_numpy(pix).cuda()].cpu().numpy()[ok]
        rn = rows["coef"][ok, :3] / np.linalg.norm(rows["coef"][ok, :3], axis=1, keepdims=True)
        assert normal_angles(gn, rn).max() <= 1e-5, form
        gr = out[form].residual.reshape(-1)[torch.from_numpy(pix).cuda()].cpu().numpy()[ok]
        np.testing.assert_allclose(gr, rows["rms"][ok], rtol=1e-4, atol=1e-9)
