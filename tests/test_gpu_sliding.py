"""Sliding-window sums under extreme dynamic range.  The tile kernels slide their column and
row window sums, so every sample that leaves a window leaves a rounding residue of about
eps x its own magnitude behind.  A window holding only millimetre depths right after metre
depths slid through its sums would inherit that residue (the reference's per-window direct
sums do not).  The kernels bound the residue per segment and queue such windows for the
tile's slow pass, which re-sums them directly (rf_fit.cu row pass and slow_pixel;
rf_lattice.cu refits them in place).

Compared: every pixel whose window holds ONE depth value class (all near or all far), so
the window itself is well conditioned and any disagreement is sliding residue.  Windows that
mix millimetres and metres are ill-conditioned for every summation order (the oracle, the
rect kernel and the tile kernels all differ there by more than the tolerances) and are not
a parity case.  All four formulations, separable and distortion-lattice cameras, the
running (r > 3) and centred (r <= 3) column passes, float32 and float64 depths."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2103_06644_b200 as rf
from oracle.compare import compare
from tests.helpers import Cam, gpu_flat, oracle_frame

pytestmark = pytest.mark.gpu

W, H = 64, 48


def _scene(far: float, near: float) -> np.ndarray:
    """Rows 0..15 and blocks at `far`; isolated `near` samples, a small `near` patch, and a
    far-to-near step inside one row segment."""
    z = np.zeros((H, W))
    z[:16, :] = far
    z[25:40, 44:50] = far
    for (y, x) in [(31, 30), (35, 25), (44, 40), (27, 36), (20, 20), (30, 3), (31, 6), (33, 60)]:
        z[y, x] = near
    z[31:34, 52:58] = near
    # a step inside one 4-pixel row segment (segments start at multiples of 4): far columns
    # that the row pass slides past, then near pixels whose windows hold only near samples
    z[40:47, 13:16] = far
    z[40:47, 16:21] = near
    return z


def _single_class(z: np.ndarray, window: int, far: float) -> np.ndarray:
    """Pixels whose clipped window has valid samples of only one class."""
    r = window // 2
    valid = z > 0
    is_far = valid & (z == np.asarray(far, z.dtype))
    pad = lambda a: np.pad(a.astype(np.int64), r)
    def box(a):
        c = pad(a).cumsum(0).cumsum(1)
        c = np.pad(c, ((1, 0), (1, 0)))
        k = 2 * r + 1
        return c[k:, k:] - c[:-k, k:] - c[k:, :-k] + c[:-k, :-k]
    nv, nf = box(valid), box(is_far)
    return ((nf == 0) | (nf == nv)).ravel()


def _subset(d: dict, sel: np.ndarray) -> dict:
    return {k: (np.asarray(v).reshape(-1, 3)[sel] if k == "normal" else np.asarray(v).ravel()[sel])
            for k, v in d.items()}


@pytest.mark.parametrize("distort", [False, True])
@pytest.mark.parametrize("window", [3, 5, 9, 15, 31])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("far,near", [(6.0, 1e-3), (1e-3, 6.0)])
def test_sliding_residue(distort, window, dtype, far, near):
    cam = Cam(60.0, 60.0, (W - 1) / 2, (H - 1) / 2, W, H)
    if distort:
        rng = np.random.default_rng(window)
        cam = Cam(cam.fx, cam.fy, cam.cx, cam.cy, W, H, rng.uniform(-.4, .4, (H, W)), rng.uniform(-.4, .4, (H, W)))
    maps = rf.compute_tan_maps(cam.intrinsics())
    z = _scene(far, near).astype(dtype)
    sel = _single_class(z, window, far)
    assert sel.sum() > 100
    out = rf.fit_pixels(torch.from_numpy(z).cuda(), maps, window, rf.FORMULATIONS)
    for form in rf.FORMULATIONS:
        ref = oracle_frame(torch.from_numpy(z), cam, window, form)
        m = compare(_subset(gpu_flat(out[form]), sel), _subset(ref, sel), explicit_fit=form.startswith("explicit"))
        assert m["ok"], f"{form} " + " ".join(f"{k}={m[k]:.3g}" for k in (
            "compared", "status_mismatch", "max_normal_rad", "max_residual_rel", "max_curvature_rel"))


@pytest.mark.parametrize("window", [5, 15])
def test_shared_tables_two_streams(window):
    """One TanAngleMaps shared by two streams fitting concurrently (different batches, the
    sliding-residue scene in both directions, rows of repeats so the launches overlap): the
    tables are immutable and the slow pass lives inside each launch, so both streams match
    the oracle (SURVEY.md 8b "tables shareable across streams")."""
    cam = Cam(60.0, 60.0, (W - 1) / 2, (H - 1) / 2, W, H)
    maps = rf.compute_tan_maps(cam.intrinsics())
    scenes_ = [_scene(6.0, 1e-3).astype(np.float32), _scene(1e-3, 6.0).astype(np.float32)]
    depths = [torch.from_numpy(np.stack([z] * 48)).cuda() for z in scenes_]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [{f: rf.PixelFits.empty(48, H, W, "cuda") for f in rf.FORMULATIONS} for _ in range(2)]
    torch.cuda.synchronize()
    for _ in range(4):
        for d, s, o in zip(depths, streams, outs):
            with torch.cuda.stream(s):
                rf.fit_pixels(d, maps, window, rf.FORMULATIONS, out=o, stream=s)
    torch.cuda.synchronize()
    for z, o, far in zip(scenes_, outs, (6.0, 1e-3)):
        sel = _single_class(z, window, far)
        for form in rf.FORMULATIONS:
            ref = oracle_frame(torch.from_numpy(z), cam, window, form)
            for frame in (0, 47):
                m = compare(_subset(gpu_flat(o[form], frame), sel), _subset(ref, sel),
                            explicit_fit=form.startswith("explicit"))
                assert m["ok"], (form, frame, m)
