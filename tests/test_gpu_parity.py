"""Parity of the sm_100a per-pixel path against the oracle (restated reference)
on identical seeded inputs, through the C ABI (ctypes) -- the north_star bar:
masks bit-exact, normals <= 1e-4 rad, residual/curvature <= 1e-4 relative."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2103_06644_b200 as rf
from paper_2103_06644_b200 import scenes
from tests.helpers import check_frame

pytestmark = pytest.mark.gpu

FORMS = ("implicit-rgbd", "implicit-standard", "explicit-rgbd", "explicit-standard")


def _run(cfg, window, frames=1, seed_base=None, mask=None):
    depth = scenes.render_batch(cfg, frames=frames, device="cpu", seed_base=seed_base).cuda()
    cam = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height)
    maps = rf.compute_tan_maps(cam)
    out = rf.fit_pixels(depth, maps, window, FORMS, mask=mask)
    # the implicit-only launch (no explicit outputs) must give the same implicit results
    imp = rf.fit_pixels(depth, maps, window, FORMS[:2], mask=mask)
    torch.cuda.synchronize()
    for f in FORMS[:2]:
        assert torch.equal(out[f].status, imp[f].status)
        assert torch.equal(torch.nan_to_num(out[f].normal), torch.nan_to_num(imp[f].normal))
    torch.cuda.synchronize()
    return depth, cam, out


@pytest.mark.parametrize("window", [3, 5, 7])
def test_c1_like_full_frame(window):
    cfg = scenes.small_config("C1", 160, 120)
    depth, cam, out = _run(cfg, window)
    for form in FORMS:
        m, _, _ = check_frame(depth, out[form], cam, window, form)
        assert m["ok"], (form, m)


@pytest.mark.parametrize("name,window", [("C2", 11), ("C3", 9), ("C4", 15), ("C5", 31)])
def test_baseline_shapes_small(name, window):
    cfg = scenes.small_config(name, 192, 144)
    depth, cam, out = _run(cfg, window)
    for form in FORMS:
        m, _, _ = check_frame(depth, out[form], cam, window, form)
        assert m["ok"], (name, form, m)


def test_c1_full_size_all_pixels():
    """BASELINE config 1 exactly (640x480, 5x5, both variants), every pixel."""
    cfg = scenes.CONFIGS["C1"]
    depth, cam, out = _run(cfg, 5)
    for form in FORMS[:2]:
        m, _, _ = check_frame(depth, out[form], cam, 5, form)
        assert m["ok"], (form, m)
