"""sm_100a path vs the REFERENCE's own per-pixel outputs (golden fixtures made
by tests/golden/make_golden.py), through the C ABI: status bits 0/1 exact,
normals <= 1e-4 rad, residual/curvature <= 1e-4 relative (oracle/compare.py)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2103_06644_b200 as rf
from oracle.compare import compare
from tests.helpers import GOLDEN_CASES, golden_mask, gpu_flat, load_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_gpu_matches_reference_golden(case):
    g = load_golden(case)
    cam = g["cam"]
    maps = rf.compute_tan_maps(cam.intrinsics())
    depth = torch.from_numpy(g["depth"].astype(np.int32)).to(torch.uint16) if g["dtype"] == "u16" \
        else torch.from_numpy(g["depth"])
    mask = golden_mask(g)
    out = rf.fit_pixels(depth.cuda(), maps, g["window"], formulations=rf.FORMULATIONS,
                        mask=None if mask is None else torch.from_numpy(mask.astype(np.uint8)).cuda())
    torch.cuda.synchronize()
    for form in rf.FORMULATIONS:
        m = compare(gpu_flat(out[form], 0) if out[form].normal.dim() == 4 else gpu_flat_2d(out[form]), g[form],
                    explicit_fit=form.startswith("explicit"))
        assert m["ok"], (case, form, m)
        # against the reference's own outputs the degenerate bit matches too (it is a float
        # threshold, so the general parity contract only reports it)
        assert m["degenerate_mismatch"] == 0, (case, form, m["degenerate_mismatch"])


def gpu_flat_2d(fits):
    return {"normal": fits.normal.cpu().numpy().reshape(-1, 3),
            **{k: getattr(fits, k).cpu().numpy().reshape(-1) for k in ("offset", "residual", "curvature", "status")}}


def test_distorted_camera_rects_and_tables():
    """Non-separable tan maps (delta lattices): batched rects against the oracle, the constant
    integral tables against numpy's cumsum of the reference lattices."""
    from oracle import oracle as O
    from oracle.compare import normal_angles
    g = load_golden("distorted_f32_w5")
    cam = g["cam"]
    maps = rf.compute_tan_maps(cam.intrinsics())
    tx, ty = O.tan_maps(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, cam.delta_x, cam.delta_y)
    np.testing.assert_array_equal(maps.tan_x, tx)
    np.testing.assert_array_equal(maps.tan_y, ty)
    const = rf.build_constant_channels(maps)
    for name, lat in (("tx", tx), ("ty", ty), ("txty", tx * ty)):
        ref = np.zeros((cam.height + 1, cam.width + 1))
        ref[1:, 1:] = np.cumsum(np.cumsum(lat, axis=0), axis=1)
        np.testing.assert_array_equal(const.channels[name].table.cpu().numpy(), ref)
    rng = np.random.default_rng(3)
    rects = []
    for _ in range(30):
        x0, y0 = int(rng.integers(0, cam.width - 2)), int(rng.integers(0, cam.height - 2))
        rects.append((x0, y0, int(rng.integers(x0 + 2, cam.width + 1)), int(rng.integers(y0 + 2, cam.height + 1))))
    values, valid = O.depth_from_meters(g["depth"])
    depth = torch.from_numpy(g["depth"]).cuda()
    for form, code in (("implicit-standard", O.STANDARD), ("implicit-rgbd", O.RGBD),
                       ("explicit-standard", O.EXPLICIT_STANDARD), ("explicit-rgbd", O.EXPLICIT_RGBD)):
        got = rf.fit_rects(depth, maps, rects, form)
        ref = O.fit_rects(values, valid, tx, ty, rects, code)
        np.testing.assert_array_equal(got["n_points"], ref["n"])
        ok = ((ref["status"] & 2) != 0) & ((ref["status"] & 4) == 0)
        assert normal_angles(got["coef"][ok, :3], ref["coef"][ok, :3]).max() <= 1e-5, form
