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
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height))
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


def gpu_flat_2d(fits):
    return {"normal": fits.normal.cpu().numpy().reshape(-1, 3),
            **{k: getattr(fits, k).cpu().numpy().reshape(-1) for k in ("offset", "residual", "curvature", "status")}}
