"""Level-synchronous quadtree segmentation on the GPU rect fits vs the reference's
own segment() (golden: tests/golden/make_golden.py:run_segment): same leaf tiles in
the same order, same statuses, same k-means clusters and label lattice."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2103_06644_b200 as rf
import importlib

S = importlib.import_module("paper_2103_06644_b200.segment")  # the package also exports segment()
from tests.helpers import GOLDEN_DIR

pytestmark = pytest.mark.gpu

KEYS = {"implicit-rgbd": "rgbd", "implicit-standard": "std", "explicit-rgbd": "xrgbd", "explicit-standard": "xstd"}


CASES = [("segment_planes", "b200"), ("segment_planes", "naive"), ("segment_planes_integral", "integral"),
         ("segment_planes_max", "b200")]


@pytest.mark.parametrize("case,backend", CASES)
@pytest.mark.parametrize("form", list(rf.FORMULATIONS))
def test_segment_matches_reference(form, case, backend):
    z = np.load(GOLDEN_DIR / f"{case}.npz")
    key = KEYS[form]
    depth = torch.from_numpy(z["depth"]).cuda()
    H, W = depth.shape
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(float(z["fx"]), float(z["fy"]), float(z["cx"]),
                                                   float(z["cy"]), W, H))
    metric = str(z["metric"]) if "metric" in z else "rms"
    thr = float(z[f"{key}_threshold"]) if f"{key}_threshold" in z else None
    cfg = S.SegConfig(formulation=form, backend=backend, initial_tile=32, max_depth=3, k=6, seed=3,
                      error_metric=metric, rms_threshold=thr)
    src = rf.DepthImage(values=z["depth"].astype(np.float64)) if backend == "integral" else depth
    seg = S.segment(src, maps, cfg)
    np.testing.assert_array_equal(np.array([tuple(t.rect) for t in seg.tiles]), z[f"{key}_rects"])
    assert [t.status.value for t in seg.tiles] == list(z[f"{key}_status"])
    np.testing.assert_array_equal(np.array([t.cluster for t in seg.tiles]), z[f"{key}_cluster"])
    np.testing.assert_array_equal(seg.labels.cpu().numpy(), z[f"{key}_labels"])


def test_segment_frame_of_a_batch_and_mask():
    """segment() on frame k of a [B,H,W] batch equals segment() of that frame alone; a mask
    equals zeroing the masked depth."""
    z = np.load(GOLDEN_DIR / "segment_planes.npz")
    d = torch.from_numpy(z["depth"]).cuda()
    H, W = d.shape
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(float(z["fx"]), float(z["fy"]), float(z["cx"]),
                                                   float(z["cy"]), W, H))
    cfg = S.SegConfig(formulation="implicit-rgbd", initial_tile=32, max_depth=3, k=6, seed=3)
    batch = torch.stack([torch.flip(d, dims=[1]), d])
    a = S.segment(batch, maps, cfg, frame=1)
    b = S.segment(d, maps, cfg)
    assert [tuple(t.rect) for t in a.tiles] == [tuple(t.rect) for t in b.tiles]
    assert torch.equal(a.labels, b.labels)
    mask = torch.ones_like(d, dtype=torch.bool)
    mask[10:40, 20:70] = False
    c = S.segment(d, maps, cfg, mask=mask)
    e = S.segment(torch.where(mask, d, torch.zeros_like(d)), maps, cfg)
    assert [t.status for t in c.tiles] == [t.status for t in e.tiles]
    assert torch.equal(c.labels, e.labels)
