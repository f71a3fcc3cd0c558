"""BASELINE config 2 at its real size (640x480 float32, 16-cell Voronoi planes, 5% invalid)
for every window of its sweep {3, 5, 7, 11, 15}: frames 0 and 63 of the bench batch (the
seeds bench.py times), every pixel of both frames against the oracle (the reference's naive
backend, fitting.py:757-786 / :339-402), all four formulations, status bits exact."""

from __future__ import annotations

import pytest
import torch

import paper_2103_06644_b200 as rf
from oracle.compare import compare
from paper_2103_06644_b200 import scenes
from paper_2103_06644_b200.shard import rank_seed_base
from tests.helpers import gpu_flat, oracle_frame

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("window", [3, 5, 7, 11, 15])
def test_c2_fullsize_window_sweep(window):
    cfg = scenes.CONFIGS["C2"]
    base = rank_seed_base(2, 0)
    depth = torch.stack([scenes.render_frame(cfg, base + k, device="cuda") for k in (0, 63)])
    cam = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height)
    maps = rf.compute_tan_maps(cam)
    out = rf.fit_pixels(depth, maps, window, rf.FORMULATIONS)
    torch.cuda.synchronize()
    host = depth.cpu()
    for frame in range(2):
        for form in rf.FORMULATIONS:
            ref = oracle_frame(host[frame], cam, window, form)
            m = compare(gpu_flat(out[form], frame), ref, explicit_fit=form.startswith("explicit"))
            assert m["ok"] and m["compared"] > 200000, (window, frame, form, m)
