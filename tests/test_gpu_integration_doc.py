"""The ctypes binding printed in INTEGRATION.md (what a maintainer would add to the
reference package) runs as written against the built library and agrees with this
package's own results."""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2103_06644_b200 as rf
from paper_2103_06644_b200 import _native as N
from paper_2103_06644_b200 import scenes

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def _binding_namespace():
    text = (ROOT / "INTEGRATION.md").read_text()
    code = re.findall(r"```python\n(.*?)```", text, re.S)[0]
    # the snippet lives inside the reference package: point its relative imports and the
    # library path at this repository
    code = code.replace("from .camera import CameraIntrinsics", "from paper_2103_06644_b200 import CameraIntrinsics")
    code = code.replace("from .fitting import FORMULATIONS", "from paper_2103_06644_b200 import FORMULATIONS")
    code = code.replace('"/path/to/paper_2103_06644_b200/librangefit_b200.so"', repr(str(N.LIB_PATH)))
    ns: dict = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    return ns


def test_integration_snippet_runs_and_agrees():
    b = _binding_namespace()
    cfg = scenes.small_config("C1", 96, 64)
    frame = scenes.render_frame(cfg, 5).numpy()
    intr = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height)
    h = b["tables"](intr)
    got = b["fit_pixels"](h, frame, 5)
    maps = rf.compute_tan_maps(intr)
    ref = rf.fit_pixels(torch.from_numpy(frame).cuda(), maps, 5, rf.FORMULATIONS)
    for f in rf.FORMULATIONS:
        np.testing.assert_array_equal(got[f]["status"][0], ref[f].status.cpu().numpy())
        np.testing.assert_array_equal(np.nan_to_num(got[f]["normal"][0]), np.nan_to_num(ref[f].normal.cpu().numpy()))
    rects = [(0, 0, 20, 20), (10, 5, 60, 40)]
    rows = b["fit_rects"](h, frame, rects, "implicit-rgbd")
    mine = rf.fit_rects(torch.from_numpy(frame).cuda(), maps, rects, "implicit-rgbd")
    np.testing.assert_array_equal(rows["coef"], mine["coef"])
