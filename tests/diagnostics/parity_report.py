"""Diagnostic: print parity metrics (and worst pixels) for small BASELINE-shaped scenes."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch
import paper_2103_06644_b200 as rf
from paper_2103_06644_b200 import scenes
from tests.helpers import check_frame
from oracle.compare import worst_pixels

cases = [("C4", 15, 192, 144), ("C5", 31, 192, 144), ("C2", 11, 192, 144), ("C1", 5, 640, 480)]
if len(sys.argv) > 1:
    cases = [c for c in cases if c[0] in sys.argv[1:]]
for name, window, W, H in cases:
    cfg = scenes.small_config(name, W, H) if (W, H) != (640, 480) else scenes.CONFIGS[name]
    depth = scenes.render_batch(cfg, frames=1, device="cpu").cuda()
    cam = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height)
    maps = rf.compute_tan_maps(cam)
    out = rf.fit_pixels(depth, maps, window, formulations=rf.FORMULATIONS)
    torch.cuda.synchronize()
    for form in rf.FORMULATIONS:
        m, got, ref = check_frame(depth, out[form], cam, window, form)
        print(json.dumps({"case": name, "window": window, "form": form, **m}))
        idx, ang = worst_pixels(got, ref, 3)
        for i, a in zip(idx, ang):
            y, x = divmod(int(i), cfg.width)
            print("   worst px", (x, y), "ang %.3e" % a, "gpu", got["normal"][i], got["residual"][i], got["curvature"][i],
                  "ref", ref["normal"][i], ref["residual"][i], ref["curvature"][i], "scale", ref["scale"][i])
        gs, rs = got["status"], ref["status"]
        bad = np.nonzero((gs & 3) != (rs & 3))[0][:3]
        for i in bad:
            y, x = divmod(int(i), cfg.width)
            print("   status mismatch px", (x, y), gs[i], rs[i])
        sel = ((rs & 2) != 0) & ((gs & 2) != 0)
        rr = np.abs(got["residual"][sel].astype(np.float64) - ref["residual"][sel]) / np.maximum(np.abs(ref["residual"][sel]), 1e-30)
        cc = np.abs(got["curvature"][sel].astype(np.float64) - ref["curvature"][sel]) / np.maximum(np.abs(ref["curvature"][sel]), 1e-30)
        ii = np.nonzero(sel)[0]
        for arr, lab in ((rr, "res"), (cc, "curv")):
            j = np.argsort(-arr)[:2]
            for jj in j:
                i = ii[jj]; y, x = divmod(int(i), cfg.width)
                print(f"   worst {lab} px", (x, y), "rel %.3e" % arr[jj], "gpu", got["residual"][i], got["curvature"][i], "ref", ref["residual"][i], ref["curvature"][i])
