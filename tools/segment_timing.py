"""Diagnostic: wall time of segment() on a 640x480 frame for each backend and error metric."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2103_06644_b200 as rf  # noqa: E402
from paper_2103_06644_b200 import scenes  # noqa: E402
from paper_2103_06644_b200.segment import SegConfig, segment  # noqa: E402

cfg = scenes.CONFIGS["C2"]
depth = scenes.render_frame(cfg, 2000, device="cuda")
maps = rf.compute_tan_maps(rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height))
for backend in ("b200", "integral"):
    for metric in ("rms", "max"):
        for form in (rf.IMPLICIT_RGBD, rf.IMPLICIT_STANDARD):
            c = SegConfig(formulation=form, backend=backend, error_metric=metric)
            segment(depth, maps, c)  # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                seg = segment(depth, maps, c)
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) / 5 * 1e3
            print(f"{backend:8s} {metric} {form:18s} {ms:7.2f} ms  tiles {len(seg.tiles)} fitted {seg.n_fitted}")
