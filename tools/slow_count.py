"""Experiment: fraction of windows leaving the fast solve (build with RF_NVCC_FLAGS=-DRF_COUNT_SLOW)."""
import ctypes, sys
sys.path.insert(0, ".")
import torch
import paper_2103_06644_b200 as rf
from paper_2103_06644_b200 import scenes, _native as N

lib = N.load()
cnt = (ctypes.c_ulonglong * 256)()
for name, frames, windows in [("C1", 1, (5,)), ("C2", 16, (3, 5, 7, 11, 15)), ("C3", 8, (9,)), ("C4", 4, (15,)), ("C5", 1, (31,))]:
    cfg = scenes.CONFIGS[name]
    depth = scenes.render_batch(cfg, frames=frames, device="cuda")
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height))
    for w in windows:
        lib.rf_debug_slow_counts(cnt, 1)
        out = rf.fit_pixels(depth, maps, w)
        torch.cuda.synchronize()
        lib.rf_debug_slow_counts(cnt, 1)
        fit = {f: int((out[f].status & 2).ne(0).sum()) for f in out}
        print(f"{name} w{w}: slow std {cnt[0] / max(1, fit[rf.IMPLICIT_STANDARD]):.5f} "
              f"rgbd {cnt[1] / max(1, fit[rf.IMPLICIT_RGBD]):.5f}", flush=True)
