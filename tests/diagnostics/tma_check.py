"""Diagnostic: a 3-frame batch through the TMA-fed kernels, parity per frame against the oracle."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch, paper_2103_06644_b200 as rf
from paper_2103_06644_b200 import scenes
from tests.helpers import check_frame
cfg = scenes.small_config("C2", 96, 64)
batch = scenes.render_batch(cfg, frames=3).cuda()
cam = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height)
maps = rf.compute_tan_maps(cam)
out = rf.fit_pixels(batch, maps, 5)
torch.cuda.synchronize()
for f in rf.PIXEL_FORMULATIONS:
    for k in range(3):
        m, _, _ = check_frame(batch, out[f], cam, 5, f, frame=k)
        print(f, k, m["ok"], m["status_mismatch"], m["max_normal_rad"])
