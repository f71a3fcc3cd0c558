"""Dump per-pixel window data for the worst parity pixels (C5-small standard)."""
import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch
import paper_2103_06644_b200 as rf
from paper_2103_06644_b200 import scenes
from tests.helpers import check_frame
from oracle.compare import worst_pixels
from oracle import oracle as O

name, window, W, H = "C5", 31, 192, 144
cfg = scenes.small_config(name, W, H)
depth = scenes.render_batch(cfg, frames=1, device="cpu")
np.save("gpurun_out/c5small_depth.npy", depth.numpy())
d = depth.cuda()
cam = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height)
maps = rf.compute_tan_maps(cam)
out = rf.fit_pixels(d, maps, window)
torch.cuda.synchronize()
m, got, ref = check_frame(d, out["implicit-standard"], cam, window, "implicit-standard")
idx, ang = worst_pixels(got, ref, 30)
np.save("gpurun_out/c5small_worst.npy", np.stack([idx, ang], 1))
print(json.dumps({"f": cfg.f, **m}))
