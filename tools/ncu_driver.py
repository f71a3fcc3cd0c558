"""Small driver for ncu captures: a few fit_pixels passes over a BASELINE workload.
usage: ncu_driver.py [frames] [window] [reps] [config]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2103_06644_b200 as rf
from paper_2103_06644_b200 import scenes

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 64
window = int(sys.argv[2]) if len(sys.argv) > 2 else 5
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = scenes.CONFIGS[sys.argv[4] if len(sys.argv) > 4 else "C2"]
depth = scenes.render_batch(cfg, frames=frames, device="cuda")
cam = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height)
maps = rf.compute_tan_maps(cam)
out = {f: rf.PixelFits.empty(frames, cfg.height, cfg.width, "cuda") for f in rf.PIXEL_FORMULATIONS}
for _ in range(reps):
    rf.fit_pixels(depth, maps, window, out=out)
torch.cuda.synchronize()
print("done")
