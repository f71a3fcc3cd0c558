"""Diagnostic: per-call latency of fit_pixels for small batches (both implicit formulations)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch, paper_2103_06644_b200 as rf  # noqa: E402
from paper_2103_06644_b200 import scenes
for name, frames in (("C1", 1), ("C1", 2), ("C1", 4), ("C3", 1), ("C2", 8)):
    cfg = scenes.CONFIGS[name]
    d = scenes.render_batch(cfg, frames=frames, device="cuda")
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height))
    out = {f: rf.PixelFits.empty(frames, cfg.height, cfg.width, "cuda") for f in rf.PIXEL_FORMULATIONS}
    w = cfg.windows[0] if name != "C2" else 5
    for _ in range(5): rf.fit_pixels(d, maps, w, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): rf.fit_pixels(d, maps, w, out=out)
    e1.record(); torch.cuda.synchronize()
    print(name, frames, "us per call %.1f" % (e0.elapsed_time(e1) / 50 * 1e3))

# the same single-frame call captured once in a CUDA graph and replayed
cfg = scenes.CONFIGS["C1"]
d = scenes.render_batch(cfg, frames=1, device="cuda")
maps = rf.compute_tan_maps(rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height))
out = {f: rf.PixelFits.empty(1, cfg.height, cfg.width, "cuda") for f in rf.PIXEL_FORMULATIONS}
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    rf.fit_pixels(d, maps, 5, out=out, stream=s)
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    rf.fit_pixels(d, maps, 5, out=out, stream=torch.cuda.current_stream())
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    g.replay()
e1.record()
torch.cuda.synchronize()
print("C1 1 graph replay us per call %.1f" % (e0.elapsed_time(e1) / 200 * 1e3))
