"""One-shot check of a whole BASELINE batch in a single fit_pixels call (default C4:
1024 x 1920x1080 uint16 mm, window 15 -- 2.1e9 pixels, past 2^31, ~110 GB of outputs for
the two implicit formulations): the batched outputs of a few frames (first, middle, last)
must equal a separate single-frame call bit for bit, and sampled pixels of the last frame
must match the oracle.  Prints one JSON line.

usage: python tests/diagnostics/full_batch_check.py [C4|C3|C5] [frames]
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2103_06644_b200 as rf  # noqa: E402
from paper_2103_06644_b200 import scenes  # noqa: E402
from oracle.compare import compare  # noqa: E402
from tests.helpers import gpu_flat, oracle_frame  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = scenes.CONFIGS[name]
frames = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.frames
window = cfg.windows[0]
cam = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height)
maps = rf.compute_tan_maps(cam)
depth = scenes.render_batch(cfg, frames=frames, device="cuda")
forms = rf.PIXEL_FORMULATIONS
out = {f: rf.PixelFits.empty(frames, cfg.height, cfg.width, "cuda") for f in forms}
torch.cuda.synchronize()
t0 = time.perf_counter()
rf.fit_pixels(depth, maps, window, forms, out=out)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
pixels = frames * cfg.height * cfg.width
result = {"config": name, "frames": frames, "pixels": pixels, "window": window,
          "seconds": dt, "Mpixel_fits_per_s": 2 * pixels / dt / 1e6,
          "gpu_mem_gb": torch.cuda.max_memory_allocated() / 1e9, "frames_checked": []}
ok = True
for fi in sorted({0, frames // 2, frames - 1}):
    single = rf.fit_pixels(depth[fi:fi + 1], maps, window, forms)
    same = all(torch.equal(torch.nan_to_num(getattr(out[f], k)[fi], nan=-7.0),
                           torch.nan_to_num(getattr(single[f], k)[0], nan=-7.0))
               for f in forms for k in ("normal", "offset", "residual", "curvature", "status"))
    result["frames_checked"].append({"frame": fi, "bit_equal_to_single_frame_call": bool(same)})
    ok &= same
last = frames - 1
host = depth[last].cpu()
pix = np.random.default_rng(5).choice(cfg.height * cfg.width, 2000, replace=False)
for f in forms:
    m = compare(gpu_flat(out[f], last, pix), oracle_frame(host, cam, window, f, pixels=pix))
    result[f"oracle_{f}"] = {k: m[k] for k in ("ok", "max_normal_rad", "max_residual_rel", "status_mismatch")}
    ok &= bool(m["ok"])
result["ok"] = bool(ok)
print(json.dumps(result, default=float))
