"""Long randomised parity sweep (diagnostic, not collected by pytest): N seeded random frames
(sizes, windows, element types, masks, hostile values, distortion lattices) through
fit_pixels against the oracle; prints failures and a summary line.

usage: python tests/diagnostics/stress_sweep.py [N] [seed0]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_06644_b200 as rf  # noqa: E402
from oracle.compare import compare  # noqa: E402
from tests.helpers import Cam, gpu_flat, oracle_frame  # noqa: E402
from tests.test_gpu_random import _frame  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 7000
fails = 0
worst = {"ang": 0.0, "res": 0.0, "cur": 0.0}
for i in range(N):
    rng = np.random.default_rng(seed0 + i)
    W = int(rng.integers(1, 150))
    H = int(rng.integers(1, 90))
    window = int(rng.choice([1, 3, 5, 7, 9, 11, 13, 15, 17, 21, 25, 31]))
    dtype = ["f32", "u16", "f64"][int(rng.integers(3))]
    z, cam = _frame(rng, W, H, dtype)
    if rng.random() < 0.2:
        cam = Cam(cam.fx, cam.fy, cam.cx, cam.cy, W, H, rng.uniform(-0.4, 0.4, (H, W)), rng.uniform(-0.4, 0.4, (H, W)))
    mask = torch.from_numpy(rng.random((H, W)) > 0.2).cuda() if rng.random() < 0.3 else None
    maps = rf.compute_tan_maps(cam.intrinsics())
    out = rf.fit_pixels(torch.from_numpy(z).cuda(), maps, window, rf.FORMULATIONS, mask=mask)
    torch.cuda.synchronize()
    for form in rf.FORMULATIONS:
        ref = oracle_frame(torch.from_numpy(z), cam, window, form, mask=None if mask is None else mask.cpu())
        m = compare(gpu_flat(out[form]), ref, explicit_fit=form.startswith("explicit"))
        worst["ang"] = max(worst["ang"], m["max_normal_rad"])
        worst["res"] = max(worst["res"], m["max_residual_rel"])
        worst["cur"] = max(worst["cur"], m["max_curvature_rel"])
        if not m["ok"]:
            fails += 1
            print("FAIL", i, W, H, window, dtype, form, {k: m[k] for k in ("status_mismatch", "max_normal_rad",
                  "max_residual_rel", "max_curvature_rel", "nonfit_is_nan", "normal_fail", "residual_fail",
                  "curvature_fail")}, flush=True)
print(f"SWEEP {N} frames x 4 formulations: {fails} failures; worst normal {worst['ang']:.2e} rad, "
      f"residual {worst['res']:.2e}, curvature {worst['cur']:.2e} (in units of the 1e-4 bars: <= 1e-4 passes)")
