"""BASELINE configs 3-5 at their real sizes and intrinsics (1280x720 w9, 1920x1080 uint16
w15, 4096x3072 w31): the GPU runs every pixel of a frame, the oracle checks a seeded
sample (uniform pixels + the worst regions: borders, hole edges, near-depth cells) plus
size-independent properties over the whole frame."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2103_06644_b200 as rf
from oracle.compare import compare
from paper_2103_06644_b200 import scenes
from tests.helpers import gpu_flat, oracle_frame

pytestmark = pytest.mark.gpu


def _sample(depth_np, n, rng):
    H, W = depth_np.shape
    pix = [rng.choice(H * W, n, replace=False)]
    # borders
    pix.append(np.concatenate([np.arange(W), (H - 1) * W + np.arange(W), np.arange(H) * W, np.arange(H) * W + W - 1]))
    # pixels next to holes
    valid = depth_np > 0
    edge = valid & ~np.roll(valid, 1, axis=1)
    idx = np.flatnonzero(edge)
    if idx.size:
        pix.append(rng.choice(idx, min(500, idx.size), replace=False))
    # nearest-depth pixels (the F5 stress region)
    z = np.where(valid, depth_np.astype(np.float64), np.inf).ravel()
    pix.append(np.argsort(z)[:300])
    return np.unique(np.concatenate(pix))


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_fullsize_sampled_parity(name):
    cfg = scenes.CONFIGS[name]
    window = cfg.windows[0]
    frame = scenes.render_frame(cfg, 1000 * int(name[1:]) + 7, device="cuda")
    cam = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height)
    maps = rf.compute_tan_maps(cam)
    out = rf.fit_pixels(frame, maps, window, formulations=rf.FORMULATIONS)
    torch.cuda.synchronize()
    host = frame.cpu()
    dnp = host.numpy()
    pix = _sample(dnp.astype(np.float64), 1500, np.random.default_rng(int(name[1:])))
    for form in rf.FORMULATIONS:
        ref = oracle_frame(host, cam, window, form, pixels=pix)
        got = gpu_flat(out[form], 0, pix) if out[form].normal.dim() == 4 else {
            "normal": out[form].normal.reshape(-1, 3).cpu().numpy()[pix],
            **{k: getattr(out[form], k).reshape(-1).cpu().numpy()[pix]
               for k in ("offset", "residual", "curvature", "status")}}
        m = compare(got, ref, explicit_fit=form.startswith("explicit"))
        assert m["ok"], (name, form, m)
        # whole-frame properties: unit normals, status consistent with the input mask
        st = out[form].status
        fit = (st & rf.STATUS_FIT) != 0
        nrm = out[form].normal[fit]
        assert torch.allclose(nrm.norm(dim=-1), torch.ones_like(nrm[:, 0]), atol=1e-5)
        valid_in = (frame > 0) if frame.dtype == torch.float32 else (frame.to(torch.int32) > 0)
        assert torch.equal((st & rf.STATUS_INPUT_VALID) != 0, valid_in)
        assert bool(torch.isnan(out[form].residual[~fit]).all())
        assert bool((out[form].curvature[fit] >= -1e-6).all()) and bool((out[form].curvature[fit] <= 1 / 3 + 1e-5).all())
