"""In-process frame sharding (shard.fit_frames_sharded): a host batch split into contiguous
frame ranges, one HostPipeline per device from its own host thread, outputs straight into one
pinned host array.  Only one GPU is available here, so the device list repeats it (two
pipelines, two threads, their own streams): the outputs must equal one fit_pixels call on
the whole batch bit for bit, for an even and an uneven split."""

from __future__ import annotations

import pytest
import torch

import paper_2103_06644_b200 as rf
from paper_2103_06644_b200 import scenes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("frames,devices", [(6, [0, 0]), (7, [0, 0, 0])])
def test_sharded_equals_single_call(frames, devices):
    cfg = scenes.small_config("C2", 160, 96)
    host = scenes.render_batch(cfg, frames=frames, device="cpu")
    cam = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height)
    got = rf.fit_frames_sharded(host.pin_memory(), cam, 5, rf.FORMULATIONS, devices=devices, chunk_frames=2)
    ref = rf.fit_pixels(host.cuda(), rf.compute_tan_maps(cam), 5, rf.FORMULATIONS)
    torch.cuda.synchronize()
    for f in rf.FORMULATIONS:
        for k in ("normal", "offset", "residual", "curvature", "status"):
            a, b = getattr(got[f], k), getattr(ref[f], k).cpu()
            assert torch.equal(torch.nan_to_num(a, nan=-7.0), torch.nan_to_num(b, nan=-7.0)), (f, k)


def test_sharded_rejects_device_tensors():
    with pytest.raises(ValueError):
        rf.fit_frames_sharded(torch.zeros(1, 8, 8, device="cuda"), None, 5)
