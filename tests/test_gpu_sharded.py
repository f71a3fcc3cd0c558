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


def test_back_to_back_calls_with_dependent_launches():
    """A call's second launch (the standard space) is a programmatic dependent launch of its
    first: consecutive calls on one stream over different inputs and outputs -- and a call
    overwriting the outputs of the previous one -- must each equal an isolated call."""
    from paper_2103_06644_b200 import scenes
    cfg = scenes.CONFIGS["C2"]
    cam = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height)
    maps = rf.compute_tan_maps(cam)
    d1 = scenes.render_batch(cfg, frames=8, device="cuda", seed_base=500)
    d2 = scenes.render_batch(cfg, frames=8, device="cuda", seed_base=900)
    ref1 = rf.fit_pixels(d1, maps, 5)
    torch.cuda.synchronize()
    ref1 = {f: {k: getattr(ref1[f], k).clone() for k in ("normal", "status")} for f in ref1}
    ref2 = rf.fit_pixels(d2, maps, 5)
    torch.cuda.synchronize()
    ref2 = {f: {k: getattr(ref2[f], k).clone() for k in ("normal", "status")} for f in ref2}
    shared = {f: rf.PixelFits.empty(8, cfg.height, cfg.width, "cuda") for f in rf.PIXEL_FORMULATIONS}
    other = {f: rf.PixelFits.empty(8, cfg.height, cfg.width, "cuda") for f in rf.PIXEL_FORMULATIONS}
    for _ in range(3):
        rf.fit_pixels(d2, maps, 5, out=other)
        rf.fit_pixels(d1, maps, 5, out=shared)
        rf.fit_pixels(d2, maps, 5, out=shared)  # overwrites the previous call's outputs
    torch.cuda.synchronize()
    for f in rf.PIXEL_FORMULATIONS:
        for k in ("normal", "status"):
            nan = lambda t: torch.nan_to_num(t.float(), nan=-7.0)
            assert torch.equal(nan(getattr(shared[f], k)), nan(ref2[f][k])), (f, k)
            assert torch.equal(nan(getattr(other[f], k)), nan(ref2[f][k])), (f, k)
    assert rf.launches_per_call(rf.PIXEL_FORMULATIONS, 5, torch.float32, (8, cfg.height, cfg.width)) == 2
