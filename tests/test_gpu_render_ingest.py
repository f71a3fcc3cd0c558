"""Device renderer against the reference's render_scene (golden: make_golden.py:run_render),
float64 depth through the fit kernels, and batched file ingest."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2103_06644_b200 as rf
from paper_2103_06644_b200 import imageio as io
from paper_2103_06644_b200 import synth
from tests.helpers import GOLDEN_DIR

pytestmark = pytest.mark.gpu


def _scene_and_maps():
    z = np.load(GOLDEN_DIR / "render_planes.npz")
    W, H = int(z["width"]), int(z["height"])
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(float(z["fx"]), float(z["fy"]), float(z["cx"]),
                                                   float(z["cy"]), W, H))
    planes = []
    for p, r in zip(z["planes"], z["rects"]):
        g = synth.GroundTruthPlane(p, None if r[0] == -1 and r[2] == -1 else tuple(int(v) for v in r))
        object.__setattr__(g, "coefficients", p.copy())  # the reference's normalised bits, not re-normalised
        planes.append(g)
    return z, synth.SyntheticScene(tuple(planes)), maps


@pytest.mark.parametrize("case", ["plain", "noise", "drop", "both"])
def test_render_matches_reference_bit_for_bit(case):
    z, scene, maps = _scene_and_maps()
    k = float(z[f"{case}_noise"])
    d, labels = synth.render_scene(scene, maps, noise=synth.NoiseModel(k) if k > 0 else None,
                                   seed=int(z[f"{case}_seed"]), dropout=float(z[f"{case}_dropout"]))
    np.testing.assert_array_equal(d.valid, z[f"{case}_valid"])
    np.testing.assert_array_equal(d.values, z[f"{case}_depth"])
    np.testing.assert_array_equal(labels, z[f"{case}_labels"])


def test_device_rng_render_properties():
    z, scene, maps = _scene_and_maps()
    depth, valid, labels = synth.render_depth(scene, maps, synth.NoiseModel(), seed=5, dropout=0.25, rng="device")
    plain, pvalid, plabels = synth.render_depth(scene, maps)
    v, pv = valid.bool(), pvalid.bool()
    assert not (v & ~pv).any()                        # dropout only removes pixels
    frac = 1.0 - v.sum().item() / pv.sum().item()
    assert 0.15 < frac < 0.35
    assert (labels[v] == plabels[v]).all() and (labels[~v] == 255).all()
    rel = ((depth[v] - plain[v]) / (1.425e-3 * plain[v] ** 2)).cpu().numpy()
    assert abs(rel.mean()) < 0.2 and 0.8 < rel.std() < 1.2  # N(0, 1) noise in units of sigma_Z
    again, _, _ = synth.render_depth(scene, maps, synth.NoiseModel(), seed=5, dropout=0.25, rng="device")
    assert torch.equal(again, depth)                  # seeded


def test_float64_depth_equals_float32_path():
    d32 = torch.from_numpy(np.load(GOLDEN_DIR / "planes_f32_w5.npz")["depth"]).cuda()
    H, W = d32.shape
    z = np.load(GOLDEN_DIR / "planes_f32_w5.npz")
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(float(z["fx"]), float(z["fy"]), float(z["cx"]),
                                                   float(z["cy"]), W, H))
    a = rf.fit_pixels(d32, maps, 5)
    b = rf.fit_pixels(d32.double(), maps, 5)
    for f in rf.PIXEL_FORMULATIONS:
        for k in ("normal", "offset", "residual", "curvature", "status"):
            torch.testing.assert_close(getattr(a[f], k), getattr(b[f], k), rtol=0, atol=0, equal_nan=True)
    ra = rf.fit_rects(d32, maps, [(0, 0, 20, 20), (5, 7, 30, 31)], "implicit-rgbd")
    rb = rf.fit_rects(d32.double(), maps, [(0, 0, 20, 20), (5, 7, 30, 31)], "implicit-rgbd")
    np.testing.assert_array_equal(ra["coef"], rb["coef"])


def test_batched_ingest(tmp_path):
    d = synth.read_depth(GOLDEN_DIR / "io_depth.pgm")
    mm = io.read_pgm16(GOLDEN_DIR / "io_depth.pgm")
    for i in range(3):
        io.write_pgm16(tmp_path / f"f{i}.pgm", mm)
        io.write_raw_float(tmp_path / f"f{i}.rf64", np.where(d.valid, d.values, np.nan))
    b16 = io.load_depth_batch(sorted(tmp_path.glob("*.pgm")))
    b64 = io.load_depth_batch(sorted(tmp_path.glob("*.rf64")))
    assert b16.dtype == torch.uint16 and b16.shape == (3, *mm.shape)
    assert b64.dtype == torch.float64
    np.testing.assert_array_equal(b16[1].cpu().numpy(), mm)
    H, W = mm.shape
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(50.0, 52.0, 19.5, 14.5, W, H))
    a = rf.fit_pixels(b16, maps, 3)
    b = rf.fit_pixels(b64, maps, 3)  # the same mm / 1000.0 values, float64 on the wire
    for f in rf.PIXEL_FORMULATIONS:
        torch.testing.assert_close(a[f].normal, b[f].normal, rtol=0, atol=0, equal_nan=True)
        torch.testing.assert_close(a[f].status, b[f].status, rtol=0, atol=0)


@pytest.mark.parametrize("dtype", ["f32", "u16", "f64"])
def test_host_pipeline_equals_device_call(dtype):
    from paper_2103_06644_b200 import scenes
    cfg = scenes.small_config("C4" if dtype == "u16" else "C2", 160, 120)
    depth = scenes.render_batch(cfg, frames=11, device="cuda")
    if dtype == "f64":
        depth = depth.double()
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height))
    ref = rf.fit_pixels(depth, maps, 5)
    pipe = rf.HostPipeline(maps, 5, chunk_frames=4, slots=2)   # 3 chunks, the last one short
    for _ in range(2):                                          # second run reuses the buffers
        got = pipe.run(depth.cpu().pin_memory())
        for f in rf.PIXEL_FORMULATIONS:
            for k in ("normal", "offset", "residual", "curvature", "status"):
                torch.testing.assert_close(getattr(got[f], k), getattr(ref[f], k).cpu(), rtol=0, atol=0,
                                           equal_nan=True)
    with pytest.raises(ValueError):
        pipe.run(depth)  # device tensors go through fit_pixels
