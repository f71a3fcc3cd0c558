"""Host-side logic of the package (no GPU): camera validation mirrors the
reference, the scene generator is deterministic and meets the BASELINE
shapes, the product path refuses CPU tensors (no CPU fallback), and the parity
metric itself behaves."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2103_06644_b200 as rf
from paper_2103_06644_b200 import scenes
from oracle.compare import compare, normal_angles


def test_camera_validation_mirrors_reference():
    with pytest.raises(ValueError, match="focal"):
        rf.CameraIntrinsics(0.0, 1.0, 0.5, 0.5, 4, 4)
    with pytest.raises(ValueError, match="principal"):
        rf.CameraIntrinsics(1.0, 1.0, 4.0, 0.5, 4, 4)
    with pytest.raises(ValueError, match="shape"):
        rf.CameraIntrinsics(1.0, 1.0, 0.5, 0.5, 4, 4, delta_x=np.zeros((3, 4)))
    cam = rf.CameraIntrinsics(525.0, 525.0, 319.5, 239.5, 640, 480)
    assert cam.delta_x.shape == (480, 640) and not cam.delta_x.any()


def test_fit_pixels_has_no_cpu_fallback():
    class FakeMaps:
        width, height, device = 8, 8, 0
    with pytest.raises(ValueError, match="CUDA"):
        rf.fit_pixels(torch.ones(8, 8), FakeMaps(), 3)


def test_scene_generator_deterministic_and_shaped():
    cfg = scenes.small_config("C2", 96, 72)
    a = scenes.render_frame(cfg, 7)
    b = scenes.render_frame(cfg, 7)
    c = scenes.render_frame(cfg, 8)
    assert torch.equal(a, b) and not torch.equal(a, c)
    assert a.dtype == torch.float32 and a.shape == (72, 96)
    valid = (a > 0).float().mean().item()
    assert 0.8 < valid < 0.97
    z = a[a > 0]
    assert z.min() > 0.45 and z.max() < 4.6


def test_u16_config_range():
    cfg = scenes.small_config("C4", 64, 48)
    mm = scenes.render_frame(cfg, 3).numpy()
    assert mm.dtype == np.uint16
    nz = mm[mm > 0]
    assert nz.min() >= 300 and nz.max() <= 8000


def test_baseline_configs_match_baseline_json():
    c = scenes.CONFIGS
    assert (c["C1"].frames, c["C1"].width, c["C1"].height, c["C1"].f, c["C1"].windows) == (1, 640, 480, 525.0, (5,))
    assert (c["C2"].frames, c["C2"].cells, c["C2"].windows) == (64, 16, (3, 5, 7, 11, 15))
    assert (c["C3"].frames, c["C3"].width, c["C3"].f, c["C3"].cells, c["C3"].spheres) == (256, 1280, 920.0, 32, 4)
    assert (c["C4"].frames, c["C4"].width, c["C4"].u16, c["C4"].windows) == (1024, 1920, True, (15,))
    assert (c["C5"].frames, c["C5"].width, c["C5"].height, c["C5"].windows) == (128, 4096, 3072, (31,))


def test_compare_metric():
    rng = np.random.default_rng(0)
    n = rng.standard_normal((10, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    ref = {"normal": n, "offset": np.ones(10), "residual": np.full(10, 1.0), "curvature": np.full(10, 0.1),
           "status": np.full(10, 3, np.uint8), "scale": np.ones(10)}
    got = {k: np.array(v, copy=True) for k, v in ref.items()}
    assert compare(got, ref)["ok"]
    got["normal"][3] = -got["normal"][3]          # orientation-blind (normal_angle)
    assert compare(got, ref)["ok"]
    got["residual"][2] *= 1 + 2e-4
    assert not compare(got, ref)["ok"]
    got["residual"][2] = ref["residual"][2]
    got["status"][5] = 1
    got["residual"][5] = np.nan
    assert compare(got, ref)["status_mismatch"] == 1
    assert normal_angles(np.array([[1.0, 0, 0]]), np.array([[1.0, 1e-6, 0]]))[0] == pytest.approx(1e-6)
