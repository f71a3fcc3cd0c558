"""Edge cases of the sm_100a path against the oracle: batches, padded rows,
uint16 input, tiny/odd frame sizes, windows larger than the frame, empty and
all-invalid inputs, maximum window, and argument errors."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2103_06644_b200 as rf
from paper_2103_06644_b200 import scenes
from tests.helpers import check_frame, gpu_flat

pytestmark = pytest.mark.gpu


def _maps(cfg):
    cam = rf.CameraIntrinsics(cfg.f, cfg.f, cfg.cx, cfg.cy, cfg.width, cfg.height)
    return cam, rf.compute_tan_maps(cam)


def test_batch_frames_are_independent():
    cfg = scenes.small_config("C2", 96, 64)
    batch = scenes.render_batch(cfg, frames=3).cuda()
    cam, maps = _maps(cfg)
    out = rf.fit_pixels(batch, maps, 5)
    single = rf.fit_pixels(batch[1].contiguous(), maps, 5)
    torch.cuda.synchronize()
    for f in rf.PIXEL_FORMULATIONS:
        assert torch.equal(out[f].status[1], single[f].status)
        assert torch.equal(torch.nan_to_num(out[f].normal[1]), torch.nan_to_num(single[f].normal))
        for k in range(3):
            m, _, _ = check_frame(batch, out[f], cam, 5, f, frame=k)
            assert m["ok"], (k, f, m)


def test_padded_rows_match_contiguous():
    cfg = scenes.small_config("C1", 100, 60)
    frame = scenes.render_frame(cfg, 3).cuda()
    padded = torch.zeros((60, 128), dtype=torch.float32, device="cuda")
    padded[:, :100] = frame
    cam, maps = _maps(cfg)
    a = rf.fit_pixels(frame, maps, 7)
    b = rf.fit_pixels(padded[:, :100], maps, 7)
    torch.cuda.synchronize()
    for f in rf.PIXEL_FORMULATIONS:
        assert torch.equal(a[f].status, b[f].status)
        assert torch.equal(torch.nan_to_num(a[f].normal), torch.nan_to_num(b[f].normal))


def test_uint16_millimetres():
    cfg = scenes.small_config("C4", 128, 72)
    mm = scenes.render_batch(cfg, frames=2).cuda()
    cam, maps = _maps(cfg)
    out = rf.fit_pixels(mm, maps, 9)
    torch.cuda.synchronize()
    for f in rf.PIXEL_FORMULATIONS:
        for k in range(2):
            m, _, _ = check_frame(mm, out[f], cam, 9, f, frame=k)
            assert m["ok"], (k, f, m)


@pytest.mark.parametrize("W,H,window,dtype", [(5, 7, 9, "f32"), (1, 1, 3, "f32"), (70, 3, 5, "f32"),
                                               (3, 70, 5, "f32"), (65, 17, 3, "f32"), (129, 33, 63, "f32"),
                                               (128, 32, 63, "f32"), (128, 32, 65, "f32"), (128, 40, 65, "f64"),
                                               (128, 24, 31, "f64")])
def test_odd_sizes_and_large_windows(W, H, window, dtype):
    """Includes 16-byte aligned rows with the largest windows (TMA smem footprint over the
    opt-in limit -> LDG halo path) and float64 input."""
    cfg = scenes.SceneConfig("C1", 1, W, H, 60.0, (window,), (0.5, 4.0), cells=0, planes=3)
    frame = scenes.render_frame(cfg, 11).cuda()
    if dtype == "f64":
        frame = frame.double()
    cam, maps = _maps(cfg)
    out = rf.fit_pixels(frame, maps, window)
    torch.cuda.synchronize()
    for f in rf.PIXEL_FORMULATIONS:
        m, _, _ = check_frame(frame, out[f], cam, window, f)
        assert m["ok"], (f, m)


def test_all_invalid_and_window_one():
    cfg = scenes.small_config("C1", 64, 32)
    cam, maps = _maps(cfg)
    zeros = torch.zeros((32, 64), dtype=torch.float32, device="cuda")
    out = rf.fit_pixels(zeros, maps, 5)
    frame = scenes.render_frame(cfg, 2).cuda()
    one = rf.fit_pixels(frame, maps, 1)
    torch.cuda.synchronize()
    for f in rf.PIXEL_FORMULATIONS:
        assert int(out[f].status.max()) == 0
        assert torch.isnan(out[f].residual).all() and torch.isnan(out[f].normal).all()
        st = one[f].status
        assert torch.equal(st, (frame > 0).to(torch.uint8))   # n = 1 < MIN_SAMPLES
        assert torch.isnan(one[f].curvature).all()


def test_nonfinite_and_negative_depth_are_invalid():
    cfg = scenes.small_config("C1", 64, 48)
    cam, maps = _maps(cfg)
    frame = scenes.render_frame(cfg, 5)
    frame[3, 4] = float("nan")
    frame[10, 10] = float("inf")
    frame[20, 30] = -1.0
    frame[21, 30] = 1e-30  # positive denormal-ish depth stays valid
    d = frame.cuda()
    out = rf.fit_pixels(d, maps, 5)
    torch.cuda.synchronize()
    for f in rf.PIXEL_FORMULATIONS:
        st = out[f].status.cpu()
        assert st[3, 4] == 0 and st[10, 10] == 0 and st[20, 30] == 0
        m, _, _ = check_frame(d, out[f], cam, 5, f)
        assert m["status_mismatch"] == 0


def test_empty_batch():
    cfg = scenes.small_config("C1", 32, 32)
    _, maps = _maps(cfg)
    out = rf.fit_pixels(torch.zeros((0, 32, 32), device="cuda"), maps, 5)
    assert out[rf.IMPLICIT_RGBD].status.shape == (0, 32, 32)


def test_argument_errors():
    cfg = scenes.small_config("C1", 32, 32)
    _, maps = _maps(cfg)
    d = torch.ones((32, 32), device="cuda")
    with pytest.raises(ValueError):
        rf.fit_pixels(d, maps, 4)                 # even window
    with pytest.raises(ValueError):
        rf.fit_pixels(d, maps, 67)                # radius > 32
    with pytest.raises(ValueError):
        rf.fit_pixels(torch.ones((32, 31), device="cuda"), maps, 5)
    with pytest.raises(ValueError):
        rf.fit_pixels(d.int(), maps, 5)           # int32 is not a depth type
    with pytest.raises(ValueError):
        rf.fit_pixels(d, maps, 5, formulations=("implicit-disparity",))


def test_single_formulation_and_stream():
    cfg = scenes.small_config("C1", 96, 64)
    frame = scenes.render_frame(cfg, 4).cuda()
    cam, maps = _maps(cfg)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out = rf.fit_pixels(frame, maps, 5, formulations=rf.IMPLICIT_STANDARD, stream=s)
    s.synchronize()
    assert list(out) == [rf.IMPLICIT_STANDARD]
    m, _, _ = check_frame(frame, out[rf.IMPLICIT_STANDARD], cam, 5, rf.IMPLICIT_STANDARD)
    assert m["ok"], m


def test_concurrent_callers_on_separate_streams():
    """Small batches fork the second space's kernel onto a side stream; concurrent callers on
    their own streams must still get exactly the single-caller results."""
    import threading
    cfg = scenes.small_config("C1", 160, 120)
    cam, maps = _maps(cfg)
    frames = [scenes.render_frame(cfg, 30 + i).cuda() for i in range(2)]
    ref = [rf.fit_pixels(f, maps, 5) for f in frames]
    torch.cuda.synchronize()
    errors = []

    def worker(i):
        try:
            st = torch.cuda.Stream()
            for _ in range(20):
                with torch.cuda.stream(st):
                    got = rf.fit_pixels(frames[i], maps, 5, stream=st)
                st.synchronize()
                for f in rf.PIXEL_FORMULATIONS:
                    if not torch.equal(torch.nan_to_num(got[f].normal), torch.nan_to_num(ref[i][f].normal)):
                        errors.append((i, f))
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(repr(e))

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[:4]


def test_fit_pixels_is_cuda_graph_capturable():
    """A streaming loop can capture fit_pixels once in a CUDA graph and replay it (the fork
    onto the side stream and the join are captured too)."""
    cfg = scenes.small_config("C1", 160, 120)
    _, maps = _maps(cfg)
    static_in = scenes.render_frame(cfg, 40).cuda()
    out = {f: rf.PixelFits.empty(1, cfg.height, cfg.width, "cuda") for f in rf.PIXEL_FORMULATIONS}
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        rf.fit_pixels(static_in, maps, 5, out=out, stream=s)  # warm-up outside capture
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        rf.fit_pixels(static_in, maps, 5, out=out, stream=torch.cuda.current_stream())
    for seed in (41, 42):
        frame = scenes.render_frame(cfg, seed).cuda()
        static_in.copy_(frame)
        g.replay()
        torch.cuda.synchronize()
        ref = rf.fit_pixels(frame, maps, 5)
        for f in rf.PIXEL_FORMULATIONS:
            assert torch.equal(out[f].status[0], ref[f].status)
            assert torch.equal(torch.nan_to_num(out[f].normal[0]), torch.nan_to_num(ref[f].normal))
