"""Host-side pieces of the reference-compatible API (no GPU): DepthImage, the scatter
value types, the argument checks that run before any launch, the CSV row format."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2103_06644_b200 as rf
from paper_2103_06644_b200 import integral as I


def test_depth_image_validity_and_millimetres():
    d = rf.DepthImage(values=np.array([[1.0, 0.0], [np.nan, -2.0]]))
    np.testing.assert_array_equal(d.valid, [[True, False], [False, False]])
    d = rf.DepthImage(values=np.array([[1.0, 2.0]]), valid=np.array([[False, True]]))
    np.testing.assert_array_equal(d.valid, [[False, True]])
    mm = np.array([[0, 1500], [65535, 3]], np.uint16)
    d = rf.DepthImage.from_millimeters(mm)
    np.testing.assert_array_equal(d.values, mm.astype(np.float64) / 1000.0)
    np.testing.assert_array_equal(d.valid, mm > 0)
    np.testing.assert_array_equal(d.to_millimeters(), mm)
    with pytest.raises(ValueError):
        rf.DepthImage(values=np.zeros(3))
    with pytest.raises(ValueError):
        rf.DepthImage(values=np.ones((2, 2)), valid=np.ones((3, 2), bool))


def test_fit_checks_run_before_the_device():
    with pytest.raises(rf.InsufficientSamplesError):
        rf.fit_implicit_standard(rf.Scatter4(matrix=np.eye(4), n=3))
    with pytest.raises(rf.InsufficientSamplesError):
        rf.fit_explicit_rgbd(rf.Scatter3(matrix=np.eye(3), rhs=np.zeros(3), n=2))
    m = np.eye(4)
    m[0, 1] = 1.0
    with pytest.raises(ValueError, match="not symmetric"):
        rf.fit_implicit_rgbd(rf.Scatter4(matrix=m, n=4))
    m = np.eye(4)
    m[2, 2] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        rf.fit_implicit_standard(rf.Scatter4(matrix=m, n=4))
    with pytest.raises(ValueError, match="requires a per-frame channel stack"):
        rf.fit_rect(None, None, rf.Rect(0, 0, 2, 2), "implicit-rgbd", backend="integral")
    with pytest.raises(ValueError, match="unknown backend"):
        rf.fit_rect(None, None, rf.Rect(0, 0, 2, 2), "implicit-rgbd", backend="cuda")
    with pytest.raises(ValueError, match="unknown formulation"):
        rf.scatter_from_integrals(None, None, rf.Rect(0, 0, 2, 2), "implicit")
    with pytest.raises(ValueError, match="out of bounds"):
        I._check_rect(rf.Rect(0, 0, 5, 2), 4, 4)


def test_csv_row_matches_reference_format():
    assert rf.CSV_HEADER == "formulation,backend,x0,y0,x1,y1,a,b,c,d,lambda,rms,n_points"
    res = rf.FitResult(rf.ImplicitPlane(np.array([0.0, 0.0, 2.0, -6.0])), 25, 0.5, 1.25, False)
    row = rf.fit_result_csv_row(res, "implicit-standard", "naive", rf.Rect(1, 2, 6, 7))
    c = 1.0 / np.sqrt(10.0)
    assert row == ",".join(["implicit-standard", "naive", "1", "2", "6", "7", repr(0.0), repr(0.0),
                            repr(float(np.float64(2.0) / np.linalg.norm([0, 0, 2.0, -6.0]))),
                            repr(float(np.float64(-6.0) / np.linalg.norm([0, 0, 2.0, -6.0]))),
                            "1.25", "0.5", "25"])
    assert abs(float(row.split(",")[8]) - c) < 1e-15
    xres = rf.FitResult(rf.ExplicitPlane(np.array([0.5, -0.25, 2.0]), "standard"), 9, None, None, False)
    xrow = rf.fit_result_csv_row(xres, "explicit-standard", "integral", rf.Rect(0, 0, 3, 3))
    assert xrow.split(",")[10:] == ["", "", "9"]


def test_channel_constants_match_reference_names():
    assert I.CONSTANT_CHANNELS == ("tx2", "txty", "ty2", "tx", "ty")
    assert I.STANDARD_IMPLICIT_CHANNELS == ("x2", "xy", "xz", "x", "y2", "yz", "y", "z2", "z")
    assert I.RGBD_IMPLICIT_CHANNELS == ("tx_over_z", "ty_over_z", "inv_z", "inv_z2")
    assert I.STANDARD_EXPLICIT_CHANNELS == ("x2", "xy", "x", "y2", "y", "xz", "yz", "z")
    assert I.RGBD_EXPLICIT_CHANNELS == ("tx_over_z", "ty_over_z", "inv_z")
    assert I.HOLE_CORRECTION_CHANNELS == ("m_tx2", "m_txty", "m_ty2", "m_tx", "m_ty")
    from paper_2103_06644_b200 import _native as N
    for name in (*I.CONSTANT_CHANNELS, *I.STANDARD_IMPLICIT_CHANNELS, *I.RGBD_IMPLICIT_CHANNELS,
                 *I.HOLE_CORRECTION_CHANNELS, I.COUNT_CHANNEL, "ones"):
        assert name in N.RF_CHANNELS
    assert len(set(N.RF_CHANNELS.values())) == len(N.RF_CHANNELS) == 25


def test_golden_integral_fixtures_are_consistent():
    """The committed reference tables: zero first row/column, count corner = valid pixels,
    and box sums of the count table equal the recorded sample counts."""
    for case in ("integral_holes", "integral_full"):
        z = np.load(rf.__path__[0] + f"/../tests/golden/{case}.npz")
        t = z["std_count"]
        assert (t[0] == 0).all() and (t[:, 0] == 0).all()
        assert t[-1, -1] == z["valid"].sum()
        for k, (x0, y0, x1, y1) in enumerate(z["rects"]):
            n = int(round(t[y1, x1] - t[y0, x1] - t[y1, x0] + t[y0, x0]))
            if z["std_n"][k] >= 0:
                assert n == z["std_n"][k]


def test_interchange_files_match_reference_bytes(tmp_path):
    from paper_2103_06644_b200 import imageio as io
    from paper_2103_06644_b200 import synth
    g = rf.__path__[0] + "/../tests/golden/"
    mm = io.read_pgm16(g + "io_depth.pgm")
    io.write_pgm16(tmp_path / "a.pgm", mm)
    assert (tmp_path / "a.pgm").read_bytes() == open(g + "io_depth.pgm", "rb").read()
    raw = io.read_raw_float(g + "io_depth.rf64")
    io.write_raw_float(tmp_path / "a.rf64", raw)
    assert (tmp_path / "a.rf64").read_bytes() == open(g + "io_depth.rf64", "rb").read()
    lab = io.read_pgm8(g + "io_labels.pgm")
    io.write_pgm8(tmp_path / "l.pgm", lab)
    assert (tmp_path / "l.pgm").read_bytes() == open(g + "io_labels.pgm", "rb").read()
    d = synth.read_depth(g + "io_depth.rf64")
    assert d.valid.sum() == np.isfinite(raw).sum()
    synth.write_depth(tmp_path / "b.pgm", d)
    assert (tmp_path / "b.pgm").read_bytes() == open(g + "io_depth.pgm", "rb").read()
    np.testing.assert_array_equal(synth.read_depth(tmp_path / "b.pgm").values, mm / 1000.0)
    rgb = np.arange(2 * 3 * 3, dtype=np.uint8).reshape(2, 3, 3)
    io.write_ppm(tmp_path / "c.ppm", rgb)
    np.testing.assert_array_equal(io.read_ppm(tmp_path / "c.ppm"), rgb)
    (tmp_path / "bad.pgm").write_bytes(b"P5\n# comment\n4 4\n65535\n\x00\x01")
    with pytest.raises(ValueError, match="truncated"):
        io.read_pgm16(tmp_path / "bad.pgm")
    with pytest.raises(ValueError, match="RF64"):
        io.read_raw_float(tmp_path / "bad.pgm")


def test_scene_parsing_and_mask_rect_slices():
    from paper_2103_06644_b200 import synth
    sc = synth.parse_scene("# two planes\n0 0 1 -2\n0.1 0 -1 3  5 6 20 30  # masked\n")
    assert len(sc.planes) == 2 and sc.planes[1].mask_rect == (5, 6, 20, 30)
    np.testing.assert_allclose(np.linalg.norm(sc.planes[1].normal), 1.0)
    with pytest.raises(ValueError, match="expected"):
        synth.parse_scene("1 2 3\n")
    with pytest.raises(ValueError, match="no planes"):
        synth.parse_scene("# nothing\n")
    rects = synth._plane_rects(synth.SyntheticScene((
        synth.GroundTruthPlane(np.array([0, 0, 1.0, -1])),
        synth.GroundTruthPlane(np.array([0, 0, 1.0, -1]), mask_rect=(-10, 22, 12, 40)),
        synth.GroundTruthPlane(np.array([0, 0, 1.0, -1]), mask_rect=(5, -3, 99, 20)))), 40, 30)
    # numpy slice semantics of masked[y0:y1, x0:x1] (synth.py:145-148)
    assert rects.tolist() == [[0, 0, 40, 30], [30, 22, 30, 30], [5, 27, 40, 27]]


def _host_maps(intr):
    """TanAngleMaps without device tables (its lattices are computed on the host)."""
    import ctypes
    from paper_2103_06644_b200.pixels import TanAngleMaps
    return TanAngleMaps(intrinsics=intr, device=0, _handle=ctypes.c_void_p())


def test_camera_helpers(tmp_path):
    intr = rf.CameraIntrinsics(fx=500.0, fy=520.0, cx=319.5, cy=239.5, width=640, height=480)
    maps = _host_maps(intr)
    p = rf.back_project((100, 200), 2.0, maps)
    assert p == rf.Point3(2.0 * (100 - 319.5) / 500.0, 2.0 * (200 - 239.5) / 520.0, 2.0)
    x, y = rf.project_point(p, intr)
    assert abs(x - 100) < 1e-9 and abs(y - 200) < 1e-9
    img = rf.back_project_image(np.full((480, 640), 3.0), maps)
    assert img.shape == (480, 640, 3) and img[200, 100, 2] == 3.0
    sx, sy, sz = rf.noise_sigma(2.0, (100, 200), maps, rf.NoiseModel())
    assert sz == pytest.approx(1.425e-3 * 4.0) and sx == pytest.approx(sz * (100 - 319.5) / 500.0)
    (tmp_path / "cam.txt").write_text("# test camera\nfx=500\nfy=520\ncx=1.5\ncy=1.0\nwidth=4\nheight=3\n"
                                      "distortion=d.raw\n")
    np.concatenate([np.full(12, 0.25), np.full(12, -0.5)]).astype("<f8").tofile(tmp_path / "d.raw")
    c = rf.load_intrinsics(tmp_path / "cam.txt")
    assert c.width == 4 and c.delta_x[2, 3] == 0.25 and c.delta_y[0, 0] == -0.5
    with pytest.raises(ValueError, match="distortion_pixel"):
        rf.project_point(rf.Point3(0.1, 0.1, 1.0), c)
    ray = rf.ray_for_pixel(maps, (319, 239))
    assert rf.intersect_plane(ray, rf.GroundTruthPlane(np.array([0.0, 0.0, 1.0, -2.0]))) == pytest.approx(2.0)
    assert rf.intersect_plane(ray, rf.GroundTruthPlane(np.array([0.0, 0.0, 1.0, 2.0]))) is None


def test_naive_helpers_and_small_solvers():
    # the reference's known answers: diag(4,3,2,1) -> e4 with lambda 1 (tests/test_fitting_kernels.py:24-27)
    v, lam = rf.smallest_eigenvector(np.diag([4.0, 3.0, 2.0, 1.0]))
    assert lam == pytest.approx(1.0) and abs(abs(v[3]) - 1.0) < 1e-12
    a = np.array([[4.0, 1.0, 0.5], [1.0, 3.0, 0.2], [0.5, 0.2, 2.0]])
    b = np.array([1.0, -2.0, 0.5])
    np.testing.assert_allclose(rf.solve_spd3(a, b), np.linalg.solve(a, b), rtol=1e-12)
    with pytest.raises(rf.DegenerateFitError):
        rf.solve_spd3(np.ones((3, 3)), b)
    intr = rf.CameraIntrinsics(fx=20.0, fy=20.0, cx=3.5, cy=2.5, width=8, height=6)
    maps = _host_maps(intr)
    d = rf.DepthImage(values=np.full((6, 8), 2.0))
    smp = rf.gather_window_samples(d, maps, rf.Rect(1, 1, 5, 4), "implicit-standard")
    assert smp.shape == (12, 3) and np.all(smp[:, 2] == 2.0)
    sc = rf.accumulate_scatter_naive(smp, "implicit-standard")
    assert sc.n == 12 and sc.matrix[3, 3] == 12.0 and sc.matrix[2, 2] == 48.0
    sx = rf.accumulate_scatter_naive(rf.gather_window_samples(d, maps, rf.Rect(1, 1, 5, 4), "explicit-rgbd"),
                                     "explicit-rgbd")
    assert sx.target_sq == pytest.approx(12 * 0.25) and sx.rhs[2] == pytest.approx(6.0)
    with pytest.raises(rf.InsufficientSamplesError):
        rf.accumulate_scatter_naive(smp[:3], "implicit-rgbd")


def test_output_planes_are_checked_before_the_launch():
    """Caller-provided outputs must hold a [B, H, W] result (fit_pixels writes through raw
    pointers): wrong shapes, element types or devices raise instead of corrupting memory."""
    import torch

    from paper_2103_06644_b200.pixels import PixelFits

    cpu = torch.device("cpu")
    o = PixelFits.empty(2, 4, 5, cpu)
    o._c(2, 4, 5, cpu)
    with pytest.raises(ValueError):
        o._c(3, 4, 5, cpu)
    with pytest.raises(ValueError):
        PixelFits(o.normal, o.offset.double(), o.residual, o.curvature, o.status)._c(2, 4, 5, cpu)
    with pytest.raises(ValueError):
        PixelFits(o.normal[:, :, :, :2], o.offset, o.residual, o.curvature, o.status)._c(2, 4, 5, cpu)
    # a single frame may come without its batch dimension
    one = PixelFits.empty(1, 4, 5, cpu)
    PixelFits(*(getattr(one, k)[0] for k in ("normal", "offset", "residual", "curvature", "status")))._c(1, 4, 5, cpu)
