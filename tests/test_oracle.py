"""The oracle (C restatement in oracle/) pinned against the reference itself:
the golden per-pixel fixtures made by tests/golden/make_golden.py from the
reference's own fit pipeline, plus the reference's known-answer tests for the
hot path (tests/test_fitting.py, tests/test_fitting_kernels.py)."""

from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import oracle as O
from oracle.compare import compare, normal_angles
from tests.helpers import GOLDEN_CASES, golden_mask, load_golden, oracle_frame


@pytest.mark.parametrize("case", GOLDEN_CASES)
@pytest.mark.parametrize("form", ["implicit-rgbd", "implicit-standard", "explicit-rgbd", "explicit-standard"])
def test_oracle_matches_reference_golden(case, form):
    g = load_golden(case)
    ref = g[form]
    mask = golden_mask(g)
    got = O.fit_pixels(*(_vals(g, mask)), *O.tan_maps(g["cam"].fx, g["cam"].fy, g["cam"].cx, g["cam"].cy,
                                                      g["cam"].width, g["cam"].height,
                                                      g["cam"].delta_x, g["cam"].delta_y),
                       g["window"], form, want_coef=True)
    # status: bit-exact (including the degenerate bit: same algorithm)
    np.testing.assert_array_equal(got["status"], ref["status"])
    fit = (ref["status"] & 2) != 0
    ok = fit & ((ref["status"] & 4) == 0)
    ang = normal_angles(got["coef"][ok, :3], ref["coef"][ok, :3])
    assert ang.max(initial=0) <= 1e-6, ang.max()
    # full canonical 4-vectors (sign convention included)
    assert np.abs(got["coef"][ok] - ref["coef"][ok]).max(initial=0) <= 1e-6
    # implicit: the smallest eigenvalue, rounding level ~eps*||S||_F; explicit: the residual
    # sum of squares sum(b^2) - alpha.rhs, whose aggregated-sum cancellation floor the
    # reference itself documents (fitting.py:592-595)
    explicit_fit = form.startswith("explicit")
    lam_floor = (1e-10 if explicit_fit else 1e-11) * ref["scale"][ok] * ref["n"][ok]
    lam_err = np.abs(got["lam"][ok] - ref["lam"][ok]) / np.maximum(np.abs(ref["lam"][ok]), lam_floor)
    assert lam_err.max(initial=0) <= (1e-4 if explicit_fit else 1e-5)
    m = compare(got, ref, explicit_fit=explicit_fit)
    assert m["ok"], m


def _vals(g, mask):
    if g["dtype"] == "u16":
        v, valid = O.depth_from_millimeters(g["depth"])
        if mask is not None:
            valid = valid & mask.astype(bool)
    else:
        v, valid = O.depth_from_meters(g["depth"], mask)
    return v, valid


def test_golden_frontal_plane_coefficients():
    """tests/test_fitting.py:266-281: Z = 3 frontal plane -> (0, 0, 1, -3)/sqrt(10)."""
    g = load_golden("frontal_z3_w5")
    expected = np.array([0.0, 0.0, 1.0, -3.0]) / math.sqrt(10.0)
    for form in ("implicit-rgbd", "implicit-standard"):
        ref = g[form]
        fit = (ref["status"] & 2) != 0
        assert fit.all()
        np.testing.assert_allclose(ref["coef"][fit], np.broadcast_to(expected, ref["coef"][fit].shape), atol=1e-9)
        got = oracle_frame(g["depth"], g["cam"], g["window"], form)
        np.testing.assert_allclose(got["normal"], np.broadcast_to([0, 0, 1.0], got["normal"].shape), atol=1e-6)
        np.testing.assert_allclose(got["offset"], -3.0, rtol=1e-6)


class TestKnownAnswers:
    """Restated reference unit tests for the dense kernels."""

    def test_jacobi_diag(self):
        # tests/test_fitting_kernels.py:24-27: diag(4,3,2,1) -> smallest e4, lambda 1
        vals, vecs, ok = O.jacobi_eigh(np.diag([4.0, 3.0, 2.0, 1.0]))
        assert ok
        i = int(np.argmin(vals))
        assert vals[i] == 1.0
        np.testing.assert_allclose(np.abs(vecs[:, i]), [0, 0, 0, 1.0])

    def test_jacobi_matches_eigvalsh(self):
        # tests/test_fitting_kernels.py:43-53
        rng = np.random.default_rng(0)
        for _ in range(50):
            a = rng.standard_normal((4, 4))
            m = a @ a.T
            vals, _, ok = O.jacobi_eigh(m)
            assert ok
            np.testing.assert_allclose(np.sort(vals), np.linalg.eigvalsh(m), rtol=1e-10, atol=1e-12)

    def test_zero_matrix(self):
        vals, vecs, ok = O.jacobi_eigh(np.zeros((4, 4)))
        assert ok and not vals.any()
        np.testing.assert_array_equal(vecs, np.eye(4))

    @pytest.mark.parametrize("coef,expected", [
        ([0.0, 0.0, 2.0, -6.0], [0, 0, 1.0, -3.0]),   # tests/test_fitting.py:100-102
        ([0.0, 0.0, -1.0, 3.0], [0, 0, 1.0, -3.0]),   # :104-106
        ([-1.0, 0.0, 0.0, 1.0], [1.0, 0, 0, -1.0]),   # :108-111
        ([0.0, 0.0, 0.0, -4.0], [0, 0, 0, 1.0]),      # :114-115
    ])
    def test_canonicalisation(self, coef, expected):
        """canonicalize_implicit (fitting.py:76-94) through _fit_implicit on a rank-3 scatter
        whose null vector is `coef`."""
        v = np.asarray(coef, float)
        v /= np.linalg.norm(v)
        basis = np.linalg.svd(v.reshape(1, 4))[2][1:]
        S = basis.T @ np.diag([3.0, 2.0, 1.0]) @ basis
        out = O.fit_scatter(S, 10, "implicit-standard")
        e = np.asarray(expected, float)
        np.testing.assert_allclose(out["coef"], e / np.linalg.norm(e), atol=1e-12)

    def test_collinear_samples_degenerate(self):
        # tests/test_fitting.py:416-420
        t = np.linspace(0.0, 1.0, 30)
        m = np.column_stack((t, np.zeros_like(t), np.full_like(t, 2.0), np.ones_like(t)))
        out = O.fit_scatter(m.T @ m, 30, "implicit-standard")
        assert out["degenerate"]

    def test_rms_identity(self):
        # tests/test_fitting.py:396-412: rms^2 * n == lambda
        rng = np.random.default_rng(6)
        pts = rng.standard_normal((40, 3)) * [1.0, 1.0, 0.01] + [0, 0, 2.0]
        m = np.column_stack((pts, np.ones(40)))
        out = O.fit_scatter(m.T @ m, 40, "implicit-standard")
        assert out["rms"] ** 2 * 40 == pytest.approx(out["lam"], rel=1e-9)


def test_integral_backend_matches_naive_on_golden():
    """The restated integral backend (the reference's fast path, timed as the CPU
    baseline) agrees with the naive one (fitting.py:420-533 vs :339-402)."""
    g = load_golden("planes_f32_w5")
    tx, ty = O.tan_maps(g["cam"].fx, g["cam"].fy, g["cam"].cx, g["cam"].cy, g["cam"].width, g["cam"].height)
    v, valid = O.depth_from_meters(g["depth"])
    for form in ("implicit-rgbd", "implicit-standard"):
        a = O.fit_pixels(v, valid, tx, ty, 5, form, backend=O.NAIVE, want_coef=True)
        b = O.fit_pixels(v, valid, tx, ty, 5, form, backend=O.INTEGRAL, want_coef=True)
        np.testing.assert_array_equal(a["status"] & 3, b["status"] & 3)
        fit = (a["status"] & 2) != 0
        assert np.abs(a["coef"][fit] - b["coef"][fit]).max() <= 1e-6


def test_threaded_equals_single_thread():
    g = load_golden("planes_f32_w3")
    tx, ty = O.tan_maps(g["cam"].fx, g["cam"].fy, g["cam"].cx, g["cam"].cy, g["cam"].width, g["cam"].height)
    v, valid = O.depth_from_meters(g["depth"])
    a = O.fit_pixels(v, valid, tx, ty, 3, "implicit-rgbd", nthreads=1, want_coef=True)
    b = O.fit_pixels(v, valid, tx, ty, 3, "implicit-rgbd", nthreads=4, want_coef=True)
    np.testing.assert_array_equal(a["status"], b["status"])
    np.testing.assert_array_equal(np.nan_to_num(a["coef"]), np.nan_to_num(b["coef"]))


def test_pixel_subset_matches_full_frame():
    g = load_golden("planes_f32_w5")
    tx, ty = O.tan_maps(g["cam"].fx, g["cam"].fy, g["cam"].cx, g["cam"].cy, g["cam"].width, g["cam"].height)
    v, valid = O.depth_from_meters(g["depth"])
    full = O.fit_pixels(v, valid, tx, ty, 5, "implicit-standard")
    pix = np.array([0, 5, 63, 64, 1000, 3071])
    sub = O.fit_pixels(v, valid, tx, ty, 5, "implicit-standard", pixels=pix)
    np.testing.assert_array_equal(sub["status"], full["status"][pix])
    np.testing.assert_array_equal(np.nan_to_num(sub["normal"]), np.nan_to_num(full["normal"][pix]))


@pytest.mark.parametrize("form", ["implicit-rgbd", "implicit-standard", "explicit-rgbd", "explicit-standard"])
def test_oracle_rects_match_reference(form):
    """rfo_fit_rects vs the reference's fit_rect (naive) on random rects incl. the whole frame."""
    from tests.helpers import load_golden_rects

    g = load_golden_rects()
    ref = g[form]
    tx, ty = O.tan_maps(g["cam"].fx, g["cam"].fy, g["cam"].cx, g["cam"].cy, g["cam"].width, g["cam"].height)
    v, valid = O.depth_from_meters(g["depth"])
    got = O.fit_rects(v, valid, tx, ty, g["rects"], form)
    np.testing.assert_array_equal(got["status"], ref["status"])
    np.testing.assert_array_equal(got["n"], ref["n"])
    ok = (ref["status"] & 2) != 0
    assert np.abs(got["coef"][ok] - ref["coef"][ok]).max() <= 1e-6
    np.testing.assert_allclose(got["rms"][ok], ref["rms"][ok], rtol=1e-5,
                               atol=float(np.sqrt(1e-10 * np.nanmax(ref["scale"]))))


def test_tan_maps_known_answers():
    """The reference's camera known-answer tests (tests/test_camera.py:27-40)."""
    tx, _ = O.tan_maps(500.0, 500.0, 320.0, 240.0, 1024, 480)
    assert tx[0, 820] == 1.0  # one focal length right of cx
    dx = np.full((480, 640), 0.25)
    tx, ty = O.tan_maps(525.0, 525.0, 319.5, 239.5, 640, 480, dx)
    assert tx[7, 100] == pytest.approx(-0.4176190476190476, rel=1e-15)
    assert ty[240, 3] == pytest.approx((240 - 239.5) / 525.0, rel=1e-15)
