"""The device integral backend against the reference's own integral backend
(golden: tests/golden/make_golden.py:run_integral): channel tables bit for bit, assembled
scatter systems bit for bit, the fits of those systems within the parity tolerances, and
the hand-made systems (Jacobi fallback, rank-deficient explicit systems)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2103_06644_b200 as rf
from oracle.compare import normal_angles
from tests.helpers import GOLDEN_DIR

pytestmark = pytest.mark.gpu

CASES = ("integral_holes", "integral_full")
BUILDERS = {"std": rf.build_standard_implicit_channels, "rgbd": rf.build_rgbd_implicit_channels,
            "xstd": rf.build_standard_explicit_channels, "xrgbd": rf.build_rgbd_explicit_channels}
FORM_KEY = {"implicit-standard": "std", "implicit-rgbd": "rgbd", "explicit-standard": "xstd",
            "explicit-rgbd": "xrgbd"}


def _load(case):
    z = np.load(GOLDEN_DIR / f"{case}.npz")
    depth = z["depth"]
    H, W = depth.shape
    maps = rf.compute_tan_maps(rf.CameraIntrinsics(float(z["fx"]), float(z["fy"]), float(z["cx"]),
                                                   float(z["cy"]), W, H))
    return z, maps


def _stacks(z, maps, source):
    if source == "depthimage":
        d = rf.DepthImage(values=z["depth"].astype(np.float64))
    else:  # float32 device tensor (RF_DEPTH_F32_M)
        d = torch.from_numpy(z["depth"]).cuda()
    st = {k: b(d, maps) for k, b in BUILDERS.items()}
    st["const"] = rf.build_constant_channels(maps)
    return st


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("source", ["depthimage", "tensor_f32"])
def test_channel_tables_bit_exact(case, source):
    z, maps = _load(case)
    stacks = _stacks(z, maps, source)
    for key, st in stacks.items():
        names = [str(n) for n in z[f"{key}_names"]]
        assert list(st.channels) == names, key
        assert st.hole_corrected == bool(z[f"{key}_hole_corrected"]), key
        np.testing.assert_array_equal(st.count.table.cpu().numpy(), z[f"{key}_count"], err_msg=f"{key} count")
        for name in names:
            got = st.channels[name].table.cpu().numpy()
            np.testing.assert_array_equal(got, z[f"{key}_t_{name}"], err_msg=f"{key}/{name}")


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("form", list(rf.FORMULATIONS))
def test_scatter_and_fit_match_reference(case, form):
    z, maps = _load(case)
    stacks = _stacks(z, maps, "depthimage")
    key = FORM_KEY[form]
    explicit_fit = form.startswith("explicit")
    for k, r in enumerate(z["rects"]):
        n_ref = int(z[f"{key}_n"][k])
        if n_ref < 0:
            with pytest.raises(rf.InsufficientSamplesError):
                rf.scatter_from_integrals(stacks[key], stacks["const"], rf.Rect(*r), form)
            continue
        sc = rf.scatter_from_integrals(stacks[key], stacks["const"], rf.Rect(*r), form)
        assert sc.n == n_ref
        size = 3 if explicit_fit else 4
        np.testing.assert_array_equal(sc.matrix, z[f"{key}_mat"][k][:size, :size])
        if explicit_fit:
            np.testing.assert_array_equal(sc.rhs, z[f"{key}_rhs"][k])
            assert sc.target_sq == z[f"{key}_tq"][k]
        res = rf.FIT_BY_FORMULATION[form](sc)
        via_rect = rf.fit_rect(None, maps, rf.Rect(*r), form, backend="integral", stack=stacks[key],
                               constant=stacks["const"])
        np.testing.assert_array_equal(via_rect.plane.coefficients, res.plane.coefficients)
        assert res.degenerate == bool(z[f"{key}_deg"][k]), (k, r)
        if res.degenerate:
            continue
        ref_coef = z[f"{key}_coef"][k]
        got_coef = (rf.explicit_to_implicit(res.plane) if explicit_fit else res.plane).coefficients
        assert normal_angles(got_coef[None, :3], ref_coef[None, :3]).max() <= 1e-6, (k, r)
        assert abs(got_coef[3] - ref_coef[3]) <= 1e-6 * max(1.0, abs(ref_coef[3]))
        scale = float(np.linalg.norm(z[f"{key}_mat"][k][:size, :size])) / n_ref
        rms_ref = float(z[f"{key}_rms"][k])
        assert abs(res.rms_residual - rms_ref) <= 1e-4 * rms_ref + np.sqrt(1e-10 * scale), (k, r)
        if explicit_fit:
            np.testing.assert_allclose(res.plane.coefficients, z[f"{key}_xcoef"][k], rtol=1e-6, atol=1e-9)
        else:
            lam_ref = float(z[f"{key}_lam"][k])
            assert abs(res.eigenvalue - lam_ref) <= 1e-6 * abs(lam_ref) + 1e-11 * scale * n_ref


def test_explicit_rgbd_fitter_equals_scatter_path():
    z, maps = _load("integral_holes")
    stacks = _stacks(z, maps, "depthimage")
    fitter = rf.ExplicitRgbdFitter(stacks["const"])
    for r in z["rects"][:12]:
        try:
            a = fitter.fit(stacks["xrgbd"], rf.Rect(*r))
        except rf.InsufficientSamplesError:
            continue
        b = rf.fit_rect(None, maps, rf.Rect(*r), "explicit-rgbd", backend="integral", stack=stacks["xrgbd"],
                        constant=stacks["const"], rgbd_fitter=fitter)
        np.testing.assert_array_equal(a.plane.coefficients, b.plane.coefficients)


@pytest.mark.parametrize("form,key", [("implicit-standard", "sp_std"), ("implicit-rgbd", "sp_rgbd")])
def test_special_implicit_systems(form, key):
    z = np.load(GOLDEN_DIR / "integral_holes.npz")
    for k, m in enumerate(z["special4"]):
        res = rf.FIT_BY_FORMULATION[form](rf.Scatter4(matrix=m, n=4))
        np.testing.assert_allclose(res.plane.coefficients, z[f"{key}_coef"][k], atol=1e-9)
        assert abs(res.eigenvalue - z[f"{key}_lam"][k]) <= 1e-9 * max(1.0, abs(z[f"{key}_lam"][k]))
        assert res.degenerate == bool(z[f"{key}_deg"][k])


@pytest.mark.parametrize("form,key", [("explicit-standard", "sp_xstd"), ("explicit-rgbd", "sp_xrgbd")])
def test_special_explicit_systems(form, key):
    z = np.load(GOLDEN_DIR / "integral_holes.npz")
    for k in range(len(z["special3_mat"])):
        sc = rf.Scatter3(matrix=z["special3_mat"][k], rhs=z["special3_rhs"][k], n=4,
                         target_sq=float(z["special3_tq"][k]))
        res = rf.FIT_BY_FORMULATION[form](sc)
        assert res.degenerate == bool(z[f"{key}_deg"][k])
        np.testing.assert_allclose(res.plane.coefficients, z[f"{key}_coef"][k], rtol=1e-7, atol=1e-9)
        assert abs(res.rms_residual - z[f"{key}_rms"][k]) <= 1e-6


def test_build_integral_matches_numpy_cumsum():
    rng = np.random.default_rng(4)
    ch = rng.standard_normal((37, 53))
    mask = rng.random(ch.shape) > 0.3
    img = rf.build_integral(ch, mask, name="c")
    ref = np.zeros((38, 54))
    ref[1:, 1:] = np.cumsum(np.cumsum(np.where(mask, ch, 0.0), axis=0), axis=1)
    np.testing.assert_array_equal(img.table.cpu().numpy(), ref)
    r = rf.Rect(3, 4, 20, 30)
    t = ref
    assert rf.box_sum(img, r) == float(t[r.y1, r.x1] - t[r.y0, r.x1] - t[r.y1, r.x0] + t[r.y0, r.x0])
    with pytest.raises(ValueError):
        rf.box_sum(img, rf.Rect(0, 0, 54, 10))


def test_batched_scatter_fits_equal_single_fits():
    z, maps = _load("integral_full")
    key, form = "std", "implicit-standard"
    ok = z[f"{key}_n"] >= 4
    mats = z[f"{key}_mat"][ok]
    rows = rf.fit_scatters(mats, z[f"{key}_n"][ok], form)
    for i, m in enumerate(mats):
        single = rf.fit_implicit_standard(rf.Scatter4(matrix=m, n=int(z[f"{key}_n"][ok][i])))
        np.testing.assert_array_equal(rf.ImplicitPlane(rows["coef"][i]).coefficients, single.plane.coefficients)


def test_tan_lattices_match_the_reference_formula():
    z, maps = _load("integral_full")
    H, W = z["depth"].shape
    tx = (np.arange(W, dtype=np.float64)[None, :] + np.zeros((H, W)) - float(z["cx"])) / float(z["fx"])
    ty = (np.arange(H, dtype=np.float64)[:, None] + np.zeros((H, W)) - float(z["cy"])) / float(z["fy"])
    np.testing.assert_array_equal(maps.tan_x, tx)
    np.testing.assert_array_equal(maps.tan_y, ty)
    # the device tables hold the same values: the constant tan_x table's first data row
    # is the running sum of row 0 of the lattice
    const = rf.build_constant_channels(maps)
    np.testing.assert_array_equal(const.channels["tx"].table.cpu().numpy()[1, 1:], np.cumsum(tx[0]))


def test_reference_timing_harness():
    """run_bench's rows, CSV schema and ratios (bench.py:86-341) on the device paths."""
    cfg = rf.BenchConfig(width=96, height=64, tile=20, plane_counts=(0, 1, 7), repetitions=3, warmup=1)
    rep = rf.run_bench(cfg)
    csv = rep.to_csv().splitlines()
    assert csv[0] == "method,backend,phase,plane_count,rep,seconds"
    # per rep x formulation x backend: build + total(0) + (fit + total) per non-zero count
    assert len(csv) - 1 == 3 * 4 * 2 * (2 + 2 * 2)
    assert rep.median_seconds("implicit-rgbd", "integral", "fit", 7) > 0
    assert rep.build_ratio("implicit") > 0 and rep.per_fit_ratio("explicit") > 0
    assert len(rep.workload_digest) == 64 and "build ratio" in rep.summary()
    for f in rf.FORMULATIONS:
        assert rf.op_count_audit(f).per_frame_channels == {"implicit-standard": 9, "implicit-rgbd": 4,
                                                           "explicit-standard": 8, "explicit-rgbd": 3}[f]
    with pytest.raises(ValueError):
        rf.BenchConfig(repetitions=2)
