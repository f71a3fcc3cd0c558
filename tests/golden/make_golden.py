"""Generate the golden per-pixel fixtures from the REFERENCE itself.

Run in the build container (the reference is importable there, read-only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

For every pixel of each small case this calls the reference's own per-window
pipeline on the clipped centred window:

    gather_window_samples + accumulate_scatter_naive   (fitting.py:339-402)
    FIT_BY_FORMULATION[formulation](scatter)            (fitting.py:546-579)

i.e. exactly ``fit_rect(depth, maps, rect, formulation, "naive")``
(fitting.py:757-786), and records the canonical coefficients, eigenvalue,
rms residual, degenerate flag and sample count.  Curvature is the A17
extension computed from the reference's own Scatter4 with numpy eigvalsh.
Inputs are rendered with the reference's renderer (synth.render_scene) and
stored as float32 (or uint16 mm) so the GPU later reads the same bits.
The reference is never needed at test time: the .npz files are committed.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

try:
    import rangefit as rf
except ImportError:  # pragma: no cover
    sys.path.insert(0, "/root/reference/pkg/src")
    import rangefit as rf

from rangefit.fitting import (FIT_BY_FORMULATION, ExplicitPlane, accumulate_scatter_naive,
                              explicit_to_implicit, gather_window_samples)

FORMS = ("implicit-rgbd", "implicit-standard", "explicit-rgbd", "explicit-standard")
KEYS = {"implicit-rgbd": "rgbd", "implicit-standard": "std", "explicit-rgbd": "xrgbd",
        "explicit-standard": "xstd"}
SPACE = {"implicit-rgbd": "implicit-rgbd", "explicit-rgbd": "implicit-rgbd",
         "implicit-standard": "implicit-standard", "explicit-standard": "implicit-standard"}


def curvature(matrix: np.ndarray, formulation: str) -> float:
    if SPACE[formulation] == "implicit-standard":
        I, k = [0, 1, 2], 3
    else:
        I, k = [0, 1, 3], 2
    S = matrix
    C3 = S[np.ix_(I, I)] - np.outer(S[I, k], S[I, k]) / S[k, k]
    ev = np.linalg.eigvalsh(C3)
    tr = float(np.trace(C3))
    return float(ev.min() / tr) if tr > 0 else 0.0


def implicit_scatter(samples: np.ndarray, formulation: str) -> np.ndarray:
    """The space's implicit 4x4 scatter (fitting.py:364-369) without the MIN_SAMPLES
    check, so explicit fits with n = 3 still get a curvature."""
    u, v, z = samples[:, 0], samples[:, 1], samples[:, 2]
    one = np.ones_like(z)
    m = np.column_stack((u, v, z, one)) if SPACE[formulation] == "implicit-standard" \
        else np.column_stack((u, v, one, 1.0 / z))
    g = m.T @ m
    return (g + g.T) * 0.5


def run_case(name, cam, depth_img: "rf.DepthImage", stored, window, dtype):
    maps = rf.compute_tan_maps(cam)
    H, W = cam.height, cam.width
    r = window // 2
    out = {"depth": stored, "fx": cam.fx, "fy": cam.fy, "cx": cam.cx, "cy": cam.cy,
           "window": window, "dtype": dtype}
    if np.any(cam.delta_x != 0) or np.any(cam.delta_y != 0):
        out["delta_x"], out["delta_y"] = cam.delta_x, cam.delta_y
    if depth_img.valid is not None:
        out["valid"] = depth_img.valid.astype(np.uint8)
    for form in FORMS:
        coef = np.full((H * W, 4), np.nan)
        lam = np.full(H * W, np.nan)
        rms = np.full(H * W, np.nan)
        curv = np.full(H * W, np.nan)
        npts = np.zeros(H * W, np.int32)
        status = np.zeros(H * W, np.uint8)
        fro = np.full(H * W, np.nan)
        for y in range(H):
            for x in range(W):
                i = y * W + x
                if not depth_img.valid[y, x]:
                    continue
                status[i] = 1
                rect = rf.Rect(max(x - r, 0), max(y - r, 0), min(x + r + 1, W), min(y + r + 1, H))
                samples = gather_window_samples(depth_img, maps, rect, form)
                try:
                    scatter = accumulate_scatter_naive(samples, form)
                except rf.InsufficientSamplesError:
                    continue
                res = FIT_BY_FORMULATION[form](scatter)
                status[i] |= 2 | (4 if res.degenerate else 0)
                if isinstance(res.plane, ExplicitPlane):
                    coef[i] = explicit_to_implicit(res.plane).coefficients   # fitting.py:729-739
                    lam[i] = res.rms_residual ** 2 * res.n_points
                else:
                    coef[i] = res.plane.coefficients
                    lam[i] = res.eigenvalue
                rms[i] = res.rms_residual
                npts[i] = res.n_points
                # curvature (A17) and the rounding scale come from the space's implicit scatter
                s4 = scatter.matrix if SPACE[form] == form else implicit_scatter(samples, form)
                curv[i] = curvature(s4, form)
                fro[i] = float(np.linalg.norm(s4)) / res.n_points
        key = KEYS[form]
        out.update({f"{key}_coef": coef, f"{key}_lam": lam, f"{key}_rms": rms, f"{key}_curv": curv,
                    f"{key}_n": npts, f"{key}_status": status, f"{key}_scale": fro})
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, "fits:", {k: int((out[f"{k}_status"] & 2).sum()) for k in KEYS.values()})


def random_plane(rng, zlo, zhi):
    while True:
        n = rng.standard_normal(3)
        n /= np.linalg.norm(n)
        if n[2] > 0:
            n = -n
        if -n[2] > 0.45:
            break
    z0 = rng.uniform(zlo, zhi)
    return rf.GroundTruthPlane(np.array([*n, -n[2] * z0]))


def run_rects(name, cam, depth_img, stored, dtype, rng, count=60):
    """Reference fit_rect (naive backend) on random rects, incl. frame-sized and tiny ones."""
    maps = rf.compute_tan_maps(cam)
    W, H = cam.width, cam.height
    rects = [(0, 0, W, H), (0, 0, 2, 2), (W - 3, H - 1, W, H)]
    while len(rects) < count:
        x0, y0 = int(rng.integers(0, W - 1)), int(rng.integers(0, H - 1))
        rects.append((x0, y0, int(rng.integers(x0 + 1, W + 1)), int(rng.integers(y0 + 1, H + 1))))
    out = {"depth": stored, "fx": cam.fx, "fy": cam.fy, "cx": cam.cx, "cy": cam.cy, "dtype": dtype,
           "rects": np.array(rects, np.int32)}
    for form in FORMS:
        coef = np.full((len(rects), 4), np.nan)
        xcoef = np.full((len(rects), 3), np.nan)
        rms = np.full(len(rects), np.nan)
        lam = np.full(len(rects), np.nan)
        curv = np.full(len(rects), np.nan)
        npts = np.zeros(len(rects), np.int32)
        status = np.zeros(len(rects), np.int32)
        scale = np.full(len(rects), np.nan)
        for k, (x0, y0, x1, y1) in enumerate(rects):
            samples = gather_window_samples(depth_img, maps, rf.Rect(x0, y0, x1, y1), form)
            npts[k] = samples.shape[0]
            try:
                res = rf.fit_rect(depth_img, maps, rf.Rect(x0, y0, x1, y1), form, "naive")
            except rf.InsufficientSamplesError:
                continue
            status[k] = 2 | (4 if res.degenerate else 0)
            if isinstance(res.plane, ExplicitPlane):
                coef[k] = explicit_to_implicit(res.plane).coefficients
                xcoef[k] = res.plane.coefficients
                lam[k] = res.rms_residual ** 2 * res.n_points
            else:
                coef[k] = res.plane.coefficients
                lam[k] = res.eigenvalue
            rms[k] = res.rms_residual
            s4 = implicit_scatter(samples, form)
            curv[k] = curvature(s4, form)
            scale[k] = float(np.linalg.norm(s4)) / res.n_points
        key = KEYS[form]
        out.update({f"{key}_coef": coef, f"{key}_xcoef": xcoef, f"{key}_rms": rms, f"{key}_lam": lam,
                    f"{key}_curv": curv, f"{key}_n": npts, f"{key}_status": status, f"{key}_scale": scale})
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, "rects:", len(rects))


def run_segment(name, cam, depth_img, stored, formulations=FORMS, backend="naive", metric="rms"):
    """Reference quadtree segmentation (segment.py:327-431) with the given backend and error
    metric."""
    from rangefit.segment import SegConfig, segment

    maps = rf.compute_tan_maps(cam)
    out = {"depth": stored, "fx": cam.fx, "fy": cam.fy, "cx": cam.cx, "cy": cam.cy,
           "backend": backend, "metric": metric}
    thresholds = {"implicit-rgbd": 3e-3, "implicit-standard": 3e-2, "explicit-rgbd": 4e-3,
                  "explicit-standard": 6e-2} if metric == "max" else {}
    for form in formulations:
        cfg = SegConfig(formulation=form, backend=backend, initial_tile=32, max_depth=3, k=6, seed=3,
                        error_metric=metric, rms_threshold=thresholds.get(form))
        seg = segment(depth_img, maps, cfg)
        key = KEYS[form]
        out[f"{key}_rects"] = np.array([tuple(t.rect) for t in seg.tiles], np.int32)
        out[f"{key}_status"] = np.array([t.status.value for t in seg.tiles])
        out[f"{key}_cluster"] = np.array([t.cluster for t in seg.tiles], np.int32)
        out[f"{key}_labels"] = seg.labels
        out[f"{key}_threshold"] = cfg.threshold
        print(name, form, "tiles", len(seg.tiles), "fitted", seg.n_fitted)
    np.savez_compressed(HERE / f"{name}.npz", **out)


def run_integral(name, cam, depth_img, stored, rng, count=40):
    """The reference's integral backend (integral.py:136-325, fitting.py:405-739): every
    channel table of the five stacks, scatter_from_integrals + FIT_BY_FORMULATION on random
    rects, and fit_implicit_* / fit_explicit_* on hand-made systems (Jacobi fallback,
    rank-deficient explicit systems)."""
    from rangefit.fitting import (Scatter3, Scatter4, fit_explicit_rgbd, fit_explicit_standard,
                                  fit_implicit_rgbd, fit_implicit_standard, scatter_from_integrals)
    from rangefit.integral import (build_constant_channels, build_rgbd_explicit_channels,
                                   build_rgbd_implicit_channels, build_standard_explicit_channels,
                                   build_standard_implicit_channels)

    maps = rf.compute_tan_maps(cam)
    W, H = cam.width, cam.height
    out = {"depth": stored, "valid": depth_img.valid, "fx": cam.fx, "fy": cam.fy, "cx": cam.cx, "cy": cam.cy}
    stacks = {"const": build_constant_channels(maps),
              "std": build_standard_implicit_channels(depth_img, maps),
              "rgbd": build_rgbd_implicit_channels(depth_img, maps),
              "xstd": build_standard_explicit_channels(depth_img, maps),
              "xrgbd": build_rgbd_explicit_channels(depth_img, maps)}
    for key, st in stacks.items():
        out[f"{key}_count"] = st.count.table
        out[f"{key}_names"] = np.array(list(st.channels))
        out[f"{key}_hole_corrected"] = st.hole_corrected
        for cname, img in st.channels.items():
            out[f"{key}_t_{cname}"] = img.table
    rects = [(0, 0, W, H), (0, 0, 2, 2), (W - 3, H - 1, W, H), (3, 3, 3, 9)]
    while len(rects) < count:
        x0, y0 = int(rng.integers(0, W - 1)), int(rng.integers(0, H - 1))
        rects.append((x0, y0, int(rng.integers(x0 + 1, min(W, x0 + 12) + 1)),
                      int(rng.integers(y0 + 1, min(H, y0 + 12) + 1))))
    out["rects"] = np.array(rects, np.int32)
    for form in FORMS:
        key = KEYS[form]
        st = stacks[key]
        n_r = len(rects)
        mats = np.full((n_r, 4, 4), np.nan)
        rhs = np.full((n_r, 3), np.nan)
        tq = np.full(n_r, np.nan)
        npts = np.full(n_r, -1, np.int64)
        coef = np.full((n_r, 4), np.nan)
        xcoef = np.full((n_r, 3), np.nan)
        lam = np.full(n_r, np.nan)
        rms = np.full(n_r, np.nan)
        deg = np.zeros(n_r, bool)
        for k, r in enumerate(rects):
            try:
                sc = scatter_from_integrals(st, stacks["const"], rf.Rect(*r), form)
            except rf.InsufficientSamplesError:
                continue
            npts[k] = sc.n
            m = np.asarray(sc.matrix)
            mats[k, :m.shape[0], :m.shape[1]] = m
            if isinstance(sc, Scatter3):
                rhs[k] = sc.rhs
                tq[k] = np.nan if sc.target_sq is None else sc.target_sq
            res = FIT_BY_FORMULATION[form](sc)
            deg[k] = res.degenerate
            rms[k] = np.nan if res.rms_residual is None else res.rms_residual
            if isinstance(res.plane, ExplicitPlane):
                xcoef[k] = res.plane.coefficients
                coef[k] = explicit_to_implicit(res.plane).coefficients
            else:
                coef[k] = res.plane.coefficients
                lam[k] = res.eigenvalue
        out.update({f"{key}_mat": mats, f"{key}_rhs": rhs, f"{key}_tq": tq, f"{key}_n": npts,
                    f"{key}_coef": coef, f"{key}_xcoef": xcoef, f"{key}_lam": lam, f"{key}_rms": rms,
                    f"{key}_deg": deg})
    # hand-made systems: a known answer (diag(4,3,2,1) -> e4, lam 1), a zero constant-monomial
    # entry (Jacobi path), collinear explicit samples (pinv path, degenerate)
    special4 = [np.diag([4.0, 3.0, 2.0, 1.0]), np.diag([1.0, 2.0, 3.0, 0.0]),
                np.array([[5.0, 1.0, 0.5, 2.0], [1.0, 4.0, 0.2, 1.0], [0.5, 0.2, 3.0, 0.5], [2.0, 1.0, 0.5, 6.0]])]
    for key, fit in (("sp_std", fit_implicit_standard), ("sp_rgbd", fit_implicit_rgbd)):
        c, l, d = [], [], []
        for m in special4:
            res = fit(Scatter4(matrix=m, n=4))
            c.append(res.plane.coefficients)
            l.append(res.eigenvalue)
            d.append(res.degenerate)
        out[f"{key}_coef"], out[f"{key}_lam"], out[f"{key}_deg"] = np.array(c), np.array(l), np.array(d)
    out["special4"] = np.array(special4)
    xs = np.array([0.0, 1.0, 2.0, 3.0])
    ys = 2.0 * xs + 1.0                   # collinear samples: rank-deficient normal equations
    zs = 0.5 * xs - 0.25 * ys + 2.0
    m = np.column_stack((xs, ys, np.ones_like(xs)))
    special3 = [(m.T @ m, m.T @ zs, float(zs @ zs))]
    m2 = np.column_stack((xs, xs ** 2, np.ones_like(xs)))
    special3.append((m2.T @ m2, m2.T @ zs, float(zs @ zs)))
    for key, fit in (("sp_xstd", fit_explicit_standard), ("sp_xrgbd", fit_explicit_rgbd)):
        c, d, r = [], [], []
        for (a, b, t) in special3:
            res = fit(Scatter3(matrix=a, rhs=b, n=4, target_sq=t))
            c.append(res.plane.coefficients)
            d.append(res.degenerate)
            r.append(res.rms_residual)
        out[f"{key}_coef"], out[f"{key}_deg"], out[f"{key}_rms"] = np.array(c), np.array(d), np.array(r)
    out["special3_mat"] = np.array([a for a, _, _ in special3])
    out["special3_rhs"] = np.array([b for _, b, _ in special3])
    out["special3_tq"] = np.array([t for _, _, t in special3])
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, "rects:", len(rects))


def run_render(name):
    """The reference renderer (synth.py:137-194) on small scenes: nearest hit with mask rects,
    quadratic noise, dropout, per-row seeded streams; plus the interchange files it writes
    (imageio.py:47-139, synth.py:224-246)."""
    from rangefit import imageio as rio
    from rangefit.synth import write_depth

    cam = rf.CameraIntrinsics(fx=50.0, fy=52.0, cx=19.5, cy=14.5, width=40, height=30)
    maps = rf.compute_tan_maps(cam)
    planes = (rf.GroundTruthPlane(np.array([0.1, -0.2, -1.0, 2.5])),
              rf.GroundTruthPlane(np.array([-0.3, 0.1, -1.0, 1.8]), mask_rect=(5, 3, 30, 20)),
              rf.GroundTruthPlane(np.array([0.0, 0.0, -1.0, 1.2]), mask_rect=(-10, 22, 12, 40)),
              rf.GroundTruthPlane(np.array([0.9, 0.0, 0.1, 0.5])))
    scene = rf.SyntheticScene(planes)
    out = {"fx": cam.fx, "fy": cam.fy, "cx": cam.cx, "cy": cam.cy, "width": cam.width, "height": cam.height,
           "planes": np.stack([p.coefficients for p in planes]),
           "rects": np.array([p.mask_rect if p.mask_rect is not None else (-1, -1, -1, -1) for p in planes])}
    cases = {"plain": dict(noise=None, seed=0, dropout=0.0),
             "noise": dict(noise=rf.NoiseModel(), seed=7, dropout=0.0),
             "drop": dict(noise=None, seed=3, dropout=0.2),
             "both": dict(noise=rf.NoiseModel(slope_coefficient=0.02), seed=11, dropout=0.1)}
    for key, kw in cases.items():
        d, labels = rf.render_scene(scene, maps, **kw)
        out[f"{key}_depth"], out[f"{key}_valid"], out[f"{key}_labels"] = d.values, d.valid, labels
        out[f"{key}_noise"] = 0.0 if kw["noise"] is None else kw["noise"].slope_coefficient
        out[f"{key}_seed"], out[f"{key}_dropout"] = kw["seed"], kw["dropout"]
    d, _ = rf.render_scene(scene, maps, noise=rf.NoiseModel(), seed=7)
    write_depth(HERE / "io_depth.pgm", d)
    write_depth(HERE / "io_depth.rf64", d)
    rio.write_pgm8(HERE / "io_labels.pgm", out["plain_labels"])
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, "render cases:", len(cases))


def main():
    # 1. noisy three-plane scene, 10% dropout, float32 metres (small_camera of the reference tests)
    cam = rf.CameraIntrinsics(fx=60.0, fy=60.0, cx=31.5, cy=23.5, width=64, height=48)
    maps = rf.compute_tan_maps(cam)
    rng = np.random.default_rng(11)
    scene = rf.SyntheticScene(tuple(random_plane(rng, 1.0, 4.0) for _ in range(3)))
    d, _ = rf.render_scene(scene, maps, noise=rf.NoiseModel(), seed=3, dropout=0.1)
    z32 = np.where(d.valid, d.values, 0.0).astype(np.float32)
    for w in (3, 5):
        run_case(f"planes_f32_w{w}", cam, rf.DepthImage(values=z32.astype(np.float64)), z32, w, "f32")

    run_rects("rects_planes_f32", cam, rf.DepthImage(values=z32.astype(np.float64)), z32, "f32",
              np.random.default_rng(21))

    run_render("render_planes")


    # integral backend: a holey frame (hole-corrected rgbd stacks) and a hole-free crop
    cam_i = rf.CameraIntrinsics(fx=60.0, fy=60.0, cx=15.5, cy=11.5, width=32, height=24)
    z_i = z32[12:36, 16:48].copy()
    run_integral("integral_holes", cam_i, rf.DepthImage(values=z_i.astype(np.float64)), z_i,
                 np.random.default_rng(31))
    d_f, _ = rf.render_scene(scene, rf.compute_tan_maps(cam_i), noise=rf.NoiseModel(), seed=6)
    z_f = np.where(d_f.valid, d_f.values, 1.5).astype(np.float32)
    run_integral("integral_full", cam_i, rf.DepthImage(values=z_f.astype(np.float64)), z_f,
                 np.random.default_rng(32))

    # quadtree segmentation of a Voronoi-like multi-plane frame
    cam_s = rf.CameraIntrinsics(fx=120.0, fy=120.0, cx=63.5, cy=47.5, width=128, height=96)
    maps_s = rf.compute_tan_maps(cam_s)
    planes = []
    for (x0, y0, x1, y1) in ((0, 0, 64, 48), (64, 0, 128, 48), (0, 48, 70, 96), (70, 48, 128, 96)):
        p = random_plane(rng, 1.0, 3.5)
        planes.append(rf.GroundTruthPlane(p.coefficients, mask_rect=(x0, y0, x1, y1)))
    d_s, _ = rf.render_scene(rf.SyntheticScene(tuple(planes)), maps_s, noise=rf.NoiseModel(), seed=8,
                             dropout=0.03)
    z_s = np.where(d_s.valid, d_s.values, 0.0).astype(np.float32)
    run_segment("segment_planes", cam_s, rf.DepthImage(values=z_s.astype(np.float64)), z_s)
    run_segment("segment_planes_integral", cam_s, rf.DepthImage(values=z_s.astype(np.float64)), z_s,
                backend="integral")
    run_segment("segment_planes_max", cam_s, rf.DepthImage(values=z_s.astype(np.float64)), z_s, metric="max")

    # 1b. explicit validity mask: DepthImage(values, valid=mask) (synth.py:88-94)
    mask = np.random.default_rng(5).random(z32.shape) > 0.2
    dm = rf.DepthImage(values=z32.astype(np.float64), valid=mask)
    run_case("planes_f32_mask_w5", cam, dm, z32, 5, "f32")

    # 2. uint16 millimetres through DepthImage.from_millimeters
    cam2 = rf.CameraIntrinsics(fx=40.0, fy=42.0, cx=15.5, cy=11.5, width=32, height=24)
    maps2 = rf.compute_tan_maps(cam2)
    scene2 = rf.SyntheticScene((random_plane(rng, 0.6, 3.0), random_plane(rng, 0.6, 3.0)))
    d2, _ = rf.render_scene(scene2, maps2, noise=rf.NoiseModel(), seed=4, dropout=0.05)
    mm = d2.to_millimeters()
    run_case("planes_u16_w5", cam2, rf.DepthImage.from_millimeters(mm), mm, 5, "u16")

    # 3. noiseless frontal plane Z = 3 (tests/test_fitting.py:266-281 golden (0,0,1,-3)/sqrt(10))
    cam3 = rf.CameraIntrinsics(fx=60.0, fy=60.0, cx=7.5, cy=5.5, width=16, height=12)
    maps3 = rf.compute_tan_maps(cam3)
    d3, _ = rf.render_scene(rf.SyntheticScene((rf.GroundTruthPlane(np.array([0.0, 0.0, 1.0, -3.0])),)), maps3)
    z3 = d3.values.astype(np.float32)
    run_case("frontal_z3_w5", cam3, rf.DepthImage(values=z3.astype(np.float64)), z3, 5, "f32")

    # 4. left half invalid (mask_rect), window 3: status bits at the hole boundary
    masked = rf.GroundTruthPlane(np.array([0.1, -0.2, 1.0, -2.0]), mask_rect=(10, 0, 24, 12))
    d4, _ = rf.render_scene(rf.SyntheticScene((masked,)), maps3, noise=rf.NoiseModel(), seed=9)
    z4 = np.where(d4.valid, d4.values, 0.0).astype(np.float32)
    run_case("half_invalid_w3", cam3, rf.DepthImage(values=z4.astype(np.float64)), z4, 3, "f32")

    # 5. high-resolution intrinsics, near and far depth (C5-like f=2900 crop), window 7
    cam5 = rf.CameraIntrinsics(fx=2900.0, fy=2900.0, cx=20.5, cy=15.5, width=40, height=32)
    maps5 = rf.compute_tan_maps(cam5)
    scene5 = rf.SyntheticScene((rf.GroundTruthPlane(np.array([0.05, 0.02, -1.0, 0.31]), mask_rect=(0, 0, 20, 32)),
                                rf.GroundTruthPlane(np.array([-0.1, 0.3, -1.0, 18.0]), mask_rect=(20, 0, 40, 32))))
    d5, _ = rf.render_scene(scene5, maps5, noise=rf.NoiseModel(), seed=12, dropout=0.05)
    z5 = np.where(d5.valid, d5.values, 0.0).astype(np.float32)
    run_case("near_far_w7", cam5, rf.DepthImage(values=z5.astype(np.float64)), z5, 7, "f32")

    # 6. non-separable tan maps: per-pixel distortion offsets (CameraIntrinsics.delta_*)
    rng_d = np.random.default_rng(41)
    cam6 = rf.CameraIntrinsics(fx=60.0, fy=58.0, cx=23.5, cy=17.5, width=48, height=36,
                               delta_x=rng_d.uniform(-0.4, 0.4, (36, 48)),
                               delta_y=rng_d.uniform(-0.4, 0.4, (36, 48)))
    maps6 = rf.compute_tan_maps(cam6)
    scene6 = rf.SyntheticScene((random_plane(rng_d, 1.0, 3.0), random_plane(rng_d, 1.0, 3.0)))
    d6, _ = rf.render_scene(scene6, maps6, noise=rf.NoiseModel(), seed=13, dropout=0.05)
    z6 = np.where(d6.valid, d6.values, 0.0).astype(np.float32)
    run_case("distorted_f32_w5", cam6, rf.DepthImage(values=z6.astype(np.float64)), z6, 5, "f32")

    # 7. larger windows: uint16 with an explicit mask at 9x9, and a 15x15 near/far crop
    rng_w = np.random.default_rng(57)
    cam7 = rf.CameraIntrinsics(fx=45.0, fy=45.0, cx=19.5, cy=15.5, width=40, height=32)
    maps7 = rf.compute_tan_maps(cam7)
    d7, _ = rf.render_scene(rf.SyntheticScene((random_plane(rng_w, 0.8, 3.0), random_plane(rng_w, 0.8, 3.0))),
                            maps7, noise=rf.NoiseModel(), seed=21, dropout=0.08)
    mm7 = d7.to_millimeters()
    mask7 = rng_w.random(mm7.shape) > 0.1
    dm7 = rf.DepthImage.from_millimeters(mm7)
    run_case("planes_u16_mask_w9", cam7, rf.DepthImage(values=dm7.values, valid=dm7.valid & mask7), mm7, 9, "u16")
    cam8 = rf.CameraIntrinsics(fx=1400.0, fy=1400.0, cx=23.5, cy=17.5, width=48, height=36)
    maps8 = rf.compute_tan_maps(cam8)
    scene8 = rf.SyntheticScene((rf.GroundTruthPlane(np.array([0.1, -0.05, -1.0, 0.45]), mask_rect=(0, 0, 30, 36)),
                                rf.GroundTruthPlane(np.array([-0.2, 0.1, -1.0, 7.5]), mask_rect=(30, 0, 48, 36))))
    d8, _ = rf.render_scene(scene8, maps8, noise=rf.NoiseModel(), seed=22, dropout=0.05)
    z8 = np.where(d8.valid, d8.values, 0.0).astype(np.float32)
    run_case("near_far_w15", cam8, rf.DepthImage(values=z8.astype(np.float64)), z8, 15, "f32")
    # C5's 31x31 windows on a 64x48 crop of an f=2900 camera, near and far planes
    cam9 = rf.CameraIntrinsics(fx=2900.0, fy=2900.0, cx=31.5, cy=23.5, width=64, height=48)
    maps9 = rf.compute_tan_maps(cam9)
    scene9 = rf.SyntheticScene((rf.GroundTruthPlane(np.array([0.03, 0.01, -1.0, 0.35]), mask_rect=(0, 0, 40, 48)),
                                rf.GroundTruthPlane(np.array([0.1, -0.2, -1.0, 16.0]), mask_rect=(40, 0, 64, 48))))
    d9, _ = rf.render_scene(scene9, maps9, noise=rf.NoiseModel(), seed=23, dropout=0.05)
    z9 = np.where(d9.valid, d9.values, 0.0).astype(np.float32)
    run_case("near_far_w31", cam9, rf.DepthImage(values=z9.astype(np.float64)), z9, 31, "f32")
    # C2's 11x11 window on a 5-plane frame with holes
    rng_11 = np.random.default_rng(61)
    cam10 = rf.CameraIntrinsics(fx=70.0, fy=70.0, cx=27.5, cy=19.5, width=56, height=40)
    maps10 = rf.compute_tan_maps(cam10)
    d10, _ = rf.render_scene(rf.SyntheticScene(tuple(random_plane(rng_11, 0.7, 3.5) for _ in range(5))), maps10,
                             noise=rf.NoiseModel(), seed=24, dropout=0.12)
    z10 = np.where(d10.valid, d10.values, 0.0).astype(np.float32)
    run_case("planes_f32_w11", cam10, rf.DepthImage(values=z10.astype(np.float64)), z10, 11, "f32")


if __name__ == "__main__":
    main()
