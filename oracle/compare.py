"""TEST INFRASTRUCTURE ONLY -- parity metrics between the sm_100a outputs and the
oracle (restated reference), with the tolerances of BASELINE.json's north_star:

* status: bit0 (input valid) and bit1 (window fit) bit-exact; bit2 (degenerate,
  a float threshold, fitting.py:553-554) is reported, not required;
* normal: angle (reference ``normal_angle``, fitting.py:742-754, atan2 of
  cross/dot) <= 1e-4 rad on fitted, non-degenerate pixels;
* residual and curvature: relative error <= 1e-4, plus an absolute allowance
  where a relative error is ill-posed (noiseless windows, where lambda is
  rounding noise of size ~eps*||S||_F): residual allowance
  sqrt(1e-11 * ||S||_F / n) (the rms of a rounding-level eigenvalue),
  curvature allowance 1e-8 plus 4e-15 * curv_cond, where curv_cond (from the oracle) is the
  uncentred monomial diagonal over the centred trace -- the factor by which centring the
  window sums amplifies rounding in lambda_min / trace (e.g. millimetre depths among metres
  in the disparity form put 1/Z^2 ~ 1e6 next to tan-angle spreads ~ 1e-3).  4e-15 (~36 eps)
  covers two fp64 implementations each off by up to ~18 eps * curv_cond: the oracle's own
  value on exactly planar millimetre windows (curv_cond ~ 3e8, true curvature 0) is
  ~2.3e-15 * curv_cond (tests/test_gpu_sliding.py).
"""

from __future__ import annotations

import numpy as np

NORMAL_TOL_RAD = 1e-4
REL_TOL = 1e-4
CURV_FLOOR = 1e-8
CURV_COND_REL = 4e-15
LAM_FLOOR_REL = 1e-11


def normal_angles(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    cross = np.linalg.norm(np.cross(a, b), axis=-1)
    dot = np.abs((a * b).sum(-1))
    return np.arctan2(cross, dot)


def compare(gpu: dict, ref: dict, explicit_fit: bool = False, include_degenerate: bool = False) -> dict:
    """gpu/ref: dicts of flat arrays normal (P,3), offset, residual, curvature, status (P,);
    ref also carries ``scale`` = ||S||_F/n.  Returns metrics and a pass flag.  Explicit fits
    compute their residual from aggregated sums, sum(b^2) - alpha.rhs, whose cancellation
    floor the reference documents (fitting.py:592-595): their allowance uses 1e-10."""
    gs = np.asarray(gpu["status"]).astype(np.uint8).ravel()
    rs = np.asarray(ref["status"]).astype(np.uint8).ravel()
    mask_bits = 0b011
    status_mismatch = int(((gs & mask_bits) != (rs & mask_bits)).sum())
    fit = ((rs & 2) != 0) & ((gs & 2) != 0)
    degen = ((rs & 4) != 0)
    # degenerate implicit windows (eigenvalue near-ties) have no well-defined normal; explicit
    # ones (failed Cholesky pivots) are the reference's minimum-norm solution and compare too
    sel = fit if include_degenerate else fit & ~degen
    gn = np.asarray(gpu["normal"], np.float64).reshape(-1, 3)
    rn = np.asarray(ref["normal"], np.float64).reshape(-1, 3)
    ang = normal_angles(gn[sel], rn[sel]) if sel.any() else np.zeros(0)
    gres = np.asarray(gpu["residual"], np.float64).ravel()[sel]
    rres = np.asarray(ref["residual"], np.float64).ravel()[sel]
    scale = np.asarray(ref["scale"], np.float64).ravel()[sel]
    res_floor = np.sqrt((1e-10 if explicit_fit else LAM_FLOOR_REL) * np.abs(scale))
    # error in units of the tolerance: <= 1 passes
    res_err = np.abs(gres - rres) / (REL_TOL * np.abs(rres) + res_floor) * REL_TOL
    gc = np.asarray(gpu["curvature"], np.float64).ravel()[sel]
    rc = np.asarray(ref["curvature"], np.float64).ravel()[sel]
    cur_floor = CURV_FLOOR
    if "curv_cond" in ref:
        cond = np.asarray(ref["curv_cond"], np.float64).ravel()[sel]
        cur_floor = CURV_FLOOR + CURV_COND_REL * np.where(np.isfinite(cond), cond, 0.0)
    cur_err = np.abs(gc - rc) / (REL_TOL * np.abs(rc) + cur_floor) * REL_TOL
    # offsets: same sign convention, relative to max(|offset|, 1e-6)
    go = np.asarray(gpu["offset"], np.float64).ravel()[sel]
    ro = np.asarray(ref["offset"], np.float64).ravel()[sel]
    # offset error is bounded by the normal error times |offset| plus relative terms
    off_err = np.abs(go - ro) / np.maximum(np.abs(ro), 1e-6)
    nonfit_nan = True
    g_nf = (gs & 2) == 0
    if g_nf.any():
        nonfit_nan = bool(np.isnan(np.asarray(gpu["residual"], np.float64).ravel()[g_nf]).all())
    m = {
        "pixels": int(rs.size),
        "fitted": int(fit.sum()),
        "compared": int(sel.sum()),
        "degenerate_ref": int((fit & degen).sum()),
        "status_mismatch": status_mismatch,
        "degenerate_mismatch": int((((gs & 4) != 0) != degen)[fit].sum()),
        "max_normal_rad": float(ang.max()) if ang.size else 0.0,
        "p999_normal_rad": float(np.quantile(ang, 0.999)) if ang.size else 0.0,
        "max_residual_rel": float(res_err.max()) if res_err.size else 0.0,
        "max_curvature_rel": float(cur_err.max()) if cur_err.size else 0.0,
        "max_offset_rel": float(off_err.max()) if off_err.size else 0.0,
        "normal_fail": int((ang > NORMAL_TOL_RAD).sum()),
        "residual_fail": int((res_err > REL_TOL).sum()),
        "curvature_fail": int((cur_err > REL_TOL).sum()),
        "nonfit_is_nan": nonfit_nan,
    }
    m["ok"] = (m["status_mismatch"] == 0 and m["normal_fail"] == 0 and m["residual_fail"] == 0
               and m["curvature_fail"] == 0 and nonfit_nan)
    return m


def worst_pixels(gpu: dict, ref: dict, k: int = 5):
    """Indices of the k worst normal-angle pixels (debug aid)."""
    rs = np.asarray(ref["status"]).ravel()
    gs = np.asarray(gpu["status"]).ravel()
    sel = np.nonzero(((rs & 2) != 0) & ((gs & 2) != 0) & ((rs & 4) == 0))[0]
    gn = np.asarray(gpu["normal"], np.float64).reshape(-1, 3)[sel]
    rn = np.asarray(ref["normal"], np.float64).reshape(-1, 3)[sel]
    ang = normal_angles(gn, rn)
    order = np.argsort(-ang)[:k]
    return sel[order], ang[order]
