"""Numerical model of the packed-fp32 pair solve that was built and measured in round 2
(correct, but not faster than the fp64 solve_fast, so not shipped).

For windows of BASELINE-shaped scenes it compares, against numpy fp64 eigensolves of the
reference's 4x4 scatter: the fp32 solve in ALIGNED coordinates (standard form sheared by the
window centre's ray), seeds from the fp32 cubics, three adjugate stages and fp64 Rayleigh
quotients of the eigenvalue and the curvature.  usage: python tools/fp32_solve_model.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2103_06644_b200 import scenes  # noqa: E402

f32 = np.float32


def windows(cfg, r, seed, crop, npix, rng):
    z = scenes.render_frame(cfg, seed).numpy()
    zv = z.astype(np.float64) / (1000.0 if cfg.u16 else 1.0)
    valid = (z > 0) if cfg.u16 else (np.isfinite(zv) & (zv > 0))
    H, W = zv.shape
    y0, x0, h, w = crop
    tx = (np.arange(W) - cfg.cx) / cfg.f
    ty = (np.arange(H) - cfg.cy) / cfg.f
    ys = rng.integers(max(y0, r), min(y0 + h, H - r), npix)
    xs = rng.integers(max(x0, r), min(x0 + w, W - r), npix)
    keep = valid[ys, xs]
    ys, xs = ys[keep], xs[keep]
    out = {}
    for sp in ("DF", "ST"):
        M = []
        for dy in range(-r, r + 1):
            for dx in range(-r, r + 1):
                yy, xx = ys + dy, xs + dx
                v = valid[yy, xx]
                Z = np.where(v, zv[yy, xx], 1.0)
                m = (np.stack([tx[xx], ty[yy], 1.0 / Z], -1) if sp == "DF"
                     else np.stack([tx[xx] * Z, ty[yy] * Z, Z], -1))
                M.append(np.where(v[:, None], m, np.nan))
        M = np.stack(M, 1)
        vm = ~np.isnan(M[..., 0])
        n = vm.sum(1).astype(np.float64)
        ok = n >= 4
        M, vm, n = M[ok], vm[ok], n[ok]
        mu = np.where(vm[..., None], M, 0.0).sum(1) / n[:, None]
        D = np.where(vm[..., None], M - mu[:, None, :], 0.0)
        out[sp] = (np.einsum("pki,pkj->pij", D, D), mu, n, tx[xs[ok]], ty[ys[ok]])
    return out


def reference(C, mu, n, sp):
    P = len(n)
    S = np.zeros((P, 4, 4))
    S[:, :3, :3] = C + n[:, None, None] * mu[:, :, None] * mu[:, None, :]
    S[:, :3, 3] = S[:, 3, :3] = n[:, None] * mu
    S[:, 3, 3] = n
    w, V = np.linalg.eigh(S)
    v = V[:, :, 0]
    normal = np.stack([v[:, 0], v[:, 1], v[:, 3]], -1) if sp == "DF" else v[:, :3]
    kap = np.linalg.eigvalsh(C)[:, 0] / np.trace(C, axis1=1, axis2=2)
    return normal, w[:, 0], kap


def sym6(M):
    return (M[:, 0, 0], M[:, 0, 1], M[:, 0, 2], M[:, 1, 1], M[:, 1, 2], M[:, 2, 2])


def adj_column(E):
    e00, e01, e02, e11, e12, e22 = E
    B00, B11, B22 = e11 * e22 - e12 * e12, e00 * e22 - e02 * e02, e00 * e11 - e01 * e01
    B01, B02, B12 = e02 * e12 - e01 * e22, e01 * e12 - e02 * e11, e01 * e02 - e00 * e12
    k = np.stack([np.abs(B00), np.abs(B11), np.abs(B22)], -1).argmax(-1)
    cols = np.stack([np.stack([B00, B01, B02], -1), np.stack([B01, B11, B12], -1),
                     np.stack([B02, B12, B22], -1)], 1)
    return cols[np.arange(len(k)), k]


def trig_cubic(a2, a1, a0):
    """roots l1 <= l2 <= l3 of l^3 - a2 l^2 + a1 l - a0 (fp32, as rf_solve.cuh trig_cubic)"""
    a2, a1, a0 = f32(a2), f32(a1), f32(a0)
    q = a2 * f32(1 / 3)
    p = np.maximum(q * q - a1 * f32(1 / 3), f32(1e-37))
    isp = f32(1) / np.sqrt(p)
    h = (q * q - f32(0.5) * a1) * q + f32(0.5) * a0
    c = np.clip(h * isp * isp * isp, f32(-1), f32(1))
    l3 = np.maximum(f32(2) * p * isp * np.cos(np.arccos(c) / f32(3)) + q, f32(1e-37))
    P = a0 / l3
    S = (a1 - P) / l3
    sd = S + np.sqrt(np.maximum(S * S - f32(4) * P, f32(0)))
    l1 = np.where(sd > 0, f32(2) * P / np.where(sd > 0, sd, f32(1)), f32(0))
    return l1.astype(f32), (f32(0.5) * sd).astype(f32), l3


def solve(C, mu, n, sp, txo, tyo):
    P = len(n)
    T = np.tile(np.eye(3), (P, 1, 1))
    if sp == "ST":
        T[:, 0, 2], T[:, 1, 2] = -txo, -tyo
    K = np.einsum("pij,pjk,plk->pil", T, C, T)          # aligned scatter (fp64)
    Kf, m, Tf = K.astype(f32), mu.astype(f32), T.astype(f32)
    pf = np.einsum("pij,pj->pi", T, mu).astype(f32)
    TTf = np.einsum("pij,pkj->pik", Tf, Tf)
    A = np.empty_like(Kf)
    k00, k01, k02, k11, k12, k22 = sym6(Kf)
    A[:, 0, 0], A[:, 1, 1], A[:, 2, 2] = k11 * k22 - k12 * k12, k00 * k22 - k02 * k02, k00 * k11 - k01 * k01
    A[:, 0, 1] = A[:, 1, 0] = k02 * k12 - k01 * k22
    A[:, 0, 2] = A[:, 2, 0] = k01 * k12 - k02 * k11
    A[:, 1, 2] = A[:, 2, 1] = k01 * k02 - k00 * k12
    det = k00 * A[:, 0, 0] + k01 * A[:, 0, 1] + k02 * A[:, 0, 2]
    nu = (m * m).sum(-1)
    Ti = np.tile(np.eye(3, dtype=f32), (P, 1, 1))
    Ti[:, 0, 2], Ti[:, 1, 2] = -Tf[:, 0, 2], -Tf[:, 1, 2]
    Bp = np.einsum("pij,pjk,plk->pil", Tf, np.eye(3, dtype=f32) + m[:, :, None] * m[:, None, :], Tf)
    adjB = np.einsum("pji,pjk,pkl->pil", Ti, (f32(1) + nu)[:, None, None] * np.eye(3, dtype=f32)
                     - m[:, :, None] * m[:, None, :], Ti)
    inv = f32(1) / (f32(1) + nu)
    g1, g2, g3 = trig_cubic((Kf * adjB).sum((1, 2)) * inv, (A * Bp).sum((1, 2)) * inv, det * inv)
    k1, k2, k3 = trig_cubic((Kf * np.einsum("pji,pjk->pik", Ti, Ti)).sum((1, 2)), (A * TTf).sum((1, 2)), det)
    nf = n.astype(f32)

    def E(l, gam):
        return sym6(Kf - l[:, None, None] * TTf - gam[:, None, None] * pf[:, :, None] * pf[:, None, :])

    def ab(v):
        u = np.einsum("pji,pj->pi", Tf, v)
        return (u * u).sum(-1), ((m * u).sum(-1)) ** 2, u

    v = adj_column(E(g1, g1)).astype(f32)                # stage 1: beta = 1
    a, b, _ = ab(v)
    lam_e = g1
    for _ in range(2):
        lam_e = g1 * (a + b) / (a + nf / (nf - lam_e) * b)
    beta = nf / (nf - lam_e)
    v = adj_column(E(lam_e, lam_e * beta)).astype(f32)  # stage 2
    R = np.einsum("pi,pij,pj->p", v.astype(np.float64), K, v.astype(np.float64))  # fp64
    a, b, _ = ab(v)
    a, b = a.astype(np.float64), b.astype(np.float64)
    lam = R / (a + b)
    for _ in range(2):
        lam = R / (a + n / (n - lam) * b)
    l32, beta = lam.astype(f32), (n / (n - lam)).astype(f32)
    v = adj_column(E(l32, l32 * beta)).astype(f32)      # stage 3: the plane
    _, _, u = ab(v)
    s = -(beta * (m * u).sum(-1))
    normal = np.stack([u[:, 0], u[:, 1], s], -1) if sp == "DF" else u
    vc = adj_column(sym6(Kf - k1[:, None, None] * TTf)).astype(np.float64)  # curvature
    uc = np.einsum("pji,pj->pi", T, vc)
    kap = np.einsum("pi,pij,pj->p", vc, K, vc) / (uc * uc).sum(-1) / np.trace(C, axis1=1, axis2=2)
    certified = ((g2 - g1) >= 0.05 * g2) & ((k2 - k1) >= 0.05 * k2)
    return normal.astype(np.float64), lam, kap, certified


def angle(a, b):
    return np.arctan2(np.linalg.norm(np.cross(a, b), axis=-1), np.abs((a * b).sum(-1)))


if __name__ == "__main__":
    cases = [("C2", 2, (0, 0, 480, 640)), ("C2", 1, (0, 0, 480, 640)), ("C2", 7, (0, 0, 480, 640)),
             ("C3", 4, (0, 0, 720, 1280)), ("C4", 7, (0, 0, 1080, 1920)),
             ("C5", 15, (2048, 3072, 1024, 1024)), ("C5", 15, (0, 0, 3072, 4096))]
    for name, r, crop in cases:
        cfg = scenes.CONFIGS[name]
        ws = windows(cfg, r, 1000 * int(name[1:]) + 1, crop, 6000 if r < 10 else 1500, np.random.default_rng(5))
        for sp in ("DF", "ST"):
            C, mu, n, txo, tyo = ws[sp]
            nr, lr, kr = reference(C, mu, n, sp)
            ng, lg, kg, ok = solve(C, mu, n, sp, txo, tyo)
            ang = angle(nr, ng)[ok]
            print(f"{name} w{2 * r + 1:2d} {sp}: {ok.sum():5d} certified ({1 - ok.mean():.2%} declined)  "
                  f"normal max {ang.max():.1e} rad  lam rel {np.max(np.abs(lg - lr)[ok] / lr[ok]):.1e}  "
                  f"curvature rel {np.max(np.abs(kg - kr)[ok] / kr[ok]):.1e}")
