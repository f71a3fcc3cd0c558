"""Design check (not product, not oracle): numpy model of the sm_100a per-window
solve.  Pencil  C u = lam (I + beta mu mu^T) u  (the Schur complement of the
uncentred 4x4 scatter on its constant monomial), solved by
  1. fp32 trigonometric roots of the beta=1 characteristic cubic (guesses),
  2. fp64 top eigenvector w of the pencil from an adjugate column at lam3,
  3. fp64 2x2 Rayleigh-Ritz on the B-orthogonal complement of w (holds u1
     exactly, so near-ties lam1 ~ lam2 are resolved in fp64),
  4. one beta refresh + second 2x2 solve.
Curvature lam_min(C)/tr(C): fp32 trig roots, then fp64 Newton on whichever
end of the spectrum is better separated (direct lam1, or lam3 + deflation)."""
import numpy as np

f32 = np.float32


def trig_cubic(a2, a1, a0):
    """Roots l1<=l2<=l3 of l^3 - a2 l^2 + a1 l - a0 (all real) in fp32."""
    a2, a1, a0 = f32(a2), f32(a1), f32(a0)
    q = a2 / f32(3)
    p = np.maximum(q * q - a1 / f32(3), f32(0))
    sp = np.sqrt(p)
    h = q * q * q - f32(0.5) * q * a1 + f32(0.5) * a0
    den = p * sp
    c = np.where(den > 0, h / np.where(den > 0, den, f32(1)), f32(1))
    c = np.clip(c, f32(-1), f32(1))
    phi = np.arccos(c) / f32(3)
    l3 = q + f32(2) * sp * np.cos(phi)
    l3 = np.maximum(l3, f32(1e-37))
    P = a0 / l3
    S = (a1 - P) / l3
    disc = np.sqrt(np.maximum(S * S - f32(4) * P, f32(0)))
    l2 = f32(0.5) * (S + disc)
    l1 = f32(2) * P / np.maximum(S + disc, f32(1e-37))
    return l1, l2, l3


def cof(c00, c01, c02, c11, c12, c22):
    return (c11 * c22 - c12 * c12, c00 * c22 - c02 * c02, c00 * c11 - c01 * c01,
            c02 * c12 - c01 * c22, c01 * c12 - c02 * c11, c01 * c02 - c00 * c12)


def rsqrt(x):
    return 1.0 / np.sqrt(x)


def ritz2(C, mu, beta, p1, p2):
    """Smallest eigenpair of the pencil restricted to span(p1, p2)."""
    c00, c01, c02, c11, c12, c22 = C
    def Cv(p):
        return np.stack([c00 * p[..., 0] + c01 * p[..., 1] + c02 * p[..., 2],
                         c01 * p[..., 0] + c11 * p[..., 1] + c12 * p[..., 2],
                         c02 * p[..., 0] + c12 * p[..., 1] + c22 * p[..., 2]], -1)
    d = lambda a, b: (a * b).sum(-1)
    Cp1, Cp2 = Cv(p1), Cv(p2)
    K11, K12, K22 = d(p1, Cp1), d(p2, Cp1), d(p2, Cp2)
    m1, m2 = d(p1, mu), d(p2, mu)
    N11 = d(p1, p1) + beta * m1 * m1
    N12 = d(p1, p2) + beta * m1 * m2
    N22 = d(p2, p2) + beta * m2 * m2
    r1 = rsqrt(N11)
    n12 = N12 * r1
    r2 = rsqrt(N22 - n12 * n12)
    k11 = K11 * r1 * r1
    k12 = r1 * r2 * (K12 - n12 * r1 * K11)
    k22 = r2 * r2 * (K22 - 2 * n12 * r1 * K12 + n12 * n12 * r1 * r1 * K11)
    hm = 0.5 * (k11 - k22)
    disc = np.sqrt(hm * hm + k12 * k12)
    big = 0.5 * (k11 + k22) + disc
    small = (k11 * k22 - k12 * k12) / np.where(big != 0, big, 1.0)
    # eigenvector of [[k11,k12],[k12,k22]] for `small`
    ya = np.stack([k12, small - k11], -1)
    yb = np.stack([small - k22, k12], -1)
    y = np.where((np.abs(small - k11) >= np.abs(small - k22))[..., None], ya, yb)
    # back to p-coordinates: q1 = r1 p1, q2 = r2 (p2 - n12 r1 p1)
    t1 = y[..., 0] * r1 - y[..., 1] * r2 * n12 * r1
    t2 = y[..., 1] * r2
    u = t1[..., None] * p1 + t2[..., None] * p2
    return small, big, u


def solve(Cm, mu, n):
    n = n.astype(np.float64)
    C = (Cm[..., 0, 0], Cm[..., 0, 1], Cm[..., 0, 2], Cm[..., 1, 1], Cm[..., 1, 2], Cm[..., 2, 2])
    c00, c01, c02, c11, c12, c22 = C
    # ---- fp64 characteristic coefficients, fp32 trigonometric roots ----
    A = cof(*C)
    t = c00 + c11 + c22
    c1 = A[0] + A[1] + A[2]
    det = c00 * A[0] + c01 * A[3] + c02 * A[4]
    nu = (mu * mu).sum(-1)
    Cmu = np.stack([c00 * mu[..., 0] + c01 * mu[..., 1] + c02 * mu[..., 2],
                    c01 * mu[..., 0] + c11 * mu[..., 1] + c12 * mu[..., 2],
                    c02 * mu[..., 0] + c12 * mu[..., 1] + c22 * mu[..., 2]], -1)
    Amu = np.stack([A[0] * mu[..., 0] + A[3] * mu[..., 1] + A[4] * mu[..., 2],
                    A[3] * mu[..., 0] + A[1] * mu[..., 1] + A[5] * mu[..., 2],
                    A[4] * mu[..., 0] + A[5] * mu[..., 1] + A[2] * mu[..., 2]], -1)
    mm = (mu * Cmu).sum(-1)
    aa = (mu * Amu).sum(-1)
    inv = 1.0 / (1.0 + nu)
    g1, g2, g3 = trig_cubic((t + t * nu - mm) * inv, (c1 + aa) * inv, det * inv)
    k1, k2, k3 = trig_cubic(t, c1, det)
    # ---- pencil: lam1 by (A) Newton on the quartic from below, or (B) for a
    # near-tie lam1 ~ lam2, deflation of lam3 (Newton from above) and lam4 ----
    n_ = n
    q3 = n_ + t + n_ * nu
    q2 = n_ * t + c1 + n_ * (t * nu - mm)
    q1 = n_ * c1 + det + n_ * aa
    q0 = n_ * det
    G = lambda l: (((l - q3) * l + q2) * l - q1) * l + q0
    dG = lambda l: ((4 * l - 3 * q3) * l + 2 * q2) * l - q1
    la = g1.astype(np.float64) * (1 - 1e-4)
    for _ in range(3):
        la = la - G(la) * (1.0 / dG(la)).astype(np.float32).astype(np.float64)
    l3 = g3.astype(np.float64)
    for _ in range(4):
        l3 = l3 - G(l3) * (1.0 / dG(l3)).astype(np.float32).astype(np.float64)
    l4 = q3 - (g1.astype(np.float64) + g2.astype(np.float64) + l3)
    l4 = l4 - G(l4) / dG(l4)
    ss = l3 + l4
    pp = l3 * l4
    e0 = q0 / pp
    e1 = (ss * e0 - q1) / pp          # quadratic l^2 + e1 l + e0 (roots lam1, lam2)
    disc = np.sqrt(np.maximum(e1 * e1 - 4 * e0, 0))
    lb = 2 * e0 / np.maximum(-e1 + disc, 1e-300)
    lb2 = 0.5 * (-e1 + disc)
    tie = (g2 - g1) < f32(0.05) * g2
    lam = np.where(tie, lb, la)
    lam2 = np.where(tie, lb2, g2.astype(np.float64))
    beta = n / (n - lam)
    gam = lam * beta
    m0, m1, m2 = mu[..., 0], mu[..., 1], mu[..., 2]
    E = (c00 - lam - gam * m0 * m0, c01 - gam * m0 * m1, c02 - gam * m0 * m2,
         c11 - lam - gam * m1 * m1, c12 - gam * m1 * m2, c22 - lam - gam * m2 * m2)
    B = cof(*E)
    k = np.argmax(np.stack([np.abs(B[0]), np.abs(B[1]), np.abs(B[2])], -1), -1)
    u = np.where((k == 0)[..., None], np.stack([B[0], B[3], B[4]], -1),
                 np.where((k == 1)[..., None], np.stack([B[3], B[1], B[5]], -1),
                          np.stack([B[4], B[5], B[2]], -1)))
    s = -beta * (u * mu).sum(-1)
    v = np.concatenate([u, s[..., None]], -1)
    # ---- curvature: lam_min(C) ----
    tt, cc1, dd = t, c1, det
    P = lambda l: ((-l + tt) * l - cc1) * l + dd
    dP = lambda l: (-3 * l + 2 * tt) * l - cc1
    # bottom: Newton from the fp32 lam1 guess (slightly lowered)
    lb = k1.astype(np.float64) * (1 - 1e-4)
    lt = k3.astype(np.float64) * (1 + 1e-6)
    for _ in range(2):
        lb = lb - P(lb) / dP(lb)
        lt = lt - P(lt) / dP(lt)
    S = tt - lt
    Pp = dd / lt
    lbd = 2 * Pp / (S + np.sqrt(np.maximum(S * S - 4 * Pp, 0)))
    use_top = (k3 - k2) / np.maximum(k3, 1e-37) > (k2 - k1) / np.maximum(k2, 1e-37)
    lk = np.where(use_top, lbd, lb)
    kappa = lk / tt
    return lam, v, kappa, lam2
