// rf_solve.cuh -- per-window solve shared by the per-pixel (rf_fit.cu) and the
// per-rect (rf_rects.cu) kernels: fp32/fp64 helpers, the smallest eigenpair of
// the uncentred implicit scatter, the explicit fits, curvature and the canonical
// output form.  See DESIGN.md section 4.4 for the derivation.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace rf_dev {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
// reciprocal to ~1 ulp: approximate seed + two Newton steps (no IEEE fixup)
__device__ __forceinline__ double rcp_fast(double x) {
  double y = rcp_approx(x);
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__device__ __forceinline__ float frcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float fsqrt(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float frsqrt(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// acos on [-1, 1], |error| <= 2e-8 rad (Abramowitz & Stegun 4.4.46)
__device__ __forceinline__ float facos(float x) {
  const float ax = fabsf(x);
  float p = fmaf(ax, -0.0012624911f, 0.0066700901f);
  p = fmaf(ax, p, -0.0170881256f);
  p = fmaf(ax, p, 0.0308918810f);
  p = fmaf(ax, p, -0.0501743046f);
  p = fmaf(ax, p, 0.0889789874f);
  p = fmaf(ax, p, -0.2145988016f);
  p = fmaf(ax, p, 1.5707963050f);
  const float r = fsqrt(fmaxf(1.0f - ax, 0.0f)) * p;
  return x < 0.0f ? 3.14159265358979f - r : r;
}

// Roots l1 <= l2 <= l3 of l^3 - a2 l^2 + a1 l - a0 (three real roots), fp32
// seeds for the fp64 refinement.  l3 by the trigonometric formula, l1/l2 by
// deflation (product a0/l3, sum (a1 - l1 l2)/l3) so that small roots keep
// their relative accuracy.  Fast approximate intrinsics throughout (~1e-6).
__device__ __forceinline__ void trig_cubic(float a2, float a1, float a0, float& l1, float& l2,
                                           float& l3) {
  const float q = a2 * (1.0f / 3.0f);
  const float p = fmaxf(fmaf(q, q, -a1 * (1.0f / 3.0f)), 1e-37f);
  const float isp = frsqrt(p);
  const float sp = p * isp;
  const float h = fmaf(q * q - 0.5f * a1, q, 0.5f * a0);
  const float c = fminf(fmaxf(h * isp * isp * isp, -1.0f), 1.0f);
  const float phi = facos(c) * (1.0f / 3.0f);
  l3 = fmaxf(fmaf(2.0f * sp, __cosf(phi), q), 1e-37f);
  const float il3 = frcp(l3);
  const float P = a0 * il3;
  const float S = (a1 - P) * il3;
  const float sd = S + fsqrt(fmaxf(fmaf(S, S, -4.0f * P), 0.0f));
  l2 = 0.5f * sd;
  l1 = sd > 0.0f ? 2.0f * P * frcp(sd) : 0.0f;
}

// ---- packed fp32 pairs (sm_100 FFMA2 / FMUL2 / FADD2): the two seed cubics of a window
// (pencil, curvature) run in lock step, one instruction for both
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 neg2(float2 a) { return f2(-a.x, -a.y); }
__device__ __forceinline__ float2 max2(float2 a, float b) { return f2(fmaxf(a.x, b), fmaxf(a.y, b)); }

// positive normal double (2^-126 <= x < 2^128) -> float, truncated, on the integer pipe (no
// F2F): rebias the exponent and funnel-shift the top mantissa bits
__device__ __forceinline__ float pos_d2f(double x) {
  return __int_as_float(__funnelshift_l((unsigned)__double2loint(x), (unsigned)(__double2hiint(x) - 0x38000000), 3));
}
// positive normal float -> double (exact), on the integer pipe
__device__ __forceinline__ double pos_f2d(float f) {
  const unsigned b = __float_as_uint(f);
  return __hiloint2double((int)((b >> 3) + 0x38000000u), (int)(b << 29));
}

// cos(acos(c) / 3) for c in [-1, 1] (the trigonometric cubic's largest-root factor):
// with u = sqrt((1 + c) / 2) = cos(3 theta / 2) it is cos(2/3 acos u), analytic on [0, 1];
// degree-7 fit, |error| < 6e-8 (replaces an acos polynomial plus a cosine)
__device__ __forceinline__ float2 cos_third_acos2(float2 c) {
  const float2 v = fma2(c, f2(0.5f), f2(0.5f));
  const float2 u = f2(fsqrt(v.x), fsqrt(v.y));
  float2 y = fma2(u, f2(0.0011383f), f2(-0.00610606f));
  y = fma2(u, y, f2(0.01603623f));
  y = fma2(u, y, f2(-0.03019835f));
  y = fma2(u, y, f2(0.05281415f));
  y = fma2(u, y, f2(-0.11103019f));
  y = fma2(u, y, f2(0.57734591f));
  return fma2(u, y, f2(0.50000006f));
}

// trig_cubic for two cubics at once (x: one, y: the other)
__device__ __forceinline__ void trig_cubic2(float2 a2, float2 a1, float2 a0, float2& l1, float2& l2, float2& l3) {
  const float2 q = mul2(a2, f2(1.0f / 3.0f));
  const float2 p = max2(fma2(q, q, mul2(a1, f2(-1.0f / 3.0f))), 1e-37f);
  const float2 isp = f2(frsqrt(p.x), frsqrt(p.y));
  const float2 sp = mul2(p, isp);
  const float2 h = fma2(fma2(q, q, mul2(a1, f2(-0.5f))), q, mul2(a0, f2(0.5f)));
  const float2 c0 = mul2(mul2(h, isp), mul2(isp, isp));
  const float2 c = f2(fminf(fmaxf(c0.x, -1.0f), 1.0f), fminf(fmaxf(c0.y, -1.0f), 1.0f));
  l3 = max2(fma2(add2(sp, sp), cos_third_acos2(c), q), 1e-37f);
  const float2 il3 = f2(frcp(l3.x), frcp(l3.y));
  const float2 P = mul2(a0, il3);
  const float2 S = mul2(add2(a1, neg2(P)), il3);
  const float2 D = max2(fma2(S, S, mul2(P, f2(-4.0f))), 0.0f);
  const float2 sd = add2(S, f2(fsqrt(D.x), fsqrt(D.y)));
  l2 = mul2(sd, f2(0.5f));
  const float2 t = mul2(add2(P, P), f2(frcp(sd.x), frcp(sd.y)));
  l1 = f2(sd.x > 0.0f ? t.x : 0.0f, sd.y > 0.0f ? t.y : 0.0f);
}

struct Sym3 {
  double c00, c01, c02, c11, c12, c22;
};

struct WindowFit {
  double lam;       // smallest eigenvalue of the 4x4 scatter
  double u0, u1, u2;  // coefficients of the three non-constant monomials
  double s;         // coefficient of the constant monomial
  float kappa;      // curvature
  bool degenerate;
};

// Curvature lam_min(C)/tr(C) from the invariants t = tr C,
// c1 = sum of principal 2x2 minors, det = det C and the fp32 roots k1<=k2<=k3 of
// l^3 - t l^2 + c1 l - det: fp64 Newton from below, or -- when the bottom pair is
// close -- Newton from above on lam_max and deflation.
// fp64 polish of the curvature eigenvalue (close bottom pair, or a bottom near-tie
// handled from the top): out of line, the common case never enters it.
static __device__ __noinline__ float curvature_slow(double t, double c1, double det, float ft, float k1, float k2,
                                             float k3, bool top) {
  auto newton = [&](double x) {
    const double P = fma(fma(t - x, x, -c1), x, det);
    const double dP = fma(fma(-3.0, x, 2.0 * t), x, -c1);
    return P * rcp_approx(dP);
  };
  double lk;
  if (!top) {
    // Newton from below lam_min (monotone)
    double l = (double)k1 * (1.0 - 1e-5);
    l -= newton(l);
    l -= newton(l);
    if ((k2 - k1) < 0.05f * k2) {  // close bottom pair: iterate to convergence
      for (int it = 0; it < 64; ++it) {
        const double step = newton(l);
        l -= step;
        if (!(fabs(step) > 1e-10 * l)) break;
      }
    }
    lk = l;
  } else {
    // near-tie at the bottom: Newton from above lam_max (well separated here), then
    // deflate; lam_max only needs ~1e-10 for a 1e-5 curvature
    double l = fmin((double)k3 * (1.0 + 1e-5), t);
    l -= newton(l);
    l -= newton(l);
    if ((k3 - k2) < 0.05f * k3) {  // top pair close too: iterate to convergence
      for (int it = 0; it < 62; ++it) {
        const double step = newton(l);
        l -= step;
        if (!(fabs(step) > 1e-12 * l)) break;
      }
    }
    const double S = t - l;
    const double Pp = det * rcp_fast(l);
    const double den = S + (double)fsqrt((float)fmax(fma(S, S, -4.0 * Pp), 0.0));
    lk = den > 0.0 ? 2.0 * Pp * rcp_fast(den) : 0.0;
  }
  return t > 0.0 ? (float)lk * frcp(ft) : 0.0f;
}

// Curvature in three pieces so that solve_window can interleave the curvature Newton
// step with its own (independent chains, half the latency):
//  * curv_seed: the Newton start -- lam_min from just below its fp32 seed when the bottom
//    pair is >= 5% apart (nearly every window), else lam_max (then deflate: lam_1 + lam_2 =
//    t - lam_max, lam_1 lam_2 = det / lam_max); both pairs close: out of line;
//  * curv_newton: one fp64 Newton step on det(C - l I);
//  * curv_finish: the ratio, the deflation, or the out-of-line path.
struct CurvSeed {
  bool top, close, slow_top;
  double x;
};
__device__ __forceinline__ CurvSeed curv_seed(float k1, float k2, float k3) {
  CurvSeed c;
  // bottom pair separated by >= 5%: Newton on lam_min from just below the fp32 seed
  // (seed error <~ 1e-4, one step leaves < 1e-6 relative); otherwise Newton on lam_max
  // and deflation; both pairs close: out of line (curvature_slow)
  const bool bclose = (k2 - k1) < 0.05f * k2;
  const bool tclose = (k3 - k2) < 0.05f * k3;
  c.top = bclose;
  c.close = bclose && tclose;
  c.slow_top = (k3 - k2) * k2 > (k2 - k1) * k3;  // the better separated side
  c.x = (double)(c.top ? k3 : k1 * (1.0f - 1e-5f));  // one conversion
  return c;
}
__device__ __forceinline__ double curv_newton(double t, double c1, double det, double x) {
  const double P = fma(fma(t - x, x, -c1), x, det);
  const double dP = fma(fma(-3.0, x, 2.0 * t), x, -c1);
  return x - P * rcp_approx(dP);
}
__device__ __forceinline__ float curv_finish(const CurvSeed& c, double t, double c1, double det, float ft,
                                             float k1, float k2, float k3) {
  if (c.close) return curvature_slow(t, c1, det, ft, k1, k2, k3, c.slow_top);  // out of line, rare
  float kmin = (float)c.x;
  if (c.top) {
    const double S = t - c.x;
    const double Pp = det * rcp_fast(c.x);
    const float D = (float)fma(S, S, -4.0 * Pp);  // (lam_2 - lam_1)^2, cancellation-free in fp64
    const float fS = (float)S;
    kmin = 2.0f * (float)Pp * frcp(fS + fsqrt(fmaxf(D, 0.0f)));
  }
  return t > 0.0 ? kmin * frcp(ft) : 0.0f;
}
__device__ __forceinline__ float curvature_from(double t, double c1, double det, float ft, float k1,
                                                float k2, float k3) {
  CurvSeed c = curv_seed(k1, k2, k3);
  if (!c.close) {
    c.x = curv_newton(t, c1, det, c.x);
    c.x = curv_newton(t, c1, det, c.x);
  }
  return curv_finish(c, t, c1, det, ft, k1, k2, k3);
}

// curvature when no implicit solve runs (explicit fits only)
__device__ __forceinline__ float curvature_only(const Sym3& C) {
  const double A00 = C.c11 * C.c22 - C.c12 * C.c12;
  const double A11 = C.c00 * C.c22 - C.c02 * C.c02;
  const double A22 = C.c00 * C.c11 - C.c01 * C.c01;
  const double A01 = C.c02 * C.c12 - C.c01 * C.c22;
  const double A02 = C.c01 * C.c12 - C.c02 * C.c11;
  const double t = C.c00 + C.c11 + C.c22;
  const double c1 = A00 + A11 + A22;
  const double det = C.c00 * A00 + C.c01 * A01 + C.c02 * A02;
  float k1, k2, k3;
  const float ft = (float)t;
  trig_cubic(ft, (float)c1, (float)det, k1, k2, k3);
  return curvature_from(t, c1, det, ft, k1, k2, k3);
}

// Explicit fits (fitting.py:582-621) on the centred moments of the space's monomials
// (m0, m1, m2) = (X, Y, Z) standard or (tx, ty, 1/Z) rgbd: the target m2 regressed on
// (m0, m1, 1).  Solved centred ([a b] from the 2x2 covariance, c = mu2 - a mu0 - b mu1),
// which equals the reference's uncentred normal equations; the residual sum of squares
// C22 - [a b].[C02 C12] equals its sum(b^2) - alpha.rhs.  degenerate replays the
// reference's Cholesky pivot test (cholesky3, fitting.py:264-293) on the uncentred
// matrix [[S00, S01, S0], [S01, S11, S1], [S0, S1, n]].
struct ExplicitFit {
  double a, b, c, ss;
  bool degenerate;
};
__device__ __forceinline__ void explicit_solve(const Sym3& C, double m0, double m1, double m2,
                                               double n, ExplicitFit& out) {
  const double det2 = fma(C.c00, C.c11, -C.c01 * C.c01);
  const double idet = det2 > 0.0 ? rcp_fast(det2) : 0.0;
  out.a = fma(C.c11, C.c02, -C.c01 * C.c12) * idet;
  out.b = fma(C.c00, C.c12, -C.c01 * C.c02) * idet;
  out.c = m2 - out.a * m0 - out.b * m1;
  // three samples (MIN_SAMPLES of the explicit fits): the plane interpolates them, the residual
  // is exactly 0 -- the centred difference below would only return the cancellation of an
  // ill-conditioned 2x2 solve (e.g. nearly collinear X-Y positions)
  out.ss = n == 3.0 ? 0.0 : C.c22 - (out.a * C.c02 + out.b * C.c12);
  // uncentred matrix and its Cholesky pivots
  const double M00 = fma(n * m0, m0, C.c00), M01 = fma(n * m0, m1, C.c01), M11 = fma(n * m1, m1, C.c11);
  const double M02 = n * m0, M12 = n * m1;
  const double trace = M00 + M11 + n;
  const double fl = 1e-12 * trace;
  const double p0 = M00;
  const double l10 = M01 * rcp_fast(M00);
  const double p1 = fma(-l10, M01, M11);
  // p2 = n - [M02 M12] M2^-1 [M02 M12]^T = n / (1 + n mu^T C2^-1 mu)
  const double q = (m0 * fma(C.c11, m0, -C.c01 * m1) + m1 * fma(C.c00, m1, -C.c01 * m0)) * idet;
  const double p2 = det2 > 0.0 ? n * rcp_fast(fma(n, q, 1.0)) : 0.0;
  (void)M02;
  (void)M12;
  out.degenerate = !(trace > 0.0) || p0 <= fl || p1 <= fl || p2 <= fl;
}

// Newton on the quartic from below until the step is below 1e-13 relative (out of line).
static __device__ __noinline__ double newton_converge(double q3, double q2, double q1, double q0, double l) {
  for (int it = 0; it < 64; ++it) {
    const double x2 = l * l;
    const double G = fma(fma(l - q3, l, q2), x2, fma(-q1, l, q0));
    const double dG = fma(fma(fma(4.0, l, -3.0 * q3), l, 2.0 * q2), l, -q1);
    const double step = G * rcp_approx(dG);
    l -= step;
    if (!(fabs(step) > 1e-13 * l)) break;
  }
  return l;
}

// Near-tie lam1 ~ lam2 (rare): exact deflation of the quartic.  lam4 (the largest
// root, ~n(1+nu)) and then lam3 are found by Newton from above (upper bounds q3 and
// lam1+lam2+lam3), each divided out by backward deflation (stable for the largest
// root); the quadratic left over has roots lam1 <= lam2, solved cancellation-free.
static __device__ __noinline__ void tie_deflation(double q3, double q2, double q1, double q0, double& lam,
                                           double& lam2) {
  double l4 = q3;
  for (int it = 0; it < 64; ++it) {
    const double G = fma(fma(fma(l4 - q3, l4, q2), l4, -q1), l4, q0);
    const double dG = fma(fma(fma(4.0, l4, -3.0 * q3), l4, 2.0 * q2), l4, -q1);
    const double step = G * rcp_approx(dG);
    l4 -= step;
    if (!(fabs(step) > 1e-15 * l4)) break;
  }
  const double i4 = rcp_fast(l4);
  const double h0 = -q0 * i4;             // -lam1 lam2 lam3
  const double h1 = (q1 + h0) * i4;       // lam1 lam2 + lam1 lam3 + lam2 lam3
  const double h2 = (h1 - q2) * i4;       // -(lam1 + lam2 + lam3)
  double l3 = -h2;
  for (int it = 0; it < 64; ++it) {
    const double H = fma(fma(l3 + h2, l3, h1), l3, h0);
    const double dH = fma(fma(3.0, l3, 2.0 * h2), l3, h1);
    const double step = H * rcp_approx(dH);
    l3 -= step;
    if (!(fabs(step) > 1e-15 * l3)) break;
  }
  const double i3 = rcp_fast(l3);
  const double e0 = -h0 * i3;             // lam1 lam2
  const double e1 = (e0 - h1) * i3;       // -(lam1 + lam2)
  const double disc = (double)fsqrt((float)fmax(fma(e1, e1, -4.0 * e0), 0.0));
  const double den = disc - e1;           // 2 lam2
  lam = den > 0.0 ? 2.0 * e0 * rcp_fast(den) : 0.0;
  lam2 = 0.5 * den;
}

// Smallest eigenpair of S = [[C + n mu mu^T, n mu], [n mu^T, n]] (the
// uncentred scatter of [m0, m1, m2, 1], fitting.py:339-381) through the
// Schur complement on the constant monomial: C u = lam (I + beta mu mu^T) u,
// beta = n/(n - lam), s = -beta mu.u.  det(S - l I) is the quartic
//   l^4 - q3 l^3 + q2 l^2 - q1 l + q0   with
//   q3 = n + t + n nu, q2 = n t + c1 + n (t nu - mu.C.mu),
//   q1 = n c1 + det C + n mu.adj(C).mu,  q0 = n det C.
// lam1 is found by fp64 Newton from a lower bound (fp32 trigonometric seeds
// of the beta=1 cubic), or -- when lam1 ~ lam2 (near-tie) -- by exact
// backward deflation of the quartic's two largest roots and the remaining
// quadratic.  The eigenvector is the
// dominant column of adj(C - lam (I + beta mu mu^T)).
// Curvature lam_min(C)/tr(C) uses the same seeds/Newton/
// deflation on det(C - l I).
template <bool MID_SEED = false>
__device__ __forceinline__ void solve_window(const Sym3& C, double m0, double m1, double m2,
                                             double n, WindowFit& out) {
  const double c00 = C.c00, c01 = C.c01, c02 = C.c02, c11 = C.c11, c12 = C.c12, c22 = C.c22;
  const double A00 = c11 * c22 - c12 * c12;
  const double A11 = c00 * c22 - c02 * c02;
  const double A22 = c00 * c11 - c01 * c01;
  const double A01 = c02 * c12 - c01 * c22;
  const double A02 = c01 * c12 - c02 * c11;
  const double A12 = c01 * c02 - c00 * c12;
  const double t = c00 + c11 + c22;
  const double c1 = A00 + A11 + A22;
  const double det = c00 * A00 + c01 * A01 + c02 * A02;
  const double nu = m0 * m0 + m1 * m1 + m2 * m2;
  const double Cm0 = c00 * m0 + c01 * m1 + c02 * m2;
  const double Cm1 = c01 * m0 + c11 * m1 + c12 * m2;
  const double Cm2 = c02 * m0 + c12 * m1 + c22 * m2;
  const double mm = m0 * Cm0 + m1 * Cm1 + m2 * Cm2;
  const double Am0 = A00 * m0 + A01 * m1 + A02 * m2;
  const double Am1 = A01 * m0 + A11 * m1 + A12 * m2;
  const double Am2 = A02 * m0 + A12 * m1 + A22 * m2;
  const double aa = m0 * Am0 + m1 * Am1 + m2 * Am2;
  const double q3 = n + t + n * nu;
  const double q2 = fma(n, t, c1) + n * (t * nu - mm);
  const double q1 = fma(n, c1, det) + n * aa;
  const double q0 = n * det;

  // fp32 seeds: roots g1 <= g2 <= g3 of the pencil's cubic at beta = 1,
  //   (1 + nu) l^3 - (t + t nu - mu.C.mu) l^2 + (c1 + mu.adj(C).mu) l - det C.
  // lam1(beta) decreases with beta and d lam/d beta >= -lam/beta, so with
  // beta(lam1) <= n/(n - g1):  g1 (1 - g1/n) <= lam1 <= g1.
  float g1, g2, g3, k1, k2, k3;
  const float ft = (float)t, fc1 = (float)c1, fdet = (float)det, fnu = (float)nu, fn = (float)n;
  {
    const float inv = frcp(1.0f + fnu);
    trig_cubic((float)(t + t * nu - mm) * inv, (float)(c1 + aa) * inv, fdet * inv, g1, g2, g3);
    trig_cubic(ft, fc1, fdet, k1, k2, k3);
  }
  const float grel = g1 * frcp(fn);

  double lam, lam2;
  const bool tie = (g2 - g1) < 0.05f * g2;
  // (A) Newton on the quartic from the lower bound: monotone convergence; the
  // curvature's two Newton steps on det(C - l I) run interleaved with the first two.
  // Quadratic convergence, e_{k+1} ~ e_k^2 / (relative gap >= 5%): from
  // e0 <= 1e-4 + lam1/n two steps leave < 1e-11 when lam1/n <= 1e-4, three when
  // <= 1e-3; pathological windows (lam/n not small) iterate to convergence.
  auto newton = [&](double x) {
    const double x2 = x * x;
    const double G = fma(fma(x - q3, x, q2), x2, fma(-q1, x, q0));
    const double dG = fma(fma(fma(4.0, x, -3.0 * q3), x, 2.0 * q2), x, -q1);
    return G * rcp_approx(dG);
  };
  CurvSeed cs = curv_seed(k1, k2, k3);
  double l;
  if constexpr (MID_SEED) {
    // seed at the middle of [g1 (1 - g1/n), g1]: error <= grel/2 + the fp32 seed error, so
    // one step leaves e^2 / gap < 1e-7 relative for grel <= 1e-4 (99% of the C2 windows of
    // both forms); above, two more steps (and iteration to convergence beyond 1e-3) follow
    l = (double)(g1 * fmaf(-0.5f, grel, 1.0f));
    l -= newton(l);
    cs.x = curv_newton(t, c1, det, cs.x);
    if (grel > 1e-4f) l -= newton(l);
  } else {
    l = (double)(g1 * fmaf(-1.0f, grel, 1.0f - 1e-4f));
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      l -= newton(l);
      // one step suffices for the curvature: outside the close (< 5% gap) cases, which
      // take curvature_slow, the fp32 seed is within ~1e-4 and one quadratic step leaves
      // < 1e-6 relative
      if (it == 0) cs.x = curv_newton(t, c1, det, cs.x);
    }
  }
  if (!tie) {
    if (grel > 1e-4f) l -= newton(l);
    if (grel > 1e-3f) l = newton_converge(q3, q2, q1, q0, l);  // large-residual windows (rare)
    lam = l;
    lam2 = (double)g2;
  } else {
    // (B) near-tie lam1 ~ lam2: exact deflation (rare)
    tie_deflation(q3, q2, q1, q0, lam, lam2);
  }

  // eigenvector: dominant column of adj(C - lam B), B = I + beta mu mu^T
  // beta = n / (n - lam) = 1 + lam / (n - lam): one Newton step on the reciprocal
  // (~1e-12 relative) is far below what the lam * beta terms need
  double beta;
  {
    const double dn = n - lam;
    double r = rcp_approx(dn);
    r = fma(r, fma(-dn, r, 1.0), r);
    beta = fma(lam, r, 1.0);
  }
  const double gam = lam * beta;
  const double E00 = c00 - lam - gam * m0 * m0;
  const double E11 = c11 - lam - gam * m1 * m1;
  const double E22 = c22 - lam - gam * m2 * m2;
  const double E01 = c01 - gam * m0 * m1;
  const double E02 = c02 - gam * m0 * m2;
  const double E12 = c12 - gam * m1 * m2;
  // the six cofactors of the symmetric E; the column with the largest diagonal is taken
  // by selects (no branches)
  const double B00 = E11 * E22 - E12 * E12;
  const double B11 = E00 * E22 - E02 * E02;
  const double B22 = E00 * E11 - E01 * E01;
  const double B01 = E02 * E12 - E01 * E22;
  const double B02 = E01 * E12 - E02 * E11;
  const double B12 = E01 * E02 - E00 * E12;
  double u0, u1, u2;
  {
    const double a0 = fabs(B00), a1 = fabs(B11), a2 = fabs(B22);
    const bool s0 = a0 >= a1 && a0 >= a2;
    const bool s1 = !s0 && a1 >= a2;
    u0 = s0 ? B00 : s1 ? B01 : B02;
    u1 = s0 ? B01 : s1 ? B11 : B12;
    u2 = s0 ? B02 : s1 ? B12 : B22;
    const double amax = s0 ? a0 : s1 ? a1 : a2;
    if (amax == 0.0) {  // all diagonal cofactors 0, rank <= 1: any null vector
      u0 = 0.0;
      u1 = 0.0;
      u2 = 1.0;
    }
  }
  out.u0 = u0;
  out.u1 = u1;
  out.u2 = u2;
  out.s = -beta * (m0 * u0 + m1 * u1 + m2 * u2);
  out.lam = lam;

  // degenerate: gap <= 1e-9 ||S||_F (fitting.py:552-554);
  // ||S||_F^2 = ||C||_F^2 + 2 n mu.C.mu + n^2 (1 + nu)^2
  // (trace(S)/2 <= ||S||_F <= trace(S) = q3 for PSD S: only near-ties need the norm)
  {
    const double gap = lam2 - lam;
    if (gap > 1e-9 * q3) {
      out.degenerate = false;
    } else {
      const double fc = c00 * c00 + c11 * c11 + c22 * c22 + 2.0 * (c01 * c01 + c02 * c02 + c12 * c12);
      const double np1 = n * (1.0 + nu);
      const double fro2 = fc + 2.0 * n * mm + np1 * np1;
      out.degenerate = gap <= 0.0 || gap * gap <= 1e-18 * fro2;
    }
  }

  // curvature: lam_min(C) / tr(C)
  out.kappa = curv_finish(cs, t, c1, det, ft, k1, k2, k3);
}

// Common-case path of solve_window<true> as straight-line code: the same seeds, quartic
// Newton steps from the middle of the seed bracket (one when lam/n <= 1e-4, two up to 1e-3,
// three up to 1e-2), one curvature Newton step (from below lam_min, or -- close bottom pair
// -- from above lam_max followed by the deflation), the dominant adjugate column.  Returns
// false when the window needs the robust path (solve_window): a pencil near-tie (< 5% gap),
// a curvature spectrum with both pairs close, lam/n above 1e-2, an adjugate of rank 0, a
// non-positive upper spectrum, or a gap small enough to ask the degenerate test
// (fitting.py:552-554).  `out` is then unspecified.
__device__ __forceinline__ bool solve_fast(const Sym3& C, double m0, double m1, double m2, double n, float finvn,
                                           WindowFit& out) {
  const double c00 = C.c00, c01 = C.c01, c02 = C.c02, c11 = C.c11, c12 = C.c12, c22 = C.c22;
  const double A00 = c11 * c22 - c12 * c12;
  const double A11 = c00 * c22 - c02 * c02;
  const double A22 = c00 * c11 - c01 * c01;
  const double A01 = c02 * c12 - c01 * c22;
  const double A02 = c01 * c12 - c02 * c11;
  const double A12 = c01 * c02 - c00 * c12;
  const double t = c00 + c11 + c22;
  const double c1 = A00 + A11 + A22;
  const double det = c00 * A00 + c01 * A01 + c02 * A02;
  const double nu = m0 * m0 + m1 * m1 + m2 * m2;
  const double Cm0 = c00 * m0 + c01 * m1 + c02 * m2;
  const double Cm1 = c01 * m0 + c11 * m1 + c12 * m2;
  const double Cm2 = c02 * m0 + c12 * m1 + c22 * m2;
  const double mm = m0 * Cm0 + m1 * Cm1 + m2 * Cm2;
  const double Am0 = A00 * m0 + A01 * m1 + A02 * m2;
  const double Am1 = A01 * m0 + A11 * m1 + A12 * m2;
  const double Am2 = A02 * m0 + A12 * m1 + A22 * m2;
  const double aa = m0 * Am0 + m1 * Am1 + m2 * Am2;
  const double q3 = n + t + n * nu;
  const double q2 = fma(n, t, c1) + n * (t * nu - mm);
  const double q1 = fma(n, c1, det) + n * aa;
  const double q0 = n * det;

  // fp32 seeds, both cubics in lock step: x = the pencil at beta = 1 (normalised by 1 + nu),
  // y = det(C - l I).  t, nu and t + t nu - mm (>= t) are positive: integer-pipe conversions
  float g1, g2, g3, k1, k2, k3;
  const float ft = pos_d2f(t), fdet = (float)det;
  {
    const float inv = frcp(1.0f + pos_d2f(nu));
    const float2 A2 = mul2(f2(pos_d2f(t + t * nu - mm), ft), f2(inv, 1.0f));
    const float2 A1 = mul2(f2((float)(c1 + aa), (float)c1), f2(inv, 1.0f));
    const float2 A0 = mul2(f2(fdet), f2(inv, 1.0f));
    float2 r1, r2, r3;
    trig_cubic2(A2, A1, A0, r1, r2, r3);
    g1 = r1.x, g2 = r2.x, g3 = r3.x, k1 = r1.y, k2 = r2.y, k3 = r3.y;
  }
  const float grel = g1 * finvn;
  // curvature: Newton on lam_min from just below k1, or on lam_max from k3 when the bottom
  // pair is close (then lam_1 from lam_1 + lam_2 = t - lam_max, lam_1 lam_2 = det / lam_max)
  const bool top = !((k2 - k1) >= 0.05f * k2);
  // NaN-safe: every comparison is written so that NaN fails it
  bool ok = ((g2 - g1) >= 0.05f * g2) & (grel <= 1e-2f) & (k2 > 0.0f) & (!top | ((k3 - k2) >= 0.05f * k3));

  auto newton = [&](double x) {
    const double x2 = x * x;
    const double G = fma(fma(x - q3, x, q2), x2, fma(-q1, x, q0));
    const double dG = fma(fma(fma(4.0, x, -3.0 * q3), x, 2.0 * q2), x, -q1);
    return G * rcp_approx(dG);
  };
  // quartic Newton from the middle of [g1 (1 - g1/n), g1] and the curvature step
  // (independent chains, interleaved)
  double l = pos_f2d(fmaxf(g1 * fmaf(-0.5f, grel, 1.0f), 1e-30f));
  double x = pos_f2d(fmaxf(top ? k3 : k1 * (1.0f - 1e-5f), 1e-30f));
  {
    const double P = fma(fma(t - x, x, -c1), x, det);
    const double dP = fma(fma(-3.0, x, 2.0 * t), x, -c1);
    l -= newton(l);
    x -= P * rcp_approx(dP);
  }
  if (grel > 1e-4f) l -= newton(l);
  if (grel > 1e-3f) l -= newton(l);
  const double lam = l;

  double beta;
  {
    const double dn = n - lam;
    double r = rcp_approx(dn);
    r = fma(r, fma(-dn, r, 1.0), r);
    beta = fma(lam, r, 1.0);
  }
  // eigenvector: the dominant column of adj(C - lam B), B = I + beta mu mu^T (error
  // ~ eps ||C|| / gap; the cheaper adj(C - lam I) mu, also parallel to it, amplifies an
  // error in lam by |mu| |u| / |mu.u|, which noise-dominated windows make large)
  const double gam = lam * beta;
  const double E00 = c00 - lam - gam * m0 * m0;
  const double E11 = c11 - lam - gam * m1 * m1;
  const double E22 = c22 - lam - gam * m2 * m2;
  const double E01 = c01 - gam * m0 * m1;
  const double E02 = c02 - gam * m0 * m2;
  const double E12 = c12 - gam * m1 * m2;
  const double B00 = E11 * E22 - E12 * E12;
  const double B11 = E00 * E22 - E02 * E02;
  const double B22 = E00 * E11 - E01 * E01;
  const double B01 = E02 * E12 - E01 * E22;
  const double B02 = E01 * E12 - E02 * E11;
  const double B12 = E01 * E02 - E00 * E12;
  // the column is chosen on the high words of |B_kk| (integer pipe; any column within 2^-20
  // of the largest diagonal is as good); all three below 2^-1022 go to the robust path
  const int a0 = __double2hiint(B00) & 0x7fffffff, a1 = __double2hiint(B11) & 0x7fffffff,
            a2 = __double2hiint(B22) & 0x7fffffff;
  const bool s0 = a0 >= a1 && a0 >= a2;
  const bool s1 = !s0 && a1 >= a2;
  const double u0 = s0 ? B00 : s1 ? B01 : B02;
  const double u1 = s0 ? B01 : s1 ? B11 : B12;
  const double u2 = s0 ? B02 : s1 ? B12 : B22;
  ok &= (a0 | a1 | a2) >= 0x00100000;
  out.u0 = u0;
  out.u1 = u1;
  out.u2 = u2;
  out.s = -beta * (m0 * u0 + m1 * u1 + m2 * u2);
  out.lam = lam;
  // degenerate (fitting.py:552-554) cannot hold while gap > 1e-9 trace(S) >= 1e-9 ||S||_F
  ok &= ((double)g2 - lam) > 1e-9 * q3;
  out.degenerate = false;
  float kmin = (float)x;
  if (top) {
    const double S = t - x;
    const double Pp = det * rcp_fast(x);
    const float D = (float)fma(S, S, -4.0 * Pp);  // (lam_2 - lam_1)^2, cancellation-free in fp64
    kmin = 2.0f * (float)Pp * frcp((float)S + fsqrt(fmaxf(D, 0.0f)));
  }
  out.kappa = t > 0.0 ? kmin * frcp(ft) : 0.0f;
  return ok;
}

// the robust solve for the windows solve_fast declines (out of line: its registers stay off
// the fast path)
static __device__ __noinline__ void solve_window_robust(const Sym3& C, double m0, double m1, double m2, double n,
                                                        WindowFit& out) {
  solve_window<true>(C, m0, m1, m2, n, out);
}

// canonical sign + unit normal / offset (fitting.py:76-94 and SURVEY A18)
__device__ __forceinline__ void finish_plane(double a, double b, double c, double d, float& nx,
                                             float& ny, float& nz, float& off) {
  // exact power-of-two rescale so the fp32 conversion neither over- nor underflows
  const int hm = max(max(__double2hiint(a) & 0x7ff00000, __double2hiint(b) & 0x7ff00000),
                     max(__double2hiint(c) & 0x7ff00000, __double2hiint(d) & 0x7ff00000));
  const int e = hm >> 20;
  const double sc = __hiloint2double((2046 - e) << 20, 0);  // 2^(1023 - e)
  const float fa = (float)(a * sc), fb = (float)(b * sc), fc = (float)(c * sc),
              fd = (float)(d * sc);
  // |u_k| / |u| > 1e-9 on the unit 4-vector.  After the rescale the largest component lies
  // in [1, 2), so 1 <= |u| < 4: |c| >= 4e-9 settles it on c (nearly every window); otherwise
  // the exact test in order c, b, a, d, squared (no reciprocal square root)
  float sign = fc > 0.0f ? 1.0f : -1.0f;
  if (!(fabsf(fc) >= 4e-9f)) {
    const float e4 = 1e-18f * (fa * fa + fb * fb + fc * fc + fd * fd);
    sign = 1.0f;
    if (fc * fc > e4) sign = fc > 0.0f ? 1.0f : -1.0f;
    else if (fb * fb > e4) sign = fb > 0.0f ? 1.0f : -1.0f;
    else if (fa * fa > e4) sign = fa > 0.0f ? 1.0f : -1.0f;
    else if (fd < 0.0f) sign = -1.0f;
  }
  const float in3 = sign * frsqrt(fa * fa + fb * fb + fc * fc);
  nx = fa * in3;
  ny = fb * in3;
  nz = fc * in3;
  off = fd * in3;
}

// canonicalize_implicit (fitting.py:76-94) in fp64
__device__ __forceinline__ void canonical4(double a, double b, double c, double d, double* out) {
  const double nrm = sqrt(a * a + b * b + c * c + d * d);
  double u[4] = {a / nrm, b / nrm, c / nrm, d / nrm};
  double sign = 1.0;
  const int order[4] = {2, 1, 0, 3};
  for (int k = 0; k < 4; ++k) {
    if (fabs(u[order[k]]) > 1e-9) {
      sign = u[order[k]] > 0.0 ? 1.0 : -1.0;
      break;
    }
  }
  for (int k = 0; k < 4; ++k) out[k] = sign * u[k];
}


}  // namespace rf_dev
