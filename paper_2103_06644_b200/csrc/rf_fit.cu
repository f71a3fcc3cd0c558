// rf_fit.cu -- sm_100a kernels + C ABI for the per-pixel windowed implicit
// plane fit (reference: rangefit fitting.py / integral.py, see
// include/rangefit_b200.h for the boundary and DESIGN.md for the design).
//
// One kernel per formulation.  A CTA owns a TW x TH tile of output pixels of
// one frame and stages its (TW+2r) x (TH+2r) input halo once:
//   1. load   : depth -> validity mask (synth.py:84,111-114) -> fp64 primary
//               p = 1/Z (disparity form, integral.py:211-214) or Z (standard),
//               0 for invalid pixels, into shared memory;
//   2. columns: running vertical window sums of the p-moments (fp64) and of
//               the validity geometry (int32), one thread per halo column;
//   3. rows   : each thread owns KSEG consecutive pixels of one output row,
//               forms the horizontal window sums with a running update,
//               giving the window's centred scatter C (3x3), mean mu and
//               count n in tile-local coordinates (exact integer geometry,
//               fp64 depth moments -- never image-global magnitudes);
//   4. solve  : smallest eigenpair of the uncentred 4x4 scatter through its
//               Schur complement on the constant monomial (solve_window),
//               curvature, canonical sign, outputs (fp32) and status byte.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/rangefit_b200.h"

namespace {

constexpr int TW = 64;       // output tile width  (pixels)
constexpr int TH = 16;       // output tile height (pixels)
constexpr int KSEG = 4;      // consecutive output pixels per thread
constexpr int NTHREADS = (TW / KSEG) * TH;  // 256
constexpr int MAX_RADIUS = 32;
#ifndef RF_ABLATE
#define RF_ABLATE 0
#endif
#ifndef RF_STAGE_OUTPUTS
#define RF_STAGE_OUTPUTS 1
#endif
#ifndef RF_MIN_BLOCKS
#define RF_MIN_BLOCKS 2
#endif

constexpr int VAR_STD = 0;   // implicit-standard
constexpr int VAR_DF = 1;    // implicit-rgbd (disparity form)

struct OutPlanes {
  float* normal;
  float* offset;
  float* residual;
  float* curvature;
  uint8_t* status;
};

struct KParams {
  const void* depth;
  const uint8_t* mask;
  const double* tan_x;  // [W]
  const double* tan_y;  // [H]
  double ifx, ify;
  int64_t row_pitch;
  int64_t frame_stride;
  int64_t out_frame;    // H*W
  int64_t batch;
  int H, W, r, dtype;
  int do_imp, do_exp;  // implicit / explicit fit of this kernel's space requested
  OutPlanes imp, exp;  // implicit-* / explicit-* output planes of the space
};

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
  const float isp = rsqrtf(p);
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
__device__ __forceinline__ float curvature_from(double t, double c1, double det, float ft, float k1,
                                                float k2, float k3) {
  {
    double lk;
    const bool top = (k3 - k2) * k2 > (k2 - k1) * k3;  // top gap better separated
    if (!top) {
      // Newton from below lam_min (monotone).  With a well separated bottom pair
      // (relative gap > 20%) the fp32 seed (deflated, ~2e-6 relative) already meets
      // the 1e-4 curvature tolerance with margin; otherwise polish in fp64.
      double l = (double)k1;
      if ((k2 - k1) < 0.2f * k2) {
        l *= (1.0 - 1e-5);
        auto newton = [&](double x) {
          const double P = fma(fma(t - x, x, -c1), x, det);
          const double dP = fma(fma(-3.0, x, 2.0 * t), x, -c1);
          return P * rcp_approx(dP);
        };
        l -= newton(l);
        l -= newton(l);
        if ((k2 - k1) < 0.05f * k2) {  // close bottom pair (rare): iterate to convergence
          for (int it = 0; it < 64; ++it) {
            const double step = newton(l);
            l -= step;
            if (!(fabs(step) > 1e-10 * l)) break;
          }
        }
      }
      lk = l;
    } else {
      // near-tie at the bottom: Newton from above lam_max (well separated here),
      // then deflate; lam_max only needs ~1e-10 for a 1e-5 curvature
      double l = fmin((double)k3 * (1.0 + 1e-5), t);
      auto newton = [&](double x) {
        const double P = fma(fma(t - x, x, -c1), x, det);
        const double dP = fma(fma(-3.0, x, 2.0 * t), x, -c1);
        return P * rcp_approx(dP);
      };
      l -= newton(l);
      l -= newton(l);
      if ((k3 - k2) < 0.05f * k3) {  // top pair close too (rare): iterate to convergence
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
  out.ss = C.c22 - (out.a * C.c02 + out.b * C.c12);
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
  if (!tie) {
    // (A) Newton on the quartic from the lower bound: monotone convergence,
    // stop once the step is below 1e-9 relative (the remaining error is then
    // ~step^2/gap).  Three steps in the common case; pathological windows
    // (lam/n not small) take longer.
    double l = (double)(g1 * fmaf(-1.0f, grel, 1.0f - 1e-4f));
    auto newton = [&](double x) {
      const double x2 = x * x;
      const double G = fma(fma(x - q3, x, q2), x2, fma(-q1, x, q0));
      const double dG = fma(fma(fma(4.0, x, -3.0 * q3), x, 2.0 * q2), x, -q1);
      return G * rcp_approx(dG);
    };
    // quadratic convergence, e_{k+1} ~ e_k^2 / (relative gap >= 5%): from
    // e0 <= 1e-4 + lam1/n two steps leave < 1e-11 when lam1/n <= 1e-4, three when <= 1e-3
    l -= newton(l);
    l -= newton(l);
    if (grel > 1e-4f) l -= newton(l);
    if (grel > 1e-3f) {  // large residual windows (rare): iterate to convergence
      for (int it = 0; it < 64; ++it) {
        const double step = newton(l);
        l -= step;
        if (!(fabs(step) > 1e-13 * l)) break;
      }
    }
    lam = l;
    lam2 = (double)g2;
  } else {
    // (B) near-tie lam1 ~ lam2: exact deflation of the quartic.  lam4 (the
    // largest root, ~n(1+nu)) and then lam3 are found by Newton from above
    // (upper bounds q3 and lam1+lam2+lam3), each divided out by backward
    // deflation (stable for the largest root); the quadratic left over has
    // roots lam1 <= lam2, solved in the cancellation-free form.
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

  // eigenvector: dominant column of adj(C - lam B), B = I + beta mu mu^T
  const double beta = n * rcp_fast(n - lam);
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
  double u0, u1, u2;
  {
    const double a0 = fabs(B00), a1 = fabs(B11), a2 = fabs(B22);
    if (a0 >= a1 && a0 >= a2) {
      u0 = B00;
      u1 = E02 * E12 - E01 * E22;
      u2 = E01 * E12 - E02 * E11;
    } else if (a1 >= a2) {
      u0 = E02 * E12 - E01 * E22;
      u1 = B11;
      u2 = E01 * E02 - E00 * E12;
    } else {
      u0 = E01 * E12 - E02 * E11;
      u1 = E01 * E02 - E00 * E12;
      u2 = B22;
    }
    if (a0 == 0.0 && a1 == 0.0 && a2 == 0.0) {  // rank <= 1: any null vector
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
  out.kappa = curvature_from(t, c1, det, ft, k1, k2, k3);
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
  const float n4 = rsqrtf(fa * fa + fb * fb + fc * fc + fd * fd);
  float sign = 1.0f;
  if (fabsf(fc * n4) > 1e-9f) sign = fc > 0.0f ? 1.0f : -1.0f;
  else if (fabsf(fb * n4) > 1e-9f) sign = fb > 0.0f ? 1.0f : -1.0f;
  else if (fabsf(fa * n4) > 1e-9f) sign = fa > 0.0f ? 1.0f : -1.0f;
  else if (fd < 0.0f) sign = -1.0f;
  const float in3 = sign * rsqrtf(fa * fa + fb * fb + fc * fc);
  nx = fa * in3;
  ny = fb * in3;
  nz = fc * in3;
  off = fd * in3;
}

// ---- TMA / mbarrier helpers (sm_90+ async proxy; SASS UTMALDG + SYNCS)
// residue-major column stride of the column-sum buffers (VQ = 4 mod 8 spreads the banks)
__host__ __device__ __forceinline__ int vq_of(int hw) {
  int q = (hw + 3) / 4;
  return q + ((4 - q % 8) + 8) % 8;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// one TMA box (HWP x HH x 1 elements) of the [B, H, W] depth tensor; coordinates past
// the right/bottom edge are zero-filled (= invalid depth).  Measured on this
// sm_100a/driver: a negative box origin, or an x origin that is not 16-byte
// aligned, raises an illegal-instruction fault -- so the caller aligns the box
// origin down to 16 bytes, clamps it to >= 0, and masks the left/top halo itself.
__device__ __forceinline__ int box_x(int x, int al) { return x > 0 ? (x / al) * al : 0; }
__device__ __forceinline__ void tma_load_tile(void* dst, const CUtensorMap* tmap, int x, int y, int z,
                                              uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

struct TileGeom {
  int64_t frame;
  int x0, y0;
};

__device__ __forceinline__ TileGeom tile_of(int64_t t, int ntx, int nty) {
  TileGeom g;
  const int64_t per_frame = (int64_t)ntx * nty;
  g.frame = t / per_frame;
  const int rem = (int)(t - g.frame * per_frame);
  const int ty = rem / ntx;
  g.y0 = ty * TH;
  g.x0 = (rem - ty * ntx) * TW;
  return g;
}

// depth element -> fp64 primary p (0 = invalid): DepthImage validity (synth.py:84, 111-114)
template <int VAR>
__device__ __forceinline__ double primary_from_f32(float zf, bool mask_ok) {
  const bool valid = mask_ok && (zf > 0.0f) && (zf <= 3.402823466e38f);  // isfinite & > 0
  const double z = (double)zf;
  return valid ? (VAR == VAR_DF ? rcp_fast(z) : z) : 0.0;
}
template <int VAR>
__device__ __forceinline__ double primary_from_u16(unsigned short mm, bool mask_ok) {
  if (!(mask_ok && mm > 0)) return 0.0;
  const double z = __ddiv_rn((double)mm, 1000.0);  // mm / 1000.0 exactly as the reference
  return VAR == VAR_DF ? rcp_fast(z) : z;
}

// One persistent CTA walks tiles t = blockIdx.x, blockIdx.x + gridDim.x, ...
// With USE_TMA the raw halo tile of the NEXT tile is fetched by TMA into the
// other of two shared buffers while this tile's column and row passes run.
// RT > 0: compile-time window radius (all halo geometry and shared-memory offsets
// fold to constants); RT == 0: runtime radius P.r.
// EXP: explicit fits compiled in (false keeps the implicit-only kernel lean).
template <int VAR, bool USE_TMA, int RT, bool EXP>
__global__ void __launch_bounds__(NTHREADS, RF_MIN_BLOCKS)
    fit_tile_kernel(const KParams P, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) unsigned char smem_dyn[];
  // TMA destinations must be 128-byte aligned: align the dynamic base explicitly
  unsigned char* smem_raw = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_dyn) + 127) & ~uintptr_t(127));
  const int r = RT > 0 ? RT : P.r;
  const int HW_ = TW + 2 * r;  // halo width
  const int HH_ = TH + 2 * r;  // halo height
  constexpr int NVD = VAR == VAR_DF ? 3 : 5;  // fp64 vertical channels
  constexpr int NVI = VAR == VAR_DF ? 3 : 1;  // int vertical channels
  const int esz = P.dtype == RF_DEPTH_U16_MM ? 2 : 4;
  const int al = 16 / esz;  // TMA box x origin must be 16-byte aligned
  const int HWP = (HW_ + al - 1 + 7) & ~7;  // TMA box width (covers the alignment shift)
  const int raw_bytes = USE_TMA ? ((HH_ * HWP * esz + 127) & ~127) : 0;
  unsigned char* raw0 = smem_raw;
  unsigned char* raw1 = smem_raw + raw_bytes;
  double* prim = reinterpret_cast<double*>(smem_raw + 2 * raw_bytes);  // [HH_][HW_]
  // column sums are stored residue-major: column c at (c % 4) * VQ + c / 4, so the row
  // pass (threads 4 columns apart) reads consecutive addresses -- no bank conflicts.
  const int VQ = vq_of(HW_);
  const int VRS = 4 * VQ;                                                // row stride
  double* vd = prim + HH_ * HW_;                                         // [NVD][TH][VRS]
  int* vi = reinterpret_cast<int*>(vd + NVD * TH * VRS);                 // [NVI][TH][VRS]
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(vi + NVI * TH * VRS) + 7) & ~uintptr_t(7));

  const int tid = threadIdx.x;
  const int ntx = (P.W + TW - 1) / TW, nty = (P.H + TH - 1) / TH;
  const int64_t total = (int64_t)ntx * nty * P.batch;
  const uint32_t box_bytes = (uint32_t)(HH_ * HWP * esz);

  if (USE_TMA) {
    if (tid == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0 && blockIdx.x < total) {
      const TileGeom g = tile_of(blockIdx.x, ntx, nty);
      mbar_expect_tx(&bars[0], box_bytes);
      tma_load_tile(raw0, &tmap, box_x(g.x0 - r, al), max(g.y0 - r, 0), (int)g.frame, &bars[0]);
    }
  }

  int it = 0;
  for (int64_t t = blockIdx.x; t < total; t += gridDim.x, ++it) {
    const TileGeom g = tile_of(t, ntx, nty);
    const int64_t frame = g.frame;
    const int x0 = g.x0, y0 = g.y0;

    // ---- 1. halo tile -> primary
    if (USE_TMA) {
      const int b = it & 1;
      mbar_wait(&bars[b], (uint32_t)((it >> 1) & 1));
      const unsigned char* raw = b ? raw1 : raw0;
      const int bx = box_x(x0 - r, al), by = max(y0 - r, 0);
      const int sx = (x0 - r) - bx, sy = (y0 - r) - by;  // raw index = tile index + shift
      for (int e = tid; e < HH_ * HW_; e += NTHREADS) {
        const int row = e / HW_, col = e - row * HW_;
        double p = 0.0;
        if (row + sy >= 0 && col + sx >= 0) {
          bool mask_ok = true;
          if (P.mask) {
            const int y = y0 - r + row, x = x0 - r + col;
            mask_ok = y < P.H && x < P.W && __ldg(P.mask + frame * P.out_frame + (int64_t)y * P.W + x) != 0;
          }
          const int ri = (row + sy) * HWP + (col + sx);
          p = esz == 2 ? primary_from_u16<VAR>(reinterpret_cast<const unsigned short*>(raw)[ri], mask_ok)
                       : primary_from_f32<VAR>(reinterpret_cast<const float*>(raw)[ri], mask_ok);
        }
        prim[e] = p;
      }
      __syncthreads();
      // the other buffer was consumed in the previous iteration: prefetch the next tile into it
      if (tid == 0 && t + gridDim.x < total) {
        const TileGeom gn = tile_of(t + gridDim.x, ntx, nty);
        unsigned char* dst = b ? raw0 : raw1;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bars[b ^ 1], box_bytes);
        tma_load_tile(dst, &tmap, box_x(gn.x0 - r, al), max(gn.y0 - r, 0), (int)gn.frame, &bars[b ^ 1]);
      }
    } else {
      for (int row = tid >> 5; row < HH_; row += NTHREADS / 32) {
        const int y = y0 - r + row;
        const bool yin = y >= 0 && y < P.H;
        for (int col = tid & 31; col < HW_; col += 32) {
          const int x = x0 - r + col;
          double p = 0.0;
          if (yin && x >= 0 && x < P.W) {
            const int64_t off = frame * P.frame_stride + (int64_t)y * P.row_pitch + x;
            const bool mask_ok =
                !P.mask || __ldg(P.mask + frame * P.out_frame + (int64_t)y * P.W + x) != 0;
            p = esz == 2 ? primary_from_u16<VAR>(__ldg(reinterpret_cast<const unsigned short*>(P.depth) + off), mask_ok)
                         : primary_from_f32<VAR>(__ldg(reinterpret_cast<const float*>(P.depth) + off), mask_ok);
          }
          prim[row * HW_ + col] = p;
        }
      }
      __syncthreads();
    }

#if RF_ABLATE >= 4
    if (false)
#endif
    // ---- 2. vertical window sums.  Small compile-time radii: every (column,
    // output row) pair sums its 2r+1 rows directly (short independent chains,
    // all threads busy).  Otherwise each halo column is split into `parts` row
    // segments that warm up on their 2r leading rows and then slide down.
    if constexpr (RT > 0 && RT <= 3) {
      constexpr int HWc = TW + 2 * RT;
      for (int e = tid; e < TH * HWc; e += NTHREADS) {
        const int o = e / HWc, col = e - o * HWc;
        double a[NVD];
        int bb[NVI];
#pragma unroll
        for (int k = 0; k < NVD; ++k) a[k] = 0.0;
#pragma unroll
        for (int k = 0; k < NVI; ++k) bb[k] = 0;
        const double fo = (double)(o - RT);
#pragma unroll
        for (int k = 0; k <= 2 * RT; ++k) {
          const double p = prim[(o + k) * HWc + col];
          const double fdy = fo + (double)k;   // dy = (o + k) - r
          const int dy = o + k - RT;
          const int v = p > 0.0 ? 1 : 0;
          if (VAR == VAR_DF) {
            a[0] += p;
            a[1] = fma(p, p, a[1]);
            a[2] = fma(fdy, p, a[2]);
            bb[0] += v;
            bb[1] += v * dy;
            bb[2] += v * dy * dy;
          } else {
            const double p2 = p * p;
            a[0] += p;
            a[1] += p2;
            a[2] = fma(fdy, p, a[2]);
            a[3] = fma(fdy, p2, a[3]);
            a[4] = fma(fdy * fdy, p2, a[4]);
            bb[0] += v;
          }
        }
        const int cpos = (col & 3) * VQ + (col >> 2);
#pragma unroll
        for (int k = 0; k < NVD; ++k) vd[(k * TH + o) * VRS + cpos] = a[k];
#pragma unroll
        for (int k = 0; k < NVI; ++k) vi[(k * TH + o) * VRS + cpos] = bb[k];
      }
    } else {
      const int parts = max(1, min(NTHREADS / HW_, TH));
      const int col = tid % HW_;
      const int part = tid / HW_;
      if (part < parts) {
        const int o0 = (part * TH) / parts, o1 = ((part + 1) * TH) / parts;  // output rows [o0, o1)
        double a[NVD];
        int bb[NVI];
#pragma unroll
        for (int k = 0; k < NVD; ++k) a[k] = 0.0;
#pragma unroll
        for (int k = 0; k < NVI; ++k) bb[k] = 0;
        // dy of input row ii is ii - r (origin: the tile's first output row)
        auto add = [&](int ii, double fdy, int dy, double sg) {
          const double p = prim[ii * HW_ + col];
          const int v = p > 0.0 ? (sg > 0.0 ? 1 : -1) : 0;
          if (VAR == VAR_DF) {
            a[0] = fma(sg, p, a[0]);
            a[1] = fma(sg * p, p, a[1]);
            a[2] = fma(sg * fdy, p, a[2]);
            bb[0] += v;
            bb[1] += v * dy;
            bb[2] += v * dy * dy;
          } else {
            const double p2 = p * p;
            const double sfdy = sg * fdy;
            a[0] = fma(sg, p, a[0]);
            a[1] = fma(sg, p2, a[1]);
            a[2] = fma(sfdy, p, a[2]);
            a[3] = fma(sfdy, p2, a[3]);
            a[4] = fma(sfdy * fdy, p2, a[4]);
            bb[0] += v;
          }
        };
        // window of output row o covers input rows [o, o + 2r]
        double fdy = (double)(o0 - r);
        for (int ii = o0; ii < o0 + 2 * r; ++ii, fdy += 1.0) add(ii, fdy, ii - r, 1.0);
        double fdy_lo = (double)(o0 - r);
        const int cpos = (col & 3) * VQ + (col >> 2);
        for (int o = o0; o < o1; ++o, fdy += 1.0, fdy_lo += 1.0) {
          add(o + 2 * r, fdy, o + r, 1.0);
#pragma unroll
          for (int k = 0; k < NVD; ++k) vd[(k * TH + o) * VRS + cpos] = a[k];
#pragma unroll
          for (int k = 0; k < NVI; ++k) vi[(k * TH + o) * VRS + cpos] = bb[k];
          add(o, fdy_lo, o - r, -1.0);
        }
      }
    }
    __syncthreads();

    // ---- 3/4. horizontal running sums + per-window solve
    {
      const int orow = tid / (TW / KSEG);
      const int xs = (tid % (TW / KSEG)) * KSEG;  // tile-local x of the segment's first pixel
      const int gy = y0 + orow;
      const int gxs = x0 + xs;
      if (gy < P.H && gxs < P.W) {
      const double txo = __ldg(P.tan_x + gxs);
      const double tyo = __ldg(P.tan_y + y0);
      const double ifx = P.ifx, ify = P.ify;
      const double* vrow = vd + orow * VRS;
      const int* irow = vi + orow * VRS;
      const int vstride = TH * VRS;

      // running horizontal sums (origin: segment start xs, tile row y0)
      double h[VAR == VAR_DF ? 4 : 9];
      int hi[VAR == VAR_DF ? 6 : 1];
    #pragma unroll
      for (int k = 0; k < (VAR == VAR_DF ? 4 : 9); ++k) h[k] = 0.0;
    #pragma unroll
      for (int k = 0; k < (VAR == VAR_DF ? 6 : 1); ++k) hi[k] = 0;

      // k: column offset from the segment start xs (xs is a multiple of 4, so the
      // residue-major position of column xs + k is a compile-time offset from vbase)
      const int vbase = xs >> 2;
      auto accum = [&](int k, double sgn) {
        const int dx = k - r;
        const int c = vbase + (k & 3) * VQ + (k >> 2);
        const double fdx = (double)dx * sgn;
        if (VAR == VAR_DF) {
          const double w = vrow[c], ww = vrow[vstride + c], yw = vrow[2 * vstride + c];
          const int m = irow[c], my = irow[vstride + c], myy = irow[2 * vstride + c];
          h[0] = fma(sgn, w, h[0]);    // sum w
          h[1] = fma(sgn, ww, h[1]);   // sum w^2
          h[2] = fma(sgn, yw, h[2]);   // sum dy w
          h[3] = fma(fdx, w, h[3]);    // sum dx w
          const int sm = sgn > 0 ? m : -m, smy = sgn > 0 ? my : -my;
          hi[0] += sm;                 // n
          hi[1] += dx * sm;            // sum dx
          hi[2] += smy;                // sum dy
          hi[3] += dx * dx * sm;       // sum dx^2
          hi[4] += dx * smy;           // sum dx dy
          hi[5] += sgn > 0 ? myy : -myy;  // sum dy^2
        } else {
          const double z = vrow[c], z2 = vrow[vstride + c], yz = vrow[2 * vstride + c],
                       yz2 = vrow[3 * vstride + c], y2z2 = vrow[4 * vstride + c];
          const double fdx2 = fdx * (double)dx;
          h[0] = fma(sgn, z, h[0]);     // S3  = sum Z
          h[1] = fma(sgn, z2, h[1]);    // S33 = sum Z^2
          h[2] = fma(sgn, yz, h[2]);    // S2  = sum dy Z
          h[3] = fma(sgn, yz2, h[3]);   // S23 = sum dy Z^2
          h[4] = fma(sgn, y2z2, h[4]);  // S22 = sum dy^2 Z^2
          h[5] = fma(fdx, z, h[5]);     // S1  = sum dx Z
          h[6] = fma(fdx, z2, h[6]);    // S13 = sum dx Z^2
          h[7] = fma(fdx, yz2, h[7]);   // S12 = sum dx dy Z^2
          h[8] = fma(fdx2, z2, h[8]);   // S11 = sum dx^2 Z^2
          hi[0] += sgn > 0 ? irow[c] : -irow[c];
        }
      };

      if constexpr (RT > 0) {
#pragma unroll
        for (int k = 0; k <= 2 * RT; ++k) accum(k, 1.0);
      } else {
        for (int k = 0; k <= 2 * r; ++k) accum(k, 1.0);
      }

    #if RF_STAGE_OUTPUTS
      float o_n[KSEG][3], o_off[KSEG], o_res[KSEG], o_cur[KSEG];
      uint8_t o_st[KSEG];
    #endif

    #pragma unroll
      for (int j = 0; j < KSEG; ++j) {
#if RF_ABLATE < 3
        if (j > 0) {
          accum(j + 2 * r, 1.0);
          accum(j - 1, -1.0);
        }
#endif
        const int gx = gxs + j;
        const double pc = prim[(orow + r) * HW_ + xs + j + r];
        uint8_t st = pc > 0.0 ? RF_PIX_INPUT_VALID : 0;
        const int nwin = (int)hi[0];
        float nx = __int_as_float(0x7fc00000), ny = nx, nz = nx, off = nx, res = nx, cur = nx;
        uint8_t stx = st;  // explicit-fit status (MIN_SAMPLES 3 instead of 4)
        if (st && nwin >= (EXP ? 3 : 4) && gx < P.W) {
          const double nd = (double)nwin;
          const double invn = rcp_fast(nd);
          Sym3 C;
          double mu0, mu1, mu2;
          if (VAR == VAR_DF) {
            const long long n = hi[0], sx = hi[1], sy = hi[2], sxx = hi[3], sxy = hi[4], syy = hi[5];
            const double cq00 = (double)(n * sxx - sx * sx) * invn;
            const double cq01 = (double)(n * sxy - sx * sy) * invn;
            const double cq11 = (double)(n * syy - sy * sy) * invn;
            const double mw = h[0] * invn;
            const double fsx = (double)sx, fsy = (double)sy;
            const double cq02 = fma(-fsx, mw, h[3]);
            const double cq12 = fma(-fsy, mw, h[2]);
            const double cq22 = fma(-h[0], mw, h[1]);
            C.c00 = cq00 * (ifx * ifx);
            C.c01 = cq01 * (ifx * ify);
            C.c11 = cq11 * (ify * ify);
            C.c02 = cq02 * ifx;
            C.c12 = cq12 * ify;
            C.c22 = cq22;
            mu0 = fma(fsx * invn, ifx, txo);
            mu1 = fma(fsy * invn, ify, tyo);
            mu2 = mw;
          } else {
            // q = (dx Z, dy Z, Z): sums S1=h5, S2=h2, S3=h0, S11=h8, S12=h7, S22=h4,
            // S13=h6, S23=h3, S33=h1; C_q = S_ab - S_a S_b / n
            const double q0 = h[5] * invn, q1 = h[2] * invn, q2 = h[0] * invn;
            const double k00 = fma(-h[5], q0, h[8]);
            const double k01 = fma(-h[5], q1, h[7]);
            const double k02 = fma(-h[5], q2, h[6]);
            const double k11 = fma(-h[2], q1, h[4]);
            const double k12 = fma(-h[2], q2, h[3]);
            const double k22 = fma(-h[0], q2, h[1]);
            // m = L q, L = [[ifx, 0, txo], [0, ify, tyo], [0, 0, 1]]
            const double r00 = fma(ifx, k00, txo * k02), r01 = fma(ifx, k01, txo * k12),
                         r02 = fma(ifx, k02, txo * k22);
            const double r11 = fma(ify, k11, tyo * k12), r12 = fma(ify, k12, tyo * k22);
            C.c00 = fma(ifx, r00, txo * r02);
            C.c01 = fma(ify, r01, tyo * r02);
            C.c02 = r02;
            C.c11 = fma(ify, r11, tyo * r12);
            C.c12 = r12;
            C.c22 = k22;
            mu0 = fma(ifx, q0, txo * q2);
            mu1 = fma(ify, q1, tyo * q2);
            mu2 = q2;
          }
          float kap = 0.0f;
          if (P.do_imp && nwin >= 4) {
          WindowFit f;
#if RF_ABLATE >= 1
          f.lam = C.c00 + C.c11; f.u0 = mu0 + C.c01; f.u1 = mu1 + C.c02; f.u2 = mu2 + C.c12; f.s = C.c22;
          f.kappa = 0.1f; f.degenerate = false;
#else
          solve_window(C, mu0, mu1, mu2, nd, f);
#endif
#if RF_ABLATE >= 2
          nx = (float)f.u0; ny = (float)f.u1; nz = (float)f.u2; off = (float)f.s;
#else
          if (VAR == VAR_DF) finish_plane(f.u0, f.u1, f.s, f.u2, nx, ny, nz, off);
          else finish_plane(f.u0, f.u1, f.u2, f.s, nx, ny, nz, off);
#endif
          res = fsqrt(fmaxf((float)(f.lam * invn), 0.0f));
          cur = f.kappa;
          kap = f.kappa;
          st |= RF_PIX_FIT;
          if (f.degenerate) st |= RF_PIX_DEGENERATE;
          }
          if (EXP && P.do_exp) {
            if (!(P.do_imp && nwin >= 4)) kap = curvature_only(C);
            ExplicitFit e;
            explicit_solve(C, mu0, mu1, mu2, nd, e);
            float ex, ey, ez, eo;
            // explicit_to_implicit (fitting.py:729-739): standard (a, b, -1, c), rgbd (a, b, c, -1)
            if (VAR == VAR_DF) finish_plane(e.a, e.b, e.c, -1.0, ex, ey, ez, eo);
            else finish_plane(e.a, e.b, -1.0, e.c, ex, ey, ez, eo);
            stx |= RF_PIX_FIT | (e.degenerate ? RF_PIX_DEGENERATE : 0);
            const int64_t p = frame * P.out_frame + (int64_t)gy * P.W + gx;
            P.exp.normal[3 * p + 0] = ex;
            P.exp.normal[3 * p + 1] = ey;
            P.exp.normal[3 * p + 2] = ez;
            P.exp.offset[p] = eo;
            P.exp.residual[p] = fsqrt(fmaxf((float)(e.ss * invn), 0.0f));
            P.exp.curvature[p] = kap;
            P.exp.status[p] = stx;
          }
        }
        if (EXP && P.do_exp && !(stx & RF_PIX_FIT) && gx < P.W) {
          const int64_t p = frame * P.out_frame + (int64_t)gy * P.W + gx;
          const float qn = __int_as_float(0x7fc00000);
          P.exp.normal[3 * p + 0] = qn;
          P.exp.normal[3 * p + 1] = qn;
          P.exp.normal[3 * p + 2] = qn;
          P.exp.offset[p] = qn;
          P.exp.residual[p] = qn;
          P.exp.curvature[p] = qn;
          P.exp.status[p] = stx;
        }
    #if RF_STAGE_OUTPUTS
        o_n[j][0] = nx;
        o_n[j][1] = ny;
        o_n[j][2] = nz;
        o_off[j] = off;
        o_res[j] = res;
        o_cur[j] = cur;
        o_st[j] = st;
    #else
        if (gx < P.W) {
          const int64_t p = frame * P.out_frame + (int64_t)gy * P.W + gx;
          P.imp.normal[3 * p + 0] = nx;
          P.imp.normal[3 * p + 1] = ny;
          P.imp.normal[3 * p + 2] = nz;
          P.imp.offset[p] = off;
          P.imp.residual[p] = res;
          P.imp.curvature[p] = cur;
          P.imp.status[p] = st;
        }
    #endif
      }

    #if RF_STAGE_OUTPUTS
      // ---- stores
      if (P.do_imp) {
      const int64_t pix0 = frame * P.out_frame + (int64_t)gy * P.W + gxs;
      const bool vec = ((P.W & (KSEG - 1)) == 0) && (gxs + KSEG <= P.W);
      if (vec) {
        float4* pn = reinterpret_cast<float4*>(P.imp.normal + 3 * pix0);
        pn[0] = make_float4(o_n[0][0], o_n[0][1], o_n[0][2], o_n[1][0]);
        pn[1] = make_float4(o_n[1][1], o_n[1][2], o_n[2][0], o_n[2][1]);
        pn[2] = make_float4(o_n[2][2], o_n[3][0], o_n[3][1], o_n[3][2]);
        *reinterpret_cast<float4*>(P.imp.offset + pix0) = make_float4(o_off[0], o_off[1], o_off[2], o_off[3]);
        *reinterpret_cast<float4*>(P.imp.residual + pix0) = make_float4(o_res[0], o_res[1], o_res[2], o_res[3]);
        *reinterpret_cast<float4*>(P.imp.curvature + pix0) = make_float4(o_cur[0], o_cur[1], o_cur[2], o_cur[3]);
        *reinterpret_cast<uchar4*>(P.imp.status + pix0) = make_uchar4(o_st[0], o_st[1], o_st[2], o_st[3]);
      } else {
    #pragma unroll
        for (int j = 0; j < KSEG; ++j) {
          if (gxs + j >= P.W) break;
          const int64_t p = pix0 + j;
          P.imp.normal[3 * p + 0] = o_n[j][0];
          P.imp.normal[3 * p + 1] = o_n[j][1];
          P.imp.normal[3 * p + 2] = o_n[j][2];
          P.imp.offset[p] = o_off[j];
          P.imp.residual[p] = o_res[j];
          P.imp.curvature[p] = o_cur[j];
          P.imp.status[p] = o_st[j];
        }
      }
      }
    #endif
      }
    }
    __syncthreads();  // prim / vd are rewritten by the next tile
  }
}

// ------------------------------------------------------------------ tables
__global__ void tan_table_kernel(double* tx, double* ty, int W, int H, double fx, double fy,
                                 double cx, double cy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  // compute_tan_maps (camera.py:131-134) with delta = 0: ((col + 0.0) - cx) / fx
  if (i < W) tx[i] = __ddiv_rn(((double)i + 0.0) - cx, fx);
  if (i < H) ty[i] = __ddiv_rn(((double)i + 0.0) - cy, fy);
}

thread_local char g_err[512] = "";

rf_status fail(rf_status s, const char* fmt, const char* a = "", long long b = 0,
               long long c = 0) {
  snprintf(g_err, sizeof(g_err), fmt, a, b, c);
  return s;
}

size_t smem_bytes(int var, int r, bool tma, int esz) {
  const int hw = TW + 2 * r, hh = TH + 2 * r, hwp = (hw + 16 / esz - 1 + 7) & ~7;
  const int nvd = var == VAR_DF ? 3 : 5, nvi = var == VAR_DF ? 3 : 1;
  const size_t raw = tma ? (((size_t)hh * hwp * esz + 127) & ~(size_t)127) : 0;
  const size_t vrs = 4 * (size_t)vq_of(hw);
  return 2 * raw + sizeof(double) * ((size_t)hh * hw + (size_t)nvd * TH * vrs) +
         sizeof(int) * (size_t)nvi * TH * vrs + 8 /* align */ + 2 * sizeof(uint64_t) + 128 /* base align */;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// 3-D tensor map over the [batch, H, W] depth (row pitch row_pitch elements), box
// (hwp, hh, 1), zero fill out of range.  Returns false when TMA cannot address it.
bool make_depth_tmap(CUtensorMap* m, const void* depth, int dtype, int64_t batch, int H, int W,
                     int64_t row_pitch, int r) {
  const int esz = dtype == RF_DEPTH_U16_MM ? 2 : 4;
  const int hw = TW + 2 * r, hh = TH + 2 * r, hwp = (hw + 16 / esz - 1 + 7) & ~7;
  if (hwp > 256 || hh > 256) return false;
  if ((reinterpret_cast<uintptr_t>(depth) & 15) != 0) return false;
  if (((row_pitch * esz) & 15) != 0 || ((row_pitch * H * esz) & 15) != 0) return false;
  if (batch > 0x7fffffff) return false;
  PFN_cuTensorMapEncodeTiled_v12000 fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)(row_pitch * esz), (cuuint64_t)(row_pitch * H * esz)};
  const cuuint32_t box[3] = {(cuuint32_t)hwp, (cuuint32_t)hh, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult res = fn(m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                          const_cast<void*>(depth), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS;
}

template <int VAR, bool TMA, int RT>
cudaError_t launch_var(const KParams& P, const CUtensorMap& tmap, size_t sm, int64_t tiles, cudaStream_t s) {
  auto kern = P.do_exp ? fit_tile_kernel<VAR, TMA, RT, true> : fit_tile_kernel<VAR, TMA, RT, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTHREADS, sm);
  if (per_sm < 1) per_sm = 1;
  const int64_t grid = tiles < (int64_t)sms * per_sm ? tiles : (int64_t)sms * per_sm;
  kern<<<(unsigned)grid, NTHREADS, sm, s>>>(P, tmap);
  return cudaGetLastError();
}

// compile-time radii for the BASELINE windows 3, 5, 7, 9, 11, 15, 31; others run generic
template <int VAR>
cudaError_t launch_radius(const KParams& P, const CUtensorMap& tmap, size_t sm, int64_t tiles, cudaStream_t s) {
  switch (P.r) {
    case 1: return launch_var<VAR, true, 1>(P, tmap, sm, tiles, s);
    case 2: return launch_var<VAR, true, 2>(P, tmap, sm, tiles, s);
    case 3: return launch_var<VAR, true, 3>(P, tmap, sm, tiles, s);
    case 4: return launch_var<VAR, true, 4>(P, tmap, sm, tiles, s);
    case 5: return launch_var<VAR, true, 5>(P, tmap, sm, tiles, s);
    case 7: return launch_var<VAR, true, 7>(P, tmap, sm, tiles, s);
    case 15: return launch_var<VAR, true, 15>(P, tmap, sm, tiles, s);
    default: return launch_var<VAR, true, 0>(P, tmap, sm, tiles, s);
  }
}

}  // namespace

struct rf_tables {
  rf_intrinsics intr;
  int device;
  double* tan_x;  // [W] device
  double* tan_y;  // [H] device
};

extern "C" {

int32_t rf_abi_version(void) { return RF_ABI_VERSION; }

const char* rf_last_error(void) { return g_err; }

int32_t rf_launches_per_call(int32_t formulation_mask) {
  return ((formulation_mask & (RF_IMPLICIT_STANDARD | RF_EXPLICIT_STANDARD)) ? 1 : 0) +
         ((formulation_mask & (RF_IMPLICIT_RGBD | RF_EXPLICIT_RGBD)) ? 1 : 0);
}

rf_status rf_tables_create(const rf_intrinsics* in, const double* delta_x, const double* delta_y,
                           int device, rf_tables** out) {
  if (!in || !out) return fail(RF_ERR_ARGUMENT, "rf_tables_create: null argument%s");
  *out = nullptr;
  // CameraIntrinsics.__post_init__ (camera.py:54-63)
  if (!(in->fx > 0) || !(in->fy > 0))
    return fail(RF_ERR_ARGUMENT, "focal lengths must be positive%s");
  if (in->width <= 0 || in->height <= 0) return fail(RF_ERR_ARGUMENT, "image size must be positive%s");
  if (!(in->cx >= 0 && in->cx < in->width && in->cy >= 0 && in->cy < in->height))
    return fail(RF_ERR_ARGUMENT, "principal point outside the image%s");
  const int64_t n = (int64_t)in->width * in->height;
  for (int64_t i = 0; delta_x && i < n; ++i)
    if (delta_x[i] != 0.0)
      return fail(RF_ERR_UNSUPPORTED, "non-zero delta_x lattice%s: the sm_100a path needs separable tan maps");
  for (int64_t i = 0; delta_y && i < n; ++i)
    if (delta_y[i] != 0.0)
      return fail(RF_ERR_UNSUPPORTED, "non-zero delta_y lattice%s: the sm_100a path needs separable tan maps");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(RF_ERR_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
  rf_tables* t = new rf_tables();
  t->intr = *in;
  t->device = device;
  e = cudaMalloc(&t->tan_x, sizeof(double) * in->width);
  if (e == cudaSuccess) e = cudaMalloc(&t->tan_y, sizeof(double) * in->height);
  if (e == cudaSuccess) {
    const int m = in->width > in->height ? in->width : in->height;
    tan_table_kernel<<<(m + 255) / 256, 256>>>(t->tan_x, t->tan_y, in->width, in->height, in->fx,
                                               in->fy, in->cx, in->cy);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    cudaFree(t->tan_x);
    cudaFree(t->tan_y);
    delete t;
    return fail(RF_ERR_CUDA, "rf_tables_create: %s", cudaGetErrorString(e));
  }
  *out = t;
  return RF_OK;
}

rf_status rf_tables_destroy(rf_tables* t) {
  if (!t) return RF_OK;
  cudaFree(t->tan_x);
  cudaFree(t->tan_y);
  delete t;
  return RF_OK;
}

rf_status rf_fit_pixels(const rf_tables* t, const void* depth, int dtype, int64_t batch,
                        int32_t H, int32_t W, int64_t row_pitch, const uint8_t* mask,
                        int32_t window, int32_t fmask, const rf_pixel_out* outs, void* stream) {
  if (!t) return fail(RF_ERR_ARGUMENT, "rf_fit_pixels: null tables%s");
  if (!depth && batch != 0) return fail(RF_ERR_ARGUMENT, "rf_fit_pixels: null depth%s");
  if (dtype != RF_DEPTH_F32_M && dtype != RF_DEPTH_U16_MM)
    return fail(RF_ERR_SHAPE, "unknown depth dtype%s %lld", "", dtype);
  if (H != t->intr.height || W != t->intr.width)
    return fail(RF_ERR_SHAPE, "depth %s%lldx%lld does not match the camera tables", "", W, H);
  if (batch < 0) return fail(RF_ERR_ARGUMENT, "batch%s %lld is negative", "", batch);
  if (row_pitch < W) return fail(RF_ERR_ARGUMENT, "row_pitch%s %lld < width", "", row_pitch);
  if (window < 1 || (window & 1) == 0 || window / 2 > MAX_RADIUS)
    return fail(RF_ERR_ARGUMENT, "window%s must be odd and in [1, %lld], got %lld", "",
                2 * MAX_RADIUS + 1, window);
  if ((fmask & ~RF_ALL_FORMULATIONS) != 0 || fmask == 0)
    return fail(RF_ERR_ARGUMENT, "formulation_mask%s %lld invalid", "", fmask);
  if (batch == 0) return RF_OK;
  if (!outs) return fail(RF_ERR_ARGUMENT, "rf_fit_pixels: null output array%s");
  for (int f = 0; f < RF_NUM_FORMULATIONS; ++f) {
    if (!(fmask & (1 << f))) continue;
    const rf_pixel_out& o = outs[f];
    if (!o.normal || !o.offset || !o.residual || !o.curvature || !o.status)
      return fail(RF_ERR_ARGUMENT, "formulation %s%lld requested without output buffers", "", f);
  }
  const int r = window / 2;
  const int64_t tiles = (int64_t)((W + TW - 1) / TW) * ((H + TH - 1) / TH) * batch;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  const bool tma = getenv("RF_DISABLE_TMA") == nullptr &&
                   make_depth_tmap(&tmap, depth, dtype, batch, H, W, row_pitch, r);
  const int esz = dtype == RF_DEPTH_U16_MM ? 2 : 4;
  // one launch per space: standard (implicit/explicit-standard), rgbd (implicit/explicit-rgbd)
  for (int var = 0; var < 2; ++var) {
    const int fi = var == VAR_STD ? RF_FORM_IMPLICIT_STANDARD : RF_FORM_IMPLICIT_RGBD;
    const int fe = var == VAR_STD ? RF_FORM_EXPLICIT_STANDARD : RF_FORM_EXPLICIT_RGBD;
    const bool di = (fmask >> fi) & 1, de = (fmask >> fe) & 1;
    if (!di && !de) continue;
    KParams P;
    memset(&P, 0, sizeof(P));
    P.depth = depth;
    P.mask = mask;
    P.tan_x = t->tan_x;
    P.tan_y = t->tan_y;
    P.ifx = 1.0 / t->intr.fx;
    P.ify = 1.0 / t->intr.fy;
    P.row_pitch = row_pitch;
    P.frame_stride = row_pitch * H;
    P.out_frame = (int64_t)H * W;
    P.H = H;
    P.W = W;
    P.r = r;
    P.dtype = dtype;
    P.do_imp = di;
    P.do_exp = de;
    if (di) P.imp = OutPlanes{outs[fi].normal, outs[fi].offset, outs[fi].residual, outs[fi].curvature, outs[fi].status};
    if (de) P.exp = OutPlanes{outs[fe].normal, outs[fe].offset, outs[fe].residual, outs[fe].curvature, outs[fe].status};
    P.batch = batch;
    const size_t sm = smem_bytes(var, r, tma, esz);
    cudaError_t e;
    if (var == VAR_STD)
      e = tma ? launch_radius<VAR_STD>(P, tmap, sm, tiles, s) : launch_var<VAR_STD, false, 0>(P, tmap, sm, tiles, s);
    else
      e = tma ? launch_radius<VAR_DF>(P, tmap, sm, tiles, s) : launch_var<VAR_DF, false, 0>(P, tmap, sm, tiles, s);
    if (e != cudaSuccess) return fail(RF_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
  }
  return RF_OK;
}

}  // extern "C"
