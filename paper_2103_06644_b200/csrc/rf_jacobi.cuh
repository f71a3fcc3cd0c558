// rf_jacobi.cuh -- the reference's cyclic Jacobi (jacobi_eigh) and the minimum-norm solve
// of rank-deficient explicit systems (_pinv_solve) on the device: the batched scatter fits
// (rf_integral.cu) and the explicit fits of windows whose Cholesky pivot test fails (per-pixel
// slow pass, rect and lattice kernels).
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include "rf_solve.cuh"

namespace rf_dev {

// ---- cyclic Jacobi (jacobi_eigh, fitting.py:193-253): same threshold (1e-13 ||A||_F),
// same sweep order and rotation formulas, no fused multiply-adds (the reference runs in
// Python floats); eigenvectors in the columns of v.
template <int N>
static __device__ __noinline__ bool jacobi(double (&a)[N][N], double (&v)[N][N], double fro) {
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) v[i][j] = i == j ? 1.0 : 0.0;
  if (fro == 0.0) {
    for (int i = 0; i < N; ++i) a[i][i] = 0.0;
    return true;
  }
  const double threshold = 1e-13 * fro;
  auto off_norm = [&]() {
    double s = 0.0;
    for (int p = 0; p < N - 1; ++p)
      for (int q = p + 1; q < N; ++q) s += a[p][q] * a[p][q];
    return sqrt(2.0 * s);
  };
  for (int sweep = 0; sweep < 50; ++sweep) {
    if (off_norm() <= threshold) return true;
    for (int p = 0; p < N - 1; ++p) {
      for (int q = p + 1; q < N; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double theta = __ddiv_rn(__dmul_rn(0.5, __dsub_rn(a[q][q], a[p][p])), apq);
        double t;
        if (fabs(theta) > 1e8) t = __ddiv_rn(0.5, theta);
        else if (theta >= 0.0) t = __ddiv_rn(1.0, __dadd_rn(theta, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(theta, theta)))));
        else t = __ddiv_rn(-1.0, __dadd_rn(-theta, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(theta, theta)))));
        const double c = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(t, t)))), s = __dmul_rn(t, c);
        const double app = a[p][p], aqq = a[q][q];
        a[p][p] = __dsub_rn(app, __dmul_rn(t, apq));
        a[q][q] = __dadd_rn(aqq, __dmul_rn(t, apq));
        a[p][q] = a[q][p] = 0.0;
        for (int k = 0; k < N; ++k) {
          if (k == p || k == q) continue;
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = a[p][k] = __dsub_rn(__dmul_rn(c, akp), __dmul_rn(s, akq));
          a[k][q] = a[q][k] = __dadd_rn(__dmul_rn(s, akp), __dmul_rn(c, akq));
        }
        for (int k = 0; k < N; ++k) {
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = __dsub_rn(__dmul_rn(c, vkp), __dmul_rn(s, vkq));
          v[k][q] = __dadd_rn(__dmul_rn(s, vkp), __dmul_rn(c, vkq));
        }
      }
    }
  }
  return off_norm() <= threshold;
}

template <int N>
__device__ __forceinline__ double frobenius(const double (&a)[N][N]) {
  double s = 0.0;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) s += a[i][j] * a[i][j];
  return sqrt(s);
}


// _pinv_solve (fitting.py:313-322) of the uncentred explicit system M x = rhs: eigenpairs by
// jacobi_eigh, components with eigenvalue above 1e-12 trace(M) only.  false when Jacobi does
// not converge (DegenerateFitError in the reference).
static __device__ __noinline__ bool explicit_min_norm(const double (&A)[3][3], const double (&b)[3], double (&x)[3]) {
  double E[3][3], V[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) E[r][c] = A[r][c];
  const double trace = __dadd_rn(__dadd_rn(A[0][0], A[1][1]), A[2][2]);
  x[0] = x[1] = x[2] = 0.0;
  if (!isfinite(trace) || !jacobi(E, V, frobenius(E))) return false;
  const double tol = __dmul_rn(1e-12, fmax(trace, 0.0));
  for (int e = 0; e < 3; ++e) {
    const double lam = E[e][e];
    if (lam > tol) {
      const double dot = __dadd_rn(__dadd_rn(__dmul_rn(V[0][e], b[0]), __dmul_rn(V[1][e], b[1])), __dmul_rn(V[2][e], b[2]));
      const double w = __ddiv_rn(dot, lam);
      x[0] = __dadd_rn(x[0], __dmul_rn(V[0][e], w));
      x[1] = __dadd_rn(x[1], __dmul_rn(V[1][e], w));
      x[2] = __dadd_rn(x[2], __dmul_rn(V[2][e], w));
    }
  }
  return true;
}

// Explicit fit of a window from its centred moments (explicit_solve), falling back, when the
// reference's Cholesky pivot test fails (fitting.py:584-589), to the minimum-norm solution of
// the uncentred system [[S00, S01, S0], [S01, S11, S1], [S0, S1, n]] x = [S02, S12, S2] and
// its residual sum(b^2) - x.rhs (fitting.py:590-597).
__device__ __forceinline__ void explicit_fit_robust(const Sym3& C, double m0, double m1, double m2, double n,
                                                    ExplicitFit& e) {
  explicit_solve(C, m0, m1, m2, n, e);
  if (!e.degenerate) return;
  const double A[3][3] = {{fma(n * m0, m0, C.c00), fma(n * m0, m1, C.c01), n * m0},
                          {fma(n * m0, m1, C.c01), fma(n * m1, m1, C.c11), n * m1},
                          {n * m0, n * m1, n}};
  const double b[3] = {fma(n * m0, m2, C.c02), fma(n * m1, m2, C.c12), n * m2};
  double x[3];
  explicit_min_norm(A, b, x);
  e.a = x[0];
  e.b = x[1];
  e.c = x[2];
  e.ss = fma(n * m2, m2, C.c22) - (x[0] * b[0] + x[1] * b[1] + x[2] * b[2]);
}

}  // namespace rf_dev
