// rf_general.cuh -- window moments for cameras whose tan maps are not separable
// (CameraIntrinsics with non-zero delta_* lattices, camera.py:35-75, 124-135).  The
// monomials are taken relative to a reference pixel's tan values (tx_c, ty_c):
//   rgbd      q = (tx - tx_c, ty - ty_c, 1/Z)       m = (tx, ty, 1/Z) = q + (tx_c, ty_c, 0)
//   standard  q = (Z (tx - tx_c), Z (ty - ty_c), Z)  m = (X, Y, Z) = L q,
//             L = [[1, 0, tx_c], [0, 1, ty_c], [0, 0, 1]]
// so the fp64 sums stay window-sized, and the centred scatter C and mean mu follow as in
// the separable kernels (the covariance is shift-invariant; the standard form maps K -> L K L^T).
#pragma once
#include "rf_solve.cuh"

namespace rf_dev {

struct QMoments {
  double n = 0, s0 = 0, s1 = 0, s2 = 0, s00 = 0, s01 = 0, s02 = 0, s11 = 0, s12 = 0, s22 = 0;
  __device__ __forceinline__ void add(double q0, double q1, double q2) {
    n += 1.0;
    s0 += q0;
    s1 += q1;
    s2 += q2;
    s00 = fma(q0, q0, s00);
    s01 = fma(q0, q1, s01);
    s02 = fma(q0, q2, s02);
    s11 = fma(q1, q1, s11);
    s12 = fma(q1, q2, s12);
    s22 = fma(q2, q2, s22);
  }
};

// sample of one valid pixel: z = depth (metres), dtx/dty = tan offsets from the reference
__device__ __forceinline__ void q_sample(bool std_space, double z, double dtx, double dty, QMoments& m) {
  if (std_space) m.add(z * dtx, z * dty, z);
  else m.add(dtx, dty, 1.0 / z);
}

__device__ __forceinline__ void q_to_scatter(bool std_space, const QMoments& m, double txc, double tyc, Sym3& C,
                                             double& mu0, double& mu1, double& mu2) {
  const double invn = 1.0 / m.n;
  const double q0 = m.s0 * invn, q1 = m.s1 * invn, q2 = m.s2 * invn;
  const double k00 = fma(-m.s0, q0, m.s00), k01 = fma(-m.s0, q1, m.s01), k02 = fma(-m.s0, q2, m.s02);
  const double k11 = fma(-m.s1, q1, m.s11), k12 = fma(-m.s1, q2, m.s12), k22 = fma(-m.s2, q2, m.s22);
  if (!std_space) {
    C.c00 = k00; C.c01 = k01; C.c02 = k02; C.c11 = k11; C.c12 = k12; C.c22 = k22;
    mu0 = txc + q0;
    mu1 = tyc + q1;
    mu2 = q2;
    return;
  }
  // C = L K L^T
  const double r00 = fma(txc, k02, k00), r01 = fma(txc, k12, k01), r02 = fma(txc, k22, k02);
  const double r11 = fma(tyc, k12, k11), r12 = fma(tyc, k22, k12);
  C.c00 = fma(txc, r02, r00);
  C.c01 = fma(tyc, r02, r01);
  C.c02 = r02;
  C.c11 = fma(tyc, r12, r11);
  C.c12 = r12;
  C.c22 = k22;
  mu0 = fma(txc, q2, q0);
  mu1 = fma(tyc, q2, q1);
  mu2 = q2;
}

}  // namespace rf_dev
