// rf_direct.cuh -- one output pixel fitted from its window summed directly (no sliding
// sums): the distortion-lattice fallback kernel's body and the lattice tile kernel's
// sliding-sum guard fix-up (rf_lattice.cu).  Window moments are
// fp64 q-moments relative to the pixel's own tan values (rf_general.cuh), then the same
// solve / canonical output as the tile kernels (rf_solve.cuh).
#pragma once
#include <stdint.h>

#include "rf_tile.cuh"
#include "rf_solve.cuh"
#include "rf_jacobi.cuh"
#include "rf_general.cuh"

namespace rf_dev {

__device__ __forceinline__ void store_fit(const rf_tile::OutPlanes& o, int64_t p, float nx, float ny, float nz,
                                          float off, float res, float cur, uint8_t st) {
  o.normal[3 * p + 0] = nx;
  o.normal[3 * p + 1] = ny;
  o.normal[3 * p + 2] = nz;
  o.offset[p] = off;
  o.residual[p] = res;
  o.curvature[p] = cur;
  o.status[p] = st;
}

// tan of pixel (y, x): the lattice when the camera has one, else the separable tables
__device__ __forceinline__ double tan_at(const double* table, const double* lattice, int W, int x, int y,
                                         bool along_x) {
  return lattice ? __ldg(lattice + (int64_t)y * W + x) : __ldg(table + (along_x ? x : y));
}

// Fit output pixel (frame, y, x) of the kernel's space and store its implicit / explicit
// outputs (MIN_SAMPLES 4 / 3, reference fitting.py:45-73).
template <int VAR, bool EXP>
__device__ __forceinline__ void fit_pixel_direct(const rf_tile::KParams& P, const double* lat_x,
                                                 const double* lat_y, int64_t frame, int y, int x) {
  const int r = P.r;
  const bool std_space = VAR == rf_tile::VAR_STD;
  const int64_t p = frame * P.out_frame + (int64_t)y * P.W + x;
  auto sample = [&](int yy, int xx, double& z) -> bool {
    const int64_t off = frame * P.frame_stride + (int64_t)yy * P.row_pitch + xx;
    bool valid;
    if (P.dtype == RF_DEPTH_U16_MM) {
      const unsigned short mm = __ldg(reinterpret_cast<const unsigned short*>(P.depth) + off);
      valid = mm > 0;
      z = __ddiv_rn((double)mm, 1000.0);
    } else if (P.dtype == RF_DEPTH_F64_M) {
      z = __ldg(reinterpret_cast<const double*>(P.depth) + off);
      valid = z > 0.0 && z <= 1.7976931348623157e308;
    } else {
      const float zf = __ldg(reinterpret_cast<const float*>(P.depth) + off);
      valid = zf > 0.0f && zf <= 3.402823466e38f;
      z = (double)zf;
    }
    if (P.mask) valid = valid && __ldg(P.mask + frame * P.out_frame + (int64_t)yy * P.W + xx) != 0;
    return valid;
  };
  const float qn = __int_as_float(0x7fc00000);
  float nx = qn, ny = qn, nz = qn, off = qn, res = qn, cur = qn;
  float ex = qn, ey = qn, ez = qn, eo = qn, eres = qn, ecur = qn;
  double zc;
  const uint8_t valid_bit = sample(y, x, zc) ? RF_PIX_INPUT_VALID : 0;
  uint8_t st = valid_bit, stx = valid_bit;
  if (valid_bit) {
    const double txc = tan_at(P.tan_x, lat_x, P.W, x, y, true), tyc = tan_at(P.tan_y, lat_y, P.W, x, y, false);
    QMoments m;
    const int ya = max(y - r, 0), yb = min(y + r, P.H - 1), xa = max(x - r, 0), xb = min(x + r, P.W - 1);
    for (int yy = ya; yy <= yb; ++yy)
      for (int xx = xa; xx <= xb; ++xx) {
        double z;
        if (!sample(yy, xx, z)) continue;
        q_sample(std_space, z, tan_at(P.tan_x, lat_x, P.W, xx, yy, true) - txc,
                 tan_at(P.tan_y, lat_y, P.W, xx, yy, false) - tyc, m);
      }
    const int nwin = (int)m.n;
    if (nwin >= (EXP ? 3 : 4)) {
      Sym3 C;
      double mu0, mu1, mu2;
      q_to_scatter(std_space, m, txc, tyc, C, mu0, mu1, mu2);
      const double nd = m.n;
      float kap = 0.0f;
      if (P.do_imp && nwin >= 4) {
        WindowFit f;
        solve_window(C, mu0, mu1, mu2, nd, f);
        if (std_space) finish_plane(f.u0, f.u1, f.u2, f.s, nx, ny, nz, off);
        else finish_plane(f.u0, f.u1, f.s, f.u2, nx, ny, nz, off);
        res = fsqrt(fmaxf((float)(f.lam / nd), 0.0f));
        cur = kap = f.kappa;
        st |= RF_PIX_FIT | (f.degenerate ? RF_PIX_DEGENERATE : 0);
      }
      if (EXP && P.do_exp) {
        if (!(P.do_imp && nwin >= 4)) kap = curvature_only(C);
        ExplicitFit e;
        explicit_fit_robust(C, mu0, mu1, mu2, nd, e);
        if (std_space) finish_plane(e.a, e.b, -1.0, e.c, ex, ey, ez, eo);
        else finish_plane(e.a, e.b, e.c, -1.0, ex, ey, ez, eo);
        eres = fsqrt(fmaxf((float)(e.ss / nd), 0.0f));
        ecur = kap;
        stx |= RF_PIX_FIT | (e.degenerate ? RF_PIX_DEGENERATE : 0);
      }
    }
  }
  if (P.do_imp) store_fit(P.imp, p, nx, ny, nz, off, res, cur, st);
  if (EXP && P.do_exp) store_fit(P.exp, p, ex, ey, ez, eo, eres, ecur, stx);
}

}  // namespace rf_dev
