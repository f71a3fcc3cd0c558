// rf_tile_kernel.cuh -- the per-pixel tile kernel (fit_tile_kernel<SP, USE_TMA, RT, EXP, MINB>)
// and its launch helper, included by the kernel translation units rf_fit_k1/k2/k3.cu (one per
// space set, compiled in parallel) -- see rf_fit.cu for the C ABI and DESIGN.md section 4.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <stdarg.h>

#include <mutex>
#include <type_traits>

#include "../../include/rangefit_b200.h"

#include "rf_tile.cuh"
// largest compile-time radius whose column pass sums each window directly (dy centred on the
// output row, warp-local, no running sums): measured r <= 5 (C3 w9 +2%; r = 7 loses 1-3%)
#ifndef RF_CENTRED_MAX
#define RF_CENTRED_MAX 5
#endif
#include "rf_solve.cuh"
#include "rf_invn.cuh"
#include "rf_jacobi.cuh"
#include "rf_general.cuh"
#include "rf_direct.cuh"

namespace rf_fitk {
using namespace rf_dev;
using namespace rf_tile;

#ifdef RF_COUNT_SLOW
__device__ unsigned long long g_slow_count[256];
#endif

// compile-time radii whose standard-space halo (Z) is staged as float, not fp64 (see ZF): the
// only way two CTAs fit per SM at r = 15; Z of a float32 input is exact in float
__host__ __device__ constexpr bool noprim_radius(int rt) { return rt == 15; }

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

// ------------------------------------------------------------------ tile kernel
// One launch fits every requested formulation of both spaces (SP bit 0: standard, bit 1:
// disparity form).  A persistent CTA owns a TW x TH tile of output pixels of one frame at a
// time; the TMA halo of the next tile streams in while the current one is processed:
//   1. convert : depth -> validity (synth.py:84, 111-114) -> fp64 primaries, 1/Z for the
//                disparity form (integral.py:211-214) and Z for the standard form, 0 where
//                invalid, both from one read of the halo;
//   then per space: 2. column pass (vertical window sums) -> 3. row pass (horizontal sums,
//   fast solve, outputs) -> 4. slow pass (the windows the fast solve declined).
// Column sums of the two spaces share one buffer (the space passes run one after the
// other); the valid-count geometry is summed once per tile.

// slow-pass queue of one tile (row pass -> slow_pixel): tile-local pixel index, with
// Q_DIRECT when the window must be re-summed directly (sliding-sum guard)
constexpr int NWARPS = NTHREADS / 32;
constexpr int RPW = TH / NWARPS;  // output rows per warp (the row pass: TW / KSEG threads per row)
static_assert(RPW * NWARPS == TH && (TW / KSEG) * RPW == 32, "a warp owns whole output rows");
constexpr int QCAP = 64;          // per warp
constexpr int Q_DIRECT = 0x8000;  // re-sum the window directly (sliding-sum guard)
constexpr int Q_EXPL = 0x4000;    // only the explicit fit: its Cholesky pivot test failed
constexpr int Q_PIX = 0x3fff;     // tile-local pixel index

// depth element -> Z (metres) and validity (DepthImage, synth.py:84, 111-114)
__device__ __forceinline__ double depth_z(float zf, bool& valid) {
  valid = (zf > 0.0f) && (zf <= 3.402823466e38f);  // isfinite & > 0
  return (double)zf;
}
__device__ __forceinline__ double depth_z(double z, bool& valid) {  // float64 metres (RF64 ingest)
  valid = (z > 0.0) && (z <= 1.7976931348623157e308);
  return z;
}
__device__ __forceinline__ double depth_z(unsigned short mm, bool& valid) {
  // mm / 1000.0 correctly rounded, as the reference divides: q = mm * RN(1/1000) and one
  // exact-remainder correction (fma(-q, 1000, mm) is exact); checked for all 65535 codes
  valid = mm > 0;
  const double m = (double)mm;
  const double q0 = m * 1e-3;
  return fma(fma(-q0, 1000.0, m), 1e-3, q0);
}
// the space's primary: 1/Z (disparity form) or Z (standard), 0 when invalid
template <int VAR, typename T>
__device__ __forceinline__ double primary_of(T v, bool mask_ok) {
  bool valid;
  const double z = depth_z(v, valid);
  return (valid && mask_ok) ? (VAR == VAR_DF ? rcp_fast(z) : z) : 0.0;
}

// Halo tile (raw TMA box, element (row, col) at raw[(row + sy) * HWP + col + sx]) -> the
// primaries of the requested spaces, [row * HW_ + col].  The plain loop covers interior
// tiles without a mask; image edges (negative shift: rows/columns left of or above the
// image) and masks take the checked loop.
template <int SP, bool ZF, typename T>
__device__ __forceinline__ void convert_halo(double* pw, double* pz, float* pzf, const T* raw, int HW_, int HH_,
                                             int HWP, int sx, int sy, const KParams& P, int64_t frame, int x0,
                                             int y0, int r, int tid) {
  const int n = HH_ * HW_;
  auto put = [&](int e, T v, bool ok) {
    bool valid;
    const double z = depth_z(v, valid);
    valid = valid && ok;
    if (SP & 2) pw[e] = valid ? rcp_fast(z) : 0.0;
    if ((SP & 1) && ZF) pzf[e] = valid ? (float)z : 0.0f;
    if ((SP & 1) && !ZF) pz[e] = valid ? z : 0.0;
  };
  if (!P.mask && (sx | sy) >= 0 && ((HW_ | HWP | sx) & 1) == 0) {
    // interior tile, even row geometry: element pairs (one 2-element load, one 16-byte store
    // per primary), half the index arithmetic
    for (int e = 2 * tid; e < n; e += 2 * NTHREADS) {
      const int row = e / HW_, col = e - row * HW_;
      const T* src = raw + (row + sy) * HWP + col + sx;
      bool v0, v1;
      const double z0 = depth_z(src[0], v0), z1 = depth_z(src[1], v1);
      if (SP & 2) *reinterpret_cast<double2*>(pw + e) = make_double2(v0 ? rcp_fast(z0) : 0.0, v1 ? rcp_fast(z1) : 0.0);
      if ((SP & 1) && ZF) *reinterpret_cast<float2*>(pzf + e) = make_float2(v0 ? (float)z0 : 0.0f, v1 ? (float)z1 : 0.0f);
      if ((SP & 1) && !ZF) *reinterpret_cast<double2*>(pz + e) = make_double2(v0 ? z0 : 0.0, v1 ? z1 : 0.0);
    }
  } else if (!P.mask && (sx | sy) >= 0) {
#pragma unroll 2
    for (int e = tid; e < n; e += NTHREADS) {
      const int row = e / HW_, col = e - row * HW_;
      put(e, raw[(row + sy) * HWP + col + sx], true);
    }
  } else {
    for (int e = tid; e < n; e += NTHREADS) {
      const int row = e / HW_, col = e - row * HW_;
      bool ok = row + sy >= 0 && col + sx >= 0;
      if (ok && P.mask) {
        const int y = y0 - r + row, x = x0 - r + col;
        ok = y < P.H && x < P.W && __ldg(P.mask + frame * P.out_frame + (int64_t)y * P.W + x) != 0;
      }
      put(e, ok ? raw[(row + sy) * HWP + col + sx] : T(0), ok);
    }
  }
}

// running horizontal sums of one space: fp64 moments and exact integer geometry
template <int VAR> struct HSums {
  static constexpr int NH = VAR == VAR_DF ? 4 : 9;
  static constexpr int NHI = VAR == VAR_DF ? 6 : 1;
};

// valid-count geometry of one column sum (count, sum dy, sum dy^2).  Compile-time radii
// (r <= 15: count < 32, |sum dy| < 1024, sum dy^2 < 65536) pack it into one int; the generic
// radius (r <= 32) into an int2.
__device__ __forceinline__ void pack_counts(int& v, int m, int my, int myy) { v = m | ((my + 1024) << 5) | (myy << 16); }
__device__ __forceinline__ void pack_counts(int2& v, int m, int my, int myy) { v = make_int2((m & 0xffff) | (my << 16), myy); }
__device__ __forceinline__ int count_of(int v) { return v & 31; }
__device__ __forceinline__ int count_of(int2 v) { return v.x & 0xffff; }
__device__ __forceinline__ void unpack_counts(int v, int& m, int& my, int& myy) {
  m = v & 31;
  my = ((v >> 5) & 2047) - 1024;
  myy = (int)((unsigned)v >> 16);
}
__device__ __forceinline__ void unpack_counts(int2 v, int& m, int& my, int& myy) {
  m = v.x & 0xffff;
  my = v.x >> 16;
  myy = v.y;
}
template <int RT> using CountT = typename std::conditional<(RT > 0), int, int2>::type;

// add (sgn = +1) or remove (sgn = -1) one column's vertical sums at offset dx from the
// horizontal origin: disparity form w, w^2, dy w (fp64) and the valid count, dy, dy^2
// (int); standard form Z, Z^2, dy Z, dy Z^2, dy^2 Z^2 (fp64) and the valid count
template <int VAR, typename VI>
__device__ __forceinline__ void accum_column(double* h, int* hi, const double* vrow, const VI* irow, int vstride,
                                             int c, int dx, double sgn) {
  const double fdx = (double)dx * sgn;
  const VI g = irow[c];
  if (VAR == VAR_DF) {
    const double w = vrow[c], ww = vrow[vstride + c], yw = vrow[2 * vstride + c];
    int m, my, myy;
    unpack_counts(g, m, my, myy);
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
    const int m = count_of(g);
    hi[0] += sgn > 0 ? m : -m;
  }
}

// one valid sample p (disparity form 1/Z, standard Z) at (dx, dy) from the origin, added
// directly (the slow pass's re-summed windows)
template <int VAR>
__device__ __forceinline__ void accum_sample(double* h, int* hi, double p, int dx, int dy) {
  const double fdx = (double)dx, fdy = (double)dy;
  if (VAR == VAR_DF) {
    h[0] += p;
    h[1] = fma(p, p, h[1]);
    h[2] = fma(fdy, p, h[2]);
    h[3] = fma(fdx, p, h[3]);
    hi[0] += 1;
    hi[1] += dx;
    hi[2] += dy;
    hi[3] += dx * dx;
    hi[4] += dx * dy;
    hi[5] += dy * dy;
  } else {
    const double p2 = p * p;
    h[0] += p;
    h[1] += p2;
    h[2] = fma(fdy, p, h[2]);
    h[3] = fma(fdy, p2, h[3]);
    h[4] = fma(fdy * fdy, p2, h[4]);
    h[5] = fma(fdx, p, h[5]);
    h[6] = fma(fdx, p2, h[6]);
    h[7] = fma(fdx * fdy, p2, h[7]);
    h[8] = fma(fdx * fdx, p2, h[8]);
    hi[0] += 1;
  }
}

// window moments -> centred scatter C (3x3) and mean mu of the space's monomials
// (scatter_from_integrals / accumulate_scatter_naive, fitting.py:339-533, centred); txo, tyo:
// tan of the dx / dy origin
template <int VAR, bool WIDE>
__device__ __forceinline__ void assemble(const double* h, const int* hi, double txo, double tyo, const KParams& P,
                                         double invn, Sym3& C, double& mu0, double& mu1, double& mu2) {
  const double ifx = P.ifx, ify = P.ify;
  if (VAR == VAR_DF) {
    // exact integer geometry: compile-time radii (r <= 15) keep n sum dx^2 - (sum dx)^2 and
    // the other two in 32 bits; the generic radius (r <= 32) needs 64
    using I = typename std::conditional<WIDE, long long, int>::type;
    const I n = hi[0], sx = hi[1], sy = hi[2], sxx = hi[3], sxy = hi[4], syy = hi[5];
    const double mw = h[0] * invn;
    const double fsx = (double)sx, fsy = (double)sy;
    C.c00 = (double)(n * sxx - sx * sx) * (invn * P.ifx2);
    C.c01 = (double)(n * sxy - sx * sy) * (invn * P.ifxy);
    C.c11 = (double)(n * syy - sy * sy) * (invn * P.ify2);
    C.c02 = fma(-fsx, mw, h[3]) * ifx;
    C.c12 = fma(-fsy, mw, h[2]) * ify;
    C.c22 = fma(-h[0], mw, h[1]);
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
}

// Per-tile context shared by the space passes: geometry, shared-memory views.
struct TileCtx {
  const KParams* P;
  int r, HW_, HH_, HWP, VQ, VRS, sx, sy, esz, it, tid;
  int64_t frame;
  int x0, y0;
  const unsigned char* raw;
  double* pw;   // [HH_][HW_] 1/Z (disparity form)
  double* pz;   // [HH_][HW_] Z (standard)
  float* pzf;   // [HH_][HW_] Z (standard, ZF kernels: float32 input only)
  double* vd;   // [NVD][TH][VRS] column sums of the current space
  void* vi;     // [TH][VRS] valid-count geometry (both spaces), CountT<RT>
  float* xstage;
  // tan of this thread's row-pass origin (segment start column, dy origin row), loaded at the
  // start of the tile so the global-load latency hides behind the TMA wait and the conversion
  double txo, tyo;
};

// primary of halo element (row, col) of the tile for space VAR (ZF: the standard space's Z
// tile is float)
template <int VAR, bool ZF>
__device__ __forceinline__ double primary_at(const TileCtx& T, int row, int col) {
  if (VAR == VAR_STD && ZF) return (double)T.pzf[row * T.HW_ + col];
  return (VAR == VAR_DF ? T.pw : T.pz)[row * T.HW_ + col];
}

// ---- 2. vertical window sums of space VAR (and, for the tile's first space, the
// valid-count geometry).  Small compile-time radii: every (column, output row) pair sums
// its 2r+1 rows directly (short independent chains, all threads busy), dy centred on the
// output row.  Otherwise each halo column is split into `parts` row segments that warm up on
// their 2r leading rows and then slide down, dy relative to the tile's first output row.
// COUNTS: 0 none (the other space already summed them), 1 the valid count only (a
// standard-form launch), 2 the count and its dy, dy^2 moments (the disparity form needs them)
template <int VAR, int RT, bool NOPRIM, int COUNTS>
__device__ __forceinline__ void column_pass(const TileCtx& T, unsigned* s_dmax) {
  constexpr int NVD = VAR == VAR_DF ? 3 : 5;
  constexpr bool CENTRED = RT > 0 && RT <= RF_CENTRED_MAX;
  const int r = T.r, VRS = T.VRS, VQ = T.VQ, tid = T.tid;
  double* vd = T.vd;
  if constexpr (CENTRED) {
    // dy = k - RT (compile-time): the dy-weighted sums fold into symmetric differences
    constexpr int HWc = TW + 2 * RT;
    constexpr int K = 2 * RT + 1;
    const double* prim = VAR == VAR_DF ? T.pw : T.pz;
    // warp-local: each warp sums the RPW rows its own row pass reads (no CTA barrier
    // between); a lane takes whole columns, so its RPW output rows share K + RPW - 1 loads
    // and, for the plain sums, the K - 1 rows common to neighbouring windows
    static_assert(RPW == 2, "column-major centred pass written for two rows per warp");
    const int o0 = (tid >> 5) * RPW;
    for (int col = tid & 31; col < HWc; col += 32) {
      double p[K + 1];
#pragma unroll
      for (int k = 0; k <= K; ++k) p[k] = prim[(o0 + k) * HWc + col];
      const int cpos = (col & 3) * VQ + (col >> 2);
      // rows o0 (window p[0..K-1]) and o0 + 1 (p[1..K]); dy centred: symmetric differences
      double t0 = p[1];
#pragma unroll
      for (int k = 2; k < K; ++k) t0 += p[k];
      double d0 = p[RT + 1] - p[RT - 1], d1 = p[RT + 2] - p[RT];
#pragma unroll
      for (int d = 2; d <= RT; ++d) {
        d0 = fma((double)d, p[RT + d] - p[RT - d], d0);
        d1 = fma((double)d, p[RT + 1 + d] - p[RT + 1 - d], d1);
      }
      double a0[NVD], a1[NVD];
      a0[0] = p[0] + t0;
      a1[0] = t0 + p[K];
      a0[2] = d0;
      a1[2] = d1;
      if (VAR == VAR_DF) {
        double t1 = p[1] * p[1];
#pragma unroll
        for (int k = 2; k < K; ++k) t1 = fma(p[k], p[k], t1);
        a0[1] = fma(p[0], p[0], t1);
        a1[1] = fma(p[K], p[K], t1);
      } else {
        double q[K + 1];
#pragma unroll
        for (int k = 0; k <= K; ++k) q[k] = p[k] * p[k];
        double t1 = q[1];
#pragma unroll
        for (int k = 2; k < K; ++k) t1 += q[k];
        a0[1] = q[0] + t1;
        a1[1] = t1 + q[K];
        double e0 = q[RT + 1] - q[RT - 1], e1 = q[RT + 2] - q[RT];
        double f0 = q[RT + 1] + q[RT - 1], f1 = q[RT + 2] + q[RT];
#pragma unroll
        for (int d = 2; d <= RT; ++d) {
          e0 = fma((double)d, q[RT + d] - q[RT - d], e0);
          e1 = fma((double)d, q[RT + 1 + d] - q[RT + 1 - d], e1);
          f0 = fma((double)(d * d), q[RT + d] + q[RT - d], f0);
          f1 = fma((double)(d * d), q[RT + 1 + d] + q[RT + 1 - d], f1);
        }
        a0[3] = e0;
        a1[3] = e1;
        a0[4] = f0;
        a1[4] = f1;
      }
#pragma unroll
      for (int k = 0; k < NVD; ++k) {
        vd[(k * TH + o0) * VRS + cpos] = a0[k];
        vd[(k * TH + o0 + 1) * VRS + cpos] = a1[k];
      }
      if (COUNTS) {
        int v[K + 1];
#pragma unroll
        for (int k = 0; k <= K; ++k) v[k] = p[k] > 0.0 ? 1 : 0;
        int mt = 0;
#pragma unroll
        for (int k = 1; k < K; ++k) mt += v[k];
        int my0 = 0, myy0 = 0, my1 = 0, myy1 = 0;
        if (COUNTS == 2) {
#pragma unroll
          for (int d = 1; d <= RT; ++d) {
            my0 += d * (v[RT + d] - v[RT - d]);
            myy0 += d * d * (v[RT + d] + v[RT - d]);
            my1 += d * (v[RT + 1 + d] - v[RT + 1 - d]);
            myy1 += d * d * (v[RT + 1 + d] + v[RT + 1 - d]);
          }
        }
        pack_counts(static_cast<CountT<RT>*>(T.vi)[o0 * VRS + cpos], mt + v[0], my0, myy0);
        pack_counts(static_cast<CountT<RT>*>(T.vi)[(o0 + 1) * VRS + cpos], mt + v[K], my1, myy1);
      }
    }
  } else {
    const int HW_ = T.HW_;
    const int parts = max(1, min(NTHREADS / HW_, TH));
    const int col = tid % HW_;
    const int part = tid / HW_;
    int dm = 0;  // high word of the largest primary that left this thread's sums
    if (part < parts) {
      const int o0 = (part * TH) / parts, o1 = ((part + 1) * TH) / parts;  // output rows [o0, o1)
      double a[NVD];
      int m = 0, my = 0, myy = 0;
#pragma unroll
      for (int k = 0; k < NVD; ++k) a[k] = 0.0;
      // dy of input row ii is ii - r (origin: the tile's first output row)
      auto add = [&](int ii, double fdy, int dy, double sg) {
        const double p = primary_at<VAR, NOPRIM>(T, ii, col);
        if (sg < 0.0) dm = max(dm, __double2hiint(p));  // p >= 0: high words order like values
        if (VAR == VAR_DF) {
          a[0] = fma(sg, p, a[0]);
          a[1] = fma(sg * p, p, a[1]);
          a[2] = fma(sg * fdy, p, a[2]);
        } else {
          const double p2 = p * p;
          const double sfdy = sg * fdy;
          a[0] = fma(sg, p, a[0]);
          a[1] = fma(sg, p2, a[1]);
          a[2] = fma(sfdy, p, a[2]);
          a[3] = fma(sfdy, p2, a[3]);
          a[4] = fma(sfdy * fdy, p2, a[4]);
        }
        if (COUNTS) {
          const int v = p > 0.0 ? (sg > 0.0 ? 1 : -1) : 0;
          m += v;
          if (COUNTS == 2) {
            my += v * dy;
            myy += v * dy * dy;
          }
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
        if (COUNTS) pack_counts(static_cast<CountT<RT>*>(T.vi)[o * VRS + cpos], m, my, myy);
        add(o, fdy_lo, o - r, -1.0);
      }
    }
    const unsigned b = __reduce_max_sync(0xffffffffu, (unsigned)dm);  // dm >= 0
    if ((tid & 31) == 0) atomicMax(&s_dmax[T.it & 1], b);
  }
}

// The slow pass for one queued pixel of the tile: its window re-summed from the column sums
// (directly, no running update) or -- Q_DIRECT with running column sums -- from the
// primaries themselves, the robust solve (solve_window), and scalar stores that overwrite
// what the row pass wrote for it.  Q_DIRECT entries (the sliding-sum guard) redo the
// explicit fits as well; other entries only refresh the explicit curvature (it is shared).
template <int VAR, int RT, bool EXP, bool NOPRIM>
__device__ __forceinline__ void slow_pixel(const TileCtx& T, const KParams& P, int e) {
  constexpr bool CENTRED = RT > 0 && RT <= RF_CENTRED_MAX;
  const int r = T.r;
  const int pix = e & Q_PIX;
  const bool direct = (e & Q_DIRECT) != 0;
  const bool expl_only = (e & Q_EXPL) != 0 && !direct;
  const int orow = pix / TW, xl = pix % TW;
  const int gy = T.y0 + orow, gx = T.x0 + xl;
  if (gy >= P.H || gx >= P.W) return;
  if (!(primary_at<VAR, NOPRIM>(T, orow + r, xl + r) > 0.0)) return;  // centre invalid: nothing was fitted
  double h[HSums<VAR>::NH];
  int hi[HSums<VAR>::NHI];
  for (int k = 0; k < HSums<VAR>::NH; ++k) h[k] = 0.0;
  for (int k = 0; k < HSums<VAR>::NHI; ++k) hi[k] = 0;
  double tyo;
  if (direct && !CENTRED) {
    tyo = __ldg(P.tan_y + gy);
    for (int dy = -r; dy <= r; ++dy)
      for (int dx = -r; dx <= r; ++dx) {
        const double p = primary_at<VAR, NOPRIM>(T, orow + r + dy, xl + r + dx);
        if (p > 0.0) accum_sample<VAR>(h, hi, p, dx, dy);
      }
  } else {
    tyo = __ldg(P.tan_y + (CENTRED ? gy : T.y0));
    const double* vrow = T.vd + orow * T.VRS;
    const CountT<RT>* irow = static_cast<const CountT<RT>*>(T.vi) + orow * T.VRS;
    for (int k = 0; k <= 2 * r; ++k) {
      const int col = xl + k;
      accum_column<VAR>(h, hi, vrow, irow, TH * T.VRS, (col & 3) * T.VQ + (col >> 2), k - r, 1.0);
    }
  }
  const double txo = __ldg(P.tan_x + gx);
  const int nwin = hi[0];
  if (nwin < (EXP && P.do_exp ? 3 : 4)) return;
  const double nd = (double)nwin;
  const double invn = 1.0 / nd;
  Sym3 C;
  double mu0, mu1, mu2;
  assemble<VAR, RT == 0>(h, hi, txo, tyo, P, invn, C, mu0, mu1, mu2);
  const int64_t p = T.frame * P.out_frame + (int64_t)gy * P.W + gx;
  float kap = 0.0f;
  bool have_kap = false;
  if (P.do_imp && nwin >= 4 && !expl_only) {
    WindowFit f;
    solve_window<true>(C, mu0, mu1, mu2, nd, f);
    float nx, ny, nz, off;
    if (VAR == VAR_DF) finish_plane(f.u0, f.u1, f.s, f.u2, nx, ny, nz, off);
    else finish_plane(f.u0, f.u1, f.u2, f.s, nx, ny, nz, off);
    store_fit(P.imp, p, nx, ny, nz, off, fsqrt(fmaxf((float)(f.lam * invn), 0.0f)), f.kappa,
              RF_PIX_INPUT_VALID | RF_PIX_FIT | (f.degenerate ? RF_PIX_DEGENERATE : 0));
    kap = f.kappa;
    have_kap = true;
  }
  if (EXP && P.do_exp) {
    if (!have_kap) kap = curvature_only(C);
    if (direct || expl_only) {
      ExplicitFit ex;
      explicit_fit_robust(C, mu0, mu1, mu2, nd, ex);
      float a, b, c, d;
      if (VAR == VAR_DF) finish_plane(ex.a, ex.b, ex.c, -1.0, a, b, c, d);
      else finish_plane(ex.a, ex.b, -1.0, ex.c, a, b, c, d);
      store_fit(P.exp, p, a, b, c, d, fsqrt(fmaxf((float)(ex.ss * invn), 0.0f)), kap,
                RF_PIX_INPUT_VALID | RF_PIX_FIT | (ex.degenerate ? RF_PIX_DEGENERATE : 0));
    } else {
      P.exp.curvature[p] = kap;
    }
  }
}

// ---- 3. horizontal running sums + per-window fast solve + outputs of space VAR; each
// thread owns KSEG consecutive pixels of one output row.  Windows the fast solve declines
// and segments the sliding-sum guard flags are queued for the slow pass.
template <int VAR, int RT, bool EXP, bool NOPRIM>
__device__ __forceinline__ void row_pass(const TileCtx& T, const KParams& P, unsigned* s_dmax,
                                         unsigned short* s_q, int* s_qn) {
  constexpr bool CENTRED = RT > 0 && RT <= RF_CENTRED_MAX;
  constexpr int NH = HSums<VAR>::NH, NHI = HSums<VAR>::NHI;
  const int r = T.r, VQ = T.VQ, VRS = T.VRS, tid = T.tid;
  const int orow = tid / (TW / KSEG);
  const int xs = (tid % (TW / KSEG)) * KSEG;  // tile-local x of the segment's first pixel
  const int gy = T.y0 + orow;
  const int gxs = T.x0 + xs;
  if (gy >= P.H || gxs >= P.W) return;
  const double txo = T.txo;
  const double tyo = T.tyo;  // origin row of dy
  const double* vrow = T.vd + orow * VRS;
  const CountT<RT>* irow = static_cast<const CountT<RT>*>(T.vi) + orow * VRS;
  const int vstride = TH * VRS;
  if (!CENTRED && tid == 0) s_dmax[(T.it + 1) & 1] = 0u;  // read by the previous tile, written by the next
  // running horizontal sums (origin: segment start xs, tile row y0)
  double h[NH];
  int hi[NHI];
#pragma unroll
  for (int k = 0; k < NH; ++k) h[k] = 0.0;
#pragma unroll
  for (int k = 0; k < NHI; ++k) hi[k] = 0;
  // k: column offset from the segment start xs (xs is a multiple of 4, so the
  // residue-major position of column xs + k is a compile-time offset from vbase)
  const int vbase = xs >> 2;
  auto accum = [&](int k, double sgn) {
    accum_column<VAR>(h, hi, vrow, irow, vstride, vbase + (k & 3) * VQ + (k >> 2), k - r, sgn);
  };
  if constexpr (RT > 0) {
#pragma unroll
    for (int k = 0; k <= 2 * RT; ++k) accum(k, 1.0);
  } else {
    for (int k = 0; k <= 2 * r; ++k) accum(k, 1.0);
  }

#if RF_ROW_UNROLL
  float o_n[KSEG][3], o_off[KSEG], o_res[KSEG], o_cur[KSEG];
  uint8_t o_st[KSEG];
#pragma unroll
#else
  // one copy of the solve code per space (a fully unrolled segment loop quadruples the
  // kernel's instruction footprint: instruction-fetch stalls); outputs stored per pixel
#pragma unroll 1
#endif
  for (int j = 0; j < KSEG; ++j) {
#if RF_ABLATE < 3
    if (j > 0) {
      accum(j + 2 * r, 1.0);
      accum(j - 1, -1.0);
    }
#endif
    const int gx = gxs + j;
    const double pc = primary_at<VAR, NOPRIM>(T, orow + r, xs + j + r);
    uint8_t st = pc > 0.0 ? RF_PIX_INPUT_VALID : 0;
    const int nwin = (int)hi[0];
    float nx = __int_as_float(0x7fc00000), ny = nx, nz = nx, off = nx, res = nx, cur = nx;
    uint8_t stx = st;  // explicit-fit status (MIN_SAMPLES 3 instead of 4)
    if (st && nwin >= (EXP ? 3 : 4) && gx < P.W) {
      const double nd = (double)nwin;
      const double invn = inv_count(nwin);
      Sym3 C;
      double mu0, mu1, mu2;
      assemble<VAR, RT == 0>(h, hi, txo, tyo, P, invn, C, mu0, mu1, mu2);
      float kap = 0.0f;
      if (P.do_imp && nwin >= 4) {
        WindowFit f;
#if RF_ABLATE >= 1
        f.lam = C.c00 + C.c11; f.u0 = mu0 + C.c01; f.u1 = mu1 + C.c02; f.u2 = mu2 + C.c12; f.s = C.c22;
        f.kappa = 0.1f; f.degenerate = false;
        const bool fast = true;
#else
        const bool fast = solve_fast(C, mu0, mu1, mu2, nd, pos_d2f(invn), f);
#endif
        // windows the fast path declines are solved again by the robust path after the row
        // pass (slow_pixel), whose outputs overwrite these
        if (!fast) {
#ifdef RF_COUNT_SLOW
          atomicAdd(&g_slow_count[VAR], 1ull);
#endif
          const int qi = atomicAdd(s_qn, 1);
          if (qi < QCAP) s_q[qi] = (unsigned short)(orow * TW + xs + j);
        }
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
        if (e.degenerate) {  // rank-deficient: the minimum-norm solution in the slow pass
          const int qi = atomicAdd(s_qn, 1);
          if (qi < QCAP) s_q[qi] = (unsigned short)(Q_EXPL | (orow * TW + xs + j));
        }
        float ex, ey, ez, eo;
        // explicit_to_implicit (fitting.py:729-739): standard (a, b, -1, c), rgbd (a, b, c, -1)
        if (VAR == VAR_DF) finish_plane(e.a, e.b, e.c, -1.0, ex, ey, ez, eo);
        else finish_plane(e.a, e.b, -1.0, e.c, ex, ey, ez, eo);
        stx |= RF_PIX_FIT | (e.degenerate ? RF_PIX_DEGENERATE : 0);
        float* xs_ = T.xstage + 28 * tid;
        xs_[3 * j + 0] = ex;
        xs_[3 * j + 1] = ey;
        xs_[3 * j + 2] = ez;
        xs_[12 + j] = eo;
        xs_[16 + j] = fsqrt(fmaxf((float)(e.ss * invn), 0.0f));
        xs_[20 + j] = kap;
      }
    }
    if (EXP && P.do_exp) {
      float* xs_ = T.xstage + 28 * tid;
      if (!(stx & RF_PIX_FIT)) {
        const float qn = __int_as_float(0x7fc00000);
        xs_[3 * j + 0] = qn;
        xs_[3 * j + 1] = qn;
        xs_[3 * j + 2] = qn;
        xs_[12 + j] = qn;
        xs_[16 + j] = qn;
        xs_[20 + j] = qn;
      }
      reinterpret_cast<uint8_t*>(xs_ + 24)[j] = stx;
    }
#if RF_ROW_UNROLL
    o_n[j][0] = nx;
    o_n[j][1] = ny;
    o_n[j][2] = nz;
    o_off[j] = off;
    o_res[j] = res;
    o_cur[j] = cur;
    o_st[j] = st;
#else
    if (P.do_imp && gx < P.W) store_fit(P.imp, T.frame * P.out_frame + (int64_t)gy * P.W + gx, nx, ny, nz, off, res, cur, st);
#endif
  }

  const int64_t pix0 = T.frame * P.out_frame + (int64_t)gy * P.W + gxs;
  const bool vec = ((P.W & (KSEG - 1)) == 0) && (gxs + KSEG <= P.W);
  if (EXP && P.do_exp) {  // staged explicit outputs -> global, as vectors when aligned
    const float* xs_ = T.xstage + 28 * tid;
    if (vec) {
      const float4* sv = reinterpret_cast<const float4*>(xs_);
      float4* pn = reinterpret_cast<float4*>(P.exp.normal + 3 * pix0);
      pn[0] = sv[0];
      pn[1] = sv[1];
      pn[2] = sv[2];
      *reinterpret_cast<float4*>(P.exp.offset + pix0) = sv[3];
      *reinterpret_cast<float4*>(P.exp.residual + pix0) = sv[4];
      *reinterpret_cast<float4*>(P.exp.curvature + pix0) = sv[5];
      *reinterpret_cast<uchar4*>(P.exp.status + pix0) = *reinterpret_cast<const uchar4*>(xs_ + 24);
    } else {
      for (int j = 0; j < KSEG; ++j) {
        if (gxs + j >= P.W) break;
        const int64_t p = pix0 + j;
        P.exp.normal[3 * p + 0] = xs_[3 * j + 0];
        P.exp.normal[3 * p + 1] = xs_[3 * j + 1];
        P.exp.normal[3 * p + 2] = xs_[3 * j + 2];
        P.exp.offset[p] = xs_[12 + j];
        P.exp.residual[p] = xs_[16 + j];
        P.exp.curvature[p] = xs_[20 + j];
        P.exp.status[p] = reinterpret_cast<const uint8_t*>(xs_ + 24)[j];
      }
    }
  }
#if RF_ROW_UNROLL
  if (P.do_imp) {
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
  {
    // Sliding-sum guard.  A running sum keeps the rounding residue (~eps x value) of every
    // sample that has left it, so a window far smaller than the samples that slid through its
    // sums (a few millimetre depths in a column that just held metres) would inherit an error
    // the reference's direct sums do not have.  Mass that passed through one of this
    // segment's window sums outside the window: the row pass's 3 leading columns (their
    // vertical sums of p^2, read back), and with running column sums also the (o - o0)
    // leading rows of the column segment over 2r + 4 columns, each sample <= the largest p^2
    // that has left the tile's column sums (s_dmax).  A lower bound of a fitted window's own
    // sum of p^2 is its centre column's vertical sum, which holds the centre sample (columns
    // whose exact valid count is 0 belong to unfitted pixels and are skipped: their running
    // sums hold nothing but residue).  When the departed mass exceeds 2^20 x that bound
    // (millimetre depths next to metres; realistic scenes stay orders of magnitude below),
    // the segment's pixels are queued for the slow pass with direct window sums.  All of it
    // runs after the unrolled loop (no register held through the solve), in whole exponent
    // steps on the high words of the non-negative doubles (they order like the values).
    const int* vhi = reinterpret_cast<const int*>(T.vd + (TH + orow) * VRS + vbase) + 1;  // channel 1
    const CountT<RT>* cnt = irow + vbase;
    auto col_hi = [&](int k) { return vhi[2 * ((k & 3) * VQ + (k >> 2))]; };
    auto col_n = [&](int k) { return count_of(cnt[(k & 3) * VQ + (k >> 2)]); };
    // log2 of the departed mass, rounded up: 3 x the largest departed column sum ...
    int te = (max(col_hi(0), max(col_hi(1), col_hi(2))) >> 20) - 1023 + 2;
    if (!CENTRED) {  // ... and the (o - o0) x (2r + 4) samples that left the column sums
      // this row's column segment starts at o0 = floor(p TH / parts), p = its segment
      const int parts = max(1, min(NTHREADS / T.HW_, TH));
      const int seg = ((orow + 1) * parts + TH - 1) / TH - 1;
      const int rows = (orow - (seg * TH) / parts) * (2 * r + KSEG);
      if (rows > 0) te = max(te, 2 * ((int)(s_dmax[T.it & 1] >> 20) - 1023) + 32 - __clz(rows)) + 1;
    }
    te -= 20;  // / 2^20
    const int thr = te < -1022 ? 0 : te > 1023 ? 0x7ff00000 : (te + 1023) << 20;
    int h1min = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < KSEG; ++j) {
      const int w = col_hi(j + r);
      h1min = min(h1min, col_n(j + r) > 0 ? w : 0x7fffffff);  // exact valid count
    }
    if (h1min < thr) {
      const int qi = atomicAdd(s_qn, KSEG);
      for (int j = 0; j < KSEG && qi + j < QCAP; ++j) s_q[qi + j] = (unsigned short)(Q_DIRECT | (orow * TW + xs + j));
    }
  }
}

// ---- 4. the robust path for the windows the fast solve declined (and the guard's
// segments, with direct sums): each warp takes its own queue right after its row pass, one
// queued pixel per lane (the column sums it reads are the warp's own rows); an overflowing
// queue (more than QCAP such windows in the warp's rows: hostile inputs) redoes all of them.
template <int VAR, int RT, bool EXP, bool NOPRIM>
__device__ __forceinline__ void slow_pass(const TileCtx& T, const KParams& P, const unsigned short* q, int nq) {
  if (nq <= 0) return;
  const bool all = nq > QCAP;
  const int lane = T.tid & 31, pix0 = (T.tid >> 5) * RPW * TW;
  for (int i = lane; i < (all ? RPW * TW : nq); i += 32)
    slow_pixel<VAR, RT, EXP, NOPRIM>(T, P, all ? (Q_DIRECT | (pix0 + i)) : q[i]);
}

// Persistent tile kernel.  SP: spaces (bit 0 standard, bit 1 disparity form); USE_TMA;
// RT > 0: compile-time window radius (all halo geometry and shared-memory offsets fold to
// constants), RT == 0: runtime radius; EXP: explicit fits compiled in.  Ps / Pd: the
// standard / disparity-form space's parameters (the same input and geometry, their own
// outputs and requested formulations).
template <int SP, bool USE_TMA, int RT, bool EXP, int MINB = RF_MIN_BLOCKS>
__global__ void __launch_bounds__(NTHREADS, MINB)
    fit_tile_kernel(const __grid_constant__ KParams Ps, const __grid_constant__ KParams Pd,
                    const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) unsigned char smem_dyn[];
  const KParams& P = (SP & 1) ? Ps : Pd;  // input and geometry (identical in both)
  if (P.pdl_trigger == 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // TMA destinations must be 128-byte aligned: align the dynamic base explicitly
  // (pointer arithmetic on the __shared__ array, not integer casts, so every derived
  // pointer stays in the shared window and compiles to LDS/STS rather than generic LD/ST)
  unsigned char* smem_raw = smem_dyn + ((128u - (smem_u32(smem_dyn) & 127u)) & 127u);
  TileCtx T;
  T.P = &P;
  const int r = RT > 0 ? RT : P.r;
  T.r = r;
  T.HW_ = TW + 2 * r;  // halo width
  T.HH_ = TH + 2 * r;  // halo height
  const int HW_ = T.HW_, HH_ = T.HH_;
  constexpr int NVD = (SP & 1) ? 5 : 3;  // fp64 column-sum channels of the larger space
  T.esz = elem_size(P.dtype);
  const int esz = T.esz;
  const int al = 16 / esz;  // TMA box x origin must be 16-byte aligned
  T.HWP = (HW_ + al - 1 + 7) & ~7;  // TMA box width (covers the alignment shift)
  const int HWP = T.HWP;
  const int raw_bytes = USE_TMA ? ((HH_ * HWP * esz + 127) & ~127) : 0;
  // ZF (the largest compile-time radius): the standard space's Z tile is float (float32 input
  // only: rf_fit_pixels routes other element types to the generic kernel), so two CTAs fit
  constexpr bool NOPRIM = noprim_radius(RT) && USE_TMA;  // ZF
  constexpr int PSP = SP;
  constexpr int NRAW = 1;  // the conversion consumes the raw box before the tile's barrier
  unsigned char* raw0 = smem_raw;
  unsigned char* raw1 = smem_raw + (NRAW - 1) * raw_bytes;
  // small compile-time radii: warp-local column and row passes; the converted halo is
  // double-buffered so that the tile's one CTA barrier (after the conversion) also orders the
  // next conversion after every warp's last read of the buffer it overwrites
  constexpr bool CENTRED = RT > 0 && RT <= RF_CENTRED_MAX;
  // one space per launch: the double buffer fits two CTAs per SM; both spaces (small
  // batches) keep one buffer and close the tile with a barrier instead
  constexpr bool DBUF = CENTRED && RT <= 3 && SP != 3 && (MINB < 3 || TH <= 8);
  const int nprim = HH_ * HW_;
  const int nsp = ((PSP & 2) ? 1 : 0) + ((PSP & 1) && !NOPRIM ? 1 : 0);  // fp64 tiles
  double* prim_base = reinterpret_cast<double*>(smem_raw + NRAW * raw_bytes);  // [DBUF ? 2 : 1][nsp][HH_][HW_]
  T.pw = prim_base;                              // [HH_][HW_]
  T.pz = T.pw + ((PSP & 2) ? nprim : 0);         // [HH_][HW_]
  T.pzf = reinterpret_cast<float*>(prim_base + (DBUF ? 2 : 1) * nsp * nprim);  // [HH_][HW_] (ZF)
  // column sums are stored residue-major: column c at (c % 4) * VQ + c / 4, so the row
  // pass (threads 4 columns apart) reads consecutive addresses -- no bank conflicts.
  T.VQ = NOPRIM ? (HW_ + 3) / 4 : vq_of(HW_);
  T.VRS = 4 * T.VQ;
  const int VRS = T.VRS;
  T.vd = prim_base + (DBUF ? 2 : 1) * nsp * nprim +
         (((SP & 1) && NOPRIM) ? (nprim + 1) / 2 : 0);                  // [NVD][TH][VRS]
  T.vi = T.vd + NVD * TH * VRS;                                        // [TH][VRS] CountT<RT>
  uint64_t* bars = reinterpret_cast<uint64_t*>(static_cast<unsigned char*>(T.vi) +
                                               ((sizeof(CountT<RT>) * TH * VRS + 7) & ~(size_t)7));
  // explicit fits stage their 4 pixels' outputs in shared memory (7 float4 per thread: the
  // implicit outputs already hold the register budget) and store them as vectors
  T.xstage = reinterpret_cast<float*>(bars + 2);

  const int tid = threadIdx.x;
  T.tid = tid;
  const int ntx = (P.W + TW - 1) / TW, nty = (P.H + TH - 1) / TH;
  const int64_t total = (int64_t)ntx * nty * P.batch;
  const uint32_t box_bytes = (uint32_t)(HH_ * HWP * esz);
  // running column sums: high word of the largest primary that has left the tile's column
  // sums (p >= 0, so high words order like the values), per space and double-buffered by
  // tile parity; the sliding-sum guard's departed-mass bound at the end of the row pass
  __shared__ unsigned s_dmax[2][2];
  // slow-pass queue (QCAP tile-local pixel indices) and its fill count
  // per-warp slow-pass queues (QCAP pixel indices of the warp's rows) and their fill counts
  __shared__ unsigned short s_q[NWARPS][QCAP];
  __shared__ int s_qn[NWARPS];
  const int warp = tid >> 5;
  if (tid == 0) s_dmax[0][0] = s_dmax[0][1] = s_dmax[1][0] = s_dmax[1][1] = 0u;
  if (tid < NWARPS) s_qn[tid] = 0;
  __syncthreads();

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
  TileIter ti(blockIdx.x, gridDim.x, ntx, nty);
  for (int64_t t = blockIdx.x; t < total; t += gridDim.x, ++it, ti.advance()) {
    const TileGeom g = ti.geom();
    T.frame = g.frame;
    T.x0 = g.x0;
    T.y0 = g.y0;
    T.it = it;
    const int64_t frame = g.frame;
    const int x0 = g.x0, y0 = g.y0;
    T.raw = (it & 1) ? raw1 : raw0;
    if (DBUF) {
      T.pw = prim_base + (it & 1) * nsp * nprim;
      T.pz = T.pw + ((PSP & 2) ? nprim : 0);
    }
    {
      // the row pass's tan origins (clamped: threads past the frame edge return before use)
      const int orow = tid / (TW / KSEG), xs = (tid % (TW / KSEG)) * KSEG;
      T.txo = __ldg(P.tan_x + min(x0 + xs, P.W - 1));
      T.tyo = __ldg(P.tan_y + (CENTRED ? min(y0 + orow, P.H - 1) : y0));
    }
    T.sx = (x0 - r) - box_x(x0 - r, al);  // raw index shift
    T.sy = (y0 - r) - max(y0 - r, 0);

    // ---- 1. halo tile -> primaries
    if (USE_TMA) {
      const int b = it & 1;
      mbar_wait(&bars[b], (uint32_t)((it >> 1) & 1));
      if (PSP != 0) {
        if (esz == 2)
          convert_halo<PSP, NOPRIM>(T.pw, T.pz, T.pzf, reinterpret_cast<const unsigned short*>(T.raw), HW_, HH_, HWP, T.sx, T.sy, P,
                           frame, x0, y0, r, tid);
        else if (esz == 8)
          convert_halo<PSP, NOPRIM>(T.pw, T.pz, T.pzf, reinterpret_cast<const double*>(T.raw), HW_, HH_, HWP, T.sx, T.sy, P, frame,
                           x0, y0, r, tid);
        else
          convert_halo<PSP, NOPRIM>(T.pw, T.pz, T.pzf, reinterpret_cast<const float*>(T.raw), HW_, HH_, HWP, T.sx, T.sy, P, frame,
                           x0, y0, r, tid);
        __syncthreads();
      }
      // the other buffer was consumed by the previous tile (its last reads precede the
      // end-of-tile barrier): prefetch the next tile into it now
      if (tid == 0 && t + gridDim.x < total) {
        TileIter tn = ti;
        tn.advance();
        const TileGeom gn = tn.geom();
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
          bool valid = false;
          double z = 0.0;
          if (yin && x >= 0 && x < P.W) {
            const int64_t off = frame * P.frame_stride + (int64_t)y * P.row_pitch + x;
            z = esz == 2   ? depth_z(__ldg(reinterpret_cast<const unsigned short*>(P.depth) + off), valid)
                : esz == 8 ? depth_z(__ldg(reinterpret_cast<const double*>(P.depth) + off), valid)
                           : depth_z(__ldg(reinterpret_cast<const float*>(P.depth) + off), valid);
            if (P.mask) valid = valid && __ldg(P.mask + frame * P.out_frame + (int64_t)y * P.W + x) != 0;
          }
          if (SP & 2) T.pw[row * HW_ + col] = valid ? rcp_fast(z) : 0.0;
          if (SP & 1) T.pz[row * HW_ + col] = valid ? z : 0.0;
        }
      }
      __syncthreads();
    }

    // ---- 2-4 per space: disparity form first, then standard (one column-sum buffer).
    // Small radii: all warp-local after the conversion's barrier.  Running column sums are
    // CTA-wide (a column segment spans many warps' rows): barriers around them.
    auto space = [&](auto var_tag, auto counts_tag, const KParams& Pv) {
      constexpr int VAR = decltype(var_tag)::value;
      constexpr bool NP = VAR == VAR_STD && NOPRIM;
#if RF_ABLATE < 4
      column_pass<VAR, RT, NP, decltype(counts_tag)::value>(T, s_dmax[VAR]);
#endif
      if (CENTRED) __syncwarp();
      else __syncthreads();
      row_pass<VAR, RT, EXP, NP>(T, Pv, s_dmax[VAR], s_q[warp], &s_qn[warp]);
      __syncwarp();  // the warp's queue is complete
      const int nq = s_qn[warp];
      slow_pass<VAR, RT, EXP, NP>(T, Pv, s_q[warp], nq);
      __syncwarp();  // every lane has read the count
      if ((tid & 31) == 0) s_qn[warp] = 0;
      if (!CENTRED) __syncthreads();  // the next column pass rewrites every warp's rows
    };
    if constexpr ((SP & 2) != 0) space(std::integral_constant<int, VAR_DF>(), std::integral_constant<int, 2>(), Pd);
    if constexpr ((SP & 1) != 0)
      space(std::integral_constant<int, VAR_STD>(), std::integral_constant<int, (SP & 2) ? 0 : 1>(), Ps);
    if (CENTRED && !DBUF) __syncthreads();  // the single halo buffer is rewritten next
    else if (CENTRED) __syncwarp();
  }
}


// per kernel instantiation: the opt-in shared memory it was last configured for and its
// occupancy at that size (cudaFuncSetAttribute / the occupancy query run once, not per call)
struct KernelCache {
  std::mutex mu;
  size_t smem = 0;
  int per_sm = 0;
};

template <int SP, bool TMA, int RT, bool EXP, int MINB = RF_MIN_BLOCKS>
cudaError_t launch_sp(const KParams& Ps, const KParams& Pd, const CUtensorMap& tmap, size_t sm, int64_t tiles,
                      int sms, cudaStream_t s, bool pdl) {
  auto kern = fit_tile_kernel<SP, TMA, RT, EXP, MINB>;
  static KernelCache kc;
  int per_sm;
  {
    std::lock_guard<std::mutex> lock(kc.mu);
    if (sm > kc.smem) {
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      kc.smem = sm;
      kc.per_sm = 0;
    }
    if (kc.per_sm == 0 || sm != kc.smem) {
      int n = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, NTHREADS, sm);
      per_sm = n < 1 ? 1 : n;
      if (sm == kc.smem) kc.per_sm = per_sm;
    } else {
      per_sm = kc.per_sm;
    }
  }
  const int64_t grid = tiles < (int64_t)sms * per_sm ? tiles : (int64_t)sms * per_sm;
  if (!pdl) {
    kern<<<(unsigned)grid, NTHREADS, sm, s>>>(Ps, Pd, tmap);
    return cudaGetLastError();
  }
  // the second space's launch of a call: programmatic dependent launch -- it shares no data
  // with the first (same input, its own outputs), so its CTAs take SMs as the first
  // kernel's CTAs retire (every CTA of fit_tile_kernel releases its dependents at entry)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, Ps, Pd, tmap);
}

template <int SP, bool TMA, int RT>
cudaError_t launch_var(const KParams& Ps, const KParams& Pd, const CUtensorMap& tmap, size_t sm, int64_t tiles,
                       int sms, cudaStream_t s, bool pdl = false, bool three = false) {
  const bool exp = ((SP & 1) && Ps.do_exp) || ((SP & 2) && Pd.do_exp);
  if constexpr (SP != 3 && TMA && RT >= 1 && RT <= 3) {
    if (three && !exp) return launch_sp<SP, TMA, RT, false, 3>(Ps, Pd, tmap, sm, tiles, sms, s, pdl);
  }
  return exp ? launch_sp<SP, TMA, RT, true>(Ps, Pd, tmap, sm, tiles, sms, s, pdl)
             : launch_sp<SP, TMA, RT, false>(Ps, Pd, tmap, sm, tiles, sms, s, pdl);
}

// compile-time radii for the BASELINE windows 3, 5, 7, 9, 11, 15, 31; others run generic
template <int SP>
cudaError_t launch_radius(const KParams& Ps, const KParams& Pd, const CUtensorMap& tmap, bool tma, size_t sm,
                          int64_t tiles, int sms, cudaStream_t s, bool pdl = false, bool three = false) {
  if (!tma) return launch_var<SP, false, 0>(Ps, Pd, tmap, sm, tiles, sms, s, pdl, three);
  switch (Ps.r) {
    case 1: return launch_var<SP, true, 1>(Ps, Pd, tmap, sm, tiles, sms, s, pdl, three);
    case 2: return launch_var<SP, true, 2>(Ps, Pd, tmap, sm, tiles, sms, s, pdl, three);
    case 3: return launch_var<SP, true, 3>(Ps, Pd, tmap, sm, tiles, sms, s, pdl, three);
    case 4: return launch_var<SP, true, 4>(Ps, Pd, tmap, sm, tiles, sms, s, pdl, three);
    case 5: return launch_var<SP, true, 5>(Ps, Pd, tmap, sm, tiles, sms, s, pdl, three);
    case 7: return launch_var<SP, true, 7>(Ps, Pd, tmap, sm, tiles, sms, s, pdl, three);
    case 15:  // the float Z tile holds float32 depths exactly; other element types: generic radius
      if ((SP & 1) && elem_size(Ps.dtype) != 4) return launch_var<SP, true, 0>(Ps, Pd, tmap, sm, tiles, sms, s, pdl, three);
      return launch_var<SP, true, 15>(Ps, Pd, tmap, sm, tiles, sms, s, pdl, three);
    default: return launch_var<SP, true, 0>(Ps, Pd, tmap, sm, tiles, sms, s, pdl, three);
  }
}

}  // namespace rf_fitk
