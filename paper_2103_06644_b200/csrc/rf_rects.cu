// rf_rects.cu -- batched arbitrary-rectangle fits ("K5"):
// the reference's per-window entry fit_rect(depth, maps, rect, formulation,
// backend) (fitting.py:757-786) evaluated for a list of rects on the device.
//
// One CTA per rect.  Threads stride over the rect's pixels (row-major, so warps
// read contiguous runs of a row), accumulate the rect's raw moments in local
// coordinates about the rect centre (exact integer geometry, fp64 depth moments
// -- the naive backend's direct sums, fitting.py:339-402, never an image-global
// summed-area table), reduce them across the CTA, and thread 0 solves with the
// same device code as the per-pixel kernels (rf_solve.cuh).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/rangefit_b200.h"
#include "rf_internal.h"
#include "rf_solve.cuh"
#include "rf_jacobi.cuh"
#include "rf_general.cuh"

namespace {
using namespace rf_dev;

constexpr int RT_THREADS = 128;

struct RectParams {
  const void* depth;
  const uint8_t* mask;
  const double* tan_x;
  const double* tan_y;
  const double* lat_x;  // non-separable tan lattices [H][W] (distortion offsets), else null
  const double* lat_y;
  double ifx, ify;
  int64_t row_pitch, frame_stride, out_frame, batch;
  int H, W, dtype, formulation;
  const rf_rect* rects;
  int64_t nrects;
  rf_rect_fit* out;
};

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < RT_THREADS / 32; ++w) t += red[w];
  return t;  // valid on thread 0
}

__device__ __forceinline__ long long block_sum_ll(long long v, long long* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  long long t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < RT_THREADS / 32; ++w) t += red[w];
  return t;
}

__global__ void __launch_bounds__(RT_THREADS) fit_rects_kernel(const RectParams P) {
  __shared__ double redd[RT_THREADS / 32];
  __shared__ long long redl[RT_THREADS / 32];
  const int64_t ri = blockIdx.x;
  if (ri >= P.nrects) return;
  const rf_rect R = P.rects[ri];
  rf_rect_fit* o = P.out + ri;
  const bool space_std = P.formulation == RF_FORM_IMPLICIT_STANDARD || P.formulation == RF_FORM_EXPLICIT_STANDARD;
  const bool explicit_fit = P.formulation >= RF_FORM_EXPLICIT_STANDARD;
  // _check_rect (integral.py:131-133): 0 <= x0 <= x1 <= W, 0 <= y0 <= y1 <= H
  if (!(R.frame >= 0 && R.frame < P.batch && 0 <= R.x0 && R.x0 <= R.x1 && R.x1 <= P.W && 0 <= R.y0 &&
        R.y0 <= R.y1 && R.y1 <= P.H)) {
    if (threadIdx.x == 0) {
      memset(o, 0, sizeof(*o));
      o->status = RF_RECT_OUT_OF_BOUNDS;
      o->n_points = 0;
    }
    return;
  }
  const int rw = R.x1 - R.x0, rh = R.y1 - R.y0;
  const int ox = R.x0 + rw / 2, oy = R.y0 + rh / 2;  // local origin near the centre
  const int64_t area = (int64_t)rw * rh;
  // moments: q = (dx, dy, w) disparity form / (dx Z, dy Z, Z) standard
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0, s7 = 0, s8 = 0;
  long long n = 0, gx = 0, gy = 0, gxx = 0, gxy = 0, gyy = 0;
  for (int64_t e = threadIdx.x; e < area; e += RT_THREADS) {
    const int yy = (int)(e / rw), xx = (int)(e - (int64_t)yy * rw);
    const int y = R.y0 + yy, x = R.x0 + xx;
    const int64_t off = (int64_t)R.frame * P.frame_stride + (int64_t)y * P.row_pitch + x;
    double z;
    bool valid;
    if (P.dtype == RF_DEPTH_U16_MM) {
      const unsigned short mm = __ldg(reinterpret_cast<const unsigned short*>(P.depth) + off);
      valid = mm > 0;
      z = __ddiv_rn((double)mm, 1000.0);
    } else if (P.dtype == RF_DEPTH_F64_M) {
      z = __ldg(reinterpret_cast<const double*>(P.depth) + off);
      valid = (z > 0.0) && (z <= 1.7976931348623157e308);
    } else {
      const float zf = __ldg(reinterpret_cast<const float*>(P.depth) + off);
      valid = (zf > 0.0f) && (zf <= 3.402823466e38f);
      z = (double)zf;
    }
    if (P.mask) valid = valid && __ldg(P.mask + (int64_t)R.frame * P.out_frame + (int64_t)y * P.W + x) != 0;
    if (!valid) continue;
    if (P.lat_x) {  // general moments of q about the rect centre's tan values (rf_general.cuh)
      const int64_t li = (int64_t)y * P.W + x, lc = (int64_t)oy * P.W + ox;
      const double dtx = P.lat_x[li] - P.lat_x[lc], dty = P.lat_y[li] - P.lat_y[lc];
      const double q0 = space_std ? z * dtx : dtx, q1 = space_std ? z * dty : dty;
      const double q2 = space_std ? z : 1.0 / z;
      s0 += q0;
      s1 += q1;
      s2 += q2;
      s3 = fma(q0, q0, s3);
      s4 = fma(q0, q1, s4);
      s5 = fma(q0, q2, s5);
      s6 = fma(q1, q1, s6);
      s7 = fma(q1, q2, s7);
      s8 = fma(q2, q2, s8);
      n += 1;
      continue;
    }
    const int dx = x - ox, dy = y - oy;
    const double fdx = (double)dx, fdy = (double)dy;
    if (!space_std) {
      const double w = rcp_fast(z);
      s0 += w;
      s1 = fma(w, w, s1);
      s2 = fma(fdx, w, s2);
      s3 = fma(fdy, w, s3);
      n += 1;
      gx += dx;
      gy += dy;
      gxx += (long long)dx * dx;
      gxy += (long long)dx * dy;
      gyy += (long long)dy * dy;
    } else {
      const double z2 = z * z, xz = fdx * z, yz = fdy * z;
      s0 += z;                   // S3
      s1 += z2;                  // S33
      s2 += xz;                  // S1
      s3 += yz;                  // S2
      s4 = fma(xz, xz, s4);      // S11
      s5 = fma(xz, yz, s5);      // S12
      s6 = fma(yz, yz, s6);      // S22
      s7 = fma(fdx, z2, s7);     // S13
      s8 = fma(fdy, z2, s8);     // S23
      n += 1;
    }
  }
  s0 = block_sum(s0, redd);
  s1 = block_sum(s1, redd);
  s2 = block_sum(s2, redd);
  s3 = block_sum(s3, redd);
  if (space_std || P.lat_x) {
    s4 = block_sum(s4, redd);
    s5 = block_sum(s5, redd);
    s6 = block_sum(s6, redd);
    s7 = block_sum(s7, redd);
    s8 = block_sum(s8, redd);
  }
  n = block_sum_ll(n, redl);
  if (!space_std && !P.lat_x) {
    gx = block_sum_ll(gx, redl);
    gy = block_sum_ll(gy, redl);
    gxx = block_sum_ll(gxx, redl);
    gxy = block_sum_ll(gxy, redl);
    gyy = block_sum_ll(gyy, redl);
  }
  if (threadIdx.x != 0) return;

  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  rf_rect_fit res;
  for (int k = 0; k < 4; ++k) res.coef[k] = qnan;
  for (int k = 0; k < 3; ++k) res.explicit_coef[k] = qnan;
  res.eigenvalue = res.rms = res.curvature = qnan;
  res.n_points = (int32_t)n;
  res.status = 0;
  const int min_samples = explicit_fit ? 3 : 4;  // MIN_SAMPLES fitting.py:55-60
  if (n >= min_samples) {
    const double txo = P.tan_x[ox], tyo = P.tan_y[oy];
    const double ifx = P.ifx, ify = P.ify;
    const double nd = (double)n, invn = 1.0 / nd;
    Sym3 C;
    double mu0, mu1, mu2;
    if (P.lat_x) {
      QMoments m;
      m.n = nd;
      m.s0 = s0; m.s1 = s1; m.s2 = s2; m.s00 = s3; m.s01 = s4; m.s02 = s5; m.s11 = s6; m.s12 = s7; m.s22 = s8;
      const int64_t lc = (int64_t)oy * P.W + ox;
      q_to_scatter(space_std, m, P.lat_x[lc], P.lat_y[lc], C, mu0, mu1, mu2);
    } else if (!space_std) {
      // geometry moments about the rect centre (|gx|, |gy| small relative to gxx, gyy)
      const double fgx = (double)gx, fgy = (double)gy;
      const double cq00 = fma(-fgx, fgx * invn, (double)gxx);
      const double cq01 = fma(-fgx, fgy * invn, (double)gxy);
      const double cq11 = fma(-fgy, fgy * invn, (double)gyy);
      const double mw = s0 * invn;
      C.c00 = cq00 * (ifx * ifx);
      C.c01 = cq01 * (ifx * ify);
      C.c11 = cq11 * (ify * ify);
      C.c02 = fma(-(double)gx, mw, s2) * ifx;
      C.c12 = fma(-(double)gy, mw, s3) * ify;
      C.c22 = fma(-s0, mw, s1);
      mu0 = fma((double)gx * invn, ifx, txo);
      mu1 = fma((double)gy * invn, ify, tyo);
      mu2 = mw;
    } else {
      const double q0 = s2 * invn, q1 = s3 * invn, q2 = s0 * invn;
      const double k00 = fma(-s2, q0, s4), k01 = fma(-s2, q1, s5), k02 = fma(-s2, q2, s7);
      const double k11 = fma(-s3, q1, s6), k12 = fma(-s3, q2, s8), k22 = fma(-s0, q2, s1);
      const double r00 = fma(ifx, k00, txo * k02), r01 = fma(ifx, k01, txo * k12), r02 = fma(ifx, k02, txo * k22);
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
    if (!explicit_fit) {
      WindowFit f;
      solve_window(C, mu0, mu1, mu2, nd, f);
      if (space_std) canonical4(f.u0, f.u1, f.u2, f.s, res.coef);
      else canonical4(f.u0, f.u1, f.s, f.u2, res.coef);
      res.eigenvalue = f.lam;
      res.rms = sqrt(fmax(f.lam, 0.0) / nd);
      res.curvature = f.kappa;
      res.status = RF_RECT_FIT | (f.degenerate ? RF_RECT_DEGENERATE : 0);
    } else {
      ExplicitFit e;
      explicit_fit_robust(C, mu0, mu1, mu2, nd, e);
      res.explicit_coef[0] = e.a;
      res.explicit_coef[1] = e.b;
      res.explicit_coef[2] = e.c;
      // explicit_to_implicit (fitting.py:729-739)
      if (space_std) canonical4(e.a, e.b, -1.0, e.c, res.coef);
      else canonical4(e.a, e.b, e.c, -1.0, res.coef);
      res.rms = sqrt(fmax(e.ss, 0.0) / nd);
      res.curvature = curvature_only(C);
      res.status = RF_RECT_FIT | (e.degenerate ? RF_RECT_DEGENERATE : 0);
    }
  }
  *o = res;
}

// _max_residual (segment.py:306-325): max |objective| over a rect's valid pixels for a
// given plane, evaluated like the reference's numpy expression (left to right, unfused),
// one CTA per rect.  coefs: [nrects][4] -- the canonical implicit coefficients (implicit
// forms) or the explicit (a, b, c, unused).
struct MaxResParams {
  RectParams base;
  const double* coefs;
  double* out;
};

__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < RT_THREADS / 32; ++w) t = fmax(t, red[w]);
  return t;
}

__global__ void __launch_bounds__(RT_THREADS) max_residual_kernel(const MaxResParams M) {
  __shared__ double red[RT_THREADS / 32];
  const RectParams& P = M.base;
  const int64_t ri = blockIdx.x;
  if (ri >= P.nrects) return;
  const rf_rect R = P.rects[ri];
  if (!(R.frame >= 0 && R.frame < P.batch && 0 <= R.x0 && R.x0 <= R.x1 && R.x1 <= P.W && 0 <= R.y0 &&
        R.y0 <= R.y1 && R.y1 <= P.H)) {
    if (threadIdx.x == 0) M.out[ri] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  const double c0 = M.coefs[4 * ri], c1 = M.coefs[4 * ri + 1], c2 = M.coefs[4 * ri + 2], c3 = M.coefs[4 * ri + 3];
  const int rw = R.x1 - R.x0;
  const int64_t area = (int64_t)rw * (R.y1 - R.y0);
  double mx = 0.0;  // max of |res| >= 0; an empty rect reports 0 as the reference
  for (int64_t e = threadIdx.x; e < area; e += RT_THREADS) {
    const int yy = (int)(e / rw), xx = (int)(e - (int64_t)yy * rw);
    const int y = R.y0 + yy, x = R.x0 + xx;
    const int64_t off = (int64_t)R.frame * P.frame_stride + (int64_t)y * P.row_pitch + x;
    double z;
    bool valid;
    if (P.dtype == RF_DEPTH_U16_MM) {
      const unsigned short mm = __ldg(reinterpret_cast<const unsigned short*>(P.depth) + off);
      valid = mm > 0;
      z = __ddiv_rn((double)mm, 1000.0);
    } else if (P.dtype == RF_DEPTH_F64_M) {
      z = __ldg(reinterpret_cast<const double*>(P.depth) + off);
      valid = (z > 0.0) && (z <= 1.7976931348623157e308);
    } else {
      const float zf = __ldg(reinterpret_cast<const float*>(P.depth) + off);
      valid = (zf > 0.0f) && (zf <= 3.402823466e38f);
      z = (double)zf;
    }
    if (P.mask) valid = valid && __ldg(P.mask + (int64_t)R.frame * P.out_frame + (int64_t)y * P.W + x) != 0;
    if (!valid) continue;
    const double tx = rf_tan(P.tan_x, P.lat_x, P.W, x, y, true), ty = rf_tan(P.tan_y, P.lat_y, P.W, x, y, false);
    double r;
    switch (P.formulation) {
      case RF_FORM_IMPLICIT_STANDARD:  // c0 z tx + c1 z ty + c2 z + c3
        r = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(c0, z), tx), __dmul_rn(__dmul_rn(c1, z), ty)),
                                __dmul_rn(c2, z)), c3);
        break;
      case RF_FORM_IMPLICIT_RGBD:  // c0 tx + c1 ty + c2 + c3 / z
        r = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(c0, tx), __dmul_rn(c1, ty)), c2), __ddiv_rn(c3, z));
        break;
      case RF_FORM_EXPLICIT_STANDARD:  // a z tx + b z ty + c - z
        r = __dsub_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(c0, z), tx), __dmul_rn(__dmul_rn(c1, z), ty)), c2), z);
        break;
      default:  // a tx + b ty + c - 1 / z
        r = __dsub_rn(__dadd_rn(__dadd_rn(__dmul_rn(c0, tx), __dmul_rn(c1, ty)), c2), __ddiv_rn(1.0, z));
        break;
    }
    mx = fmax(mx, fabs(r));
  }
  mx = block_max(mx, red);
  if (threadIdx.x == 0) M.out[ri] = mx;
}

}  // namespace

extern "C" {

rf_status rf_max_residuals(const rf_tables* t, const void* depth, int dtype, int64_t batch, int32_t H,
                           int32_t W, int64_t row_pitch, const uint8_t* mask, const rf_rect* rects,
                           int64_t nrects, int32_t formulation, const double* coefs, double* out, void* stream) {
  if (!t) return rf_set_error(RF_ERR_ARGUMENT, "rf_max_residuals: null tables");
  if (dtype != RF_DEPTH_F32_M && dtype != RF_DEPTH_U16_MM && dtype != RF_DEPTH_F64_M)
    return rf_set_error(RF_ERR_SHAPE, "rf_max_residuals: unknown depth dtype");
  if (H != t->intr.height || W != t->intr.width)
    return rf_set_error(RF_ERR_SHAPE, "rf_max_residuals: depth size does not match the camera tables");
  if (formulation < 0 || formulation >= RF_NUM_FORMULATIONS)
    return rf_set_error(RF_ERR_ARGUMENT, "rf_max_residuals: unknown formulation");
  if (batch < 0 || nrects < 0 || row_pitch < W)
    return rf_set_error(RF_ERR_ARGUMENT, "rf_max_residuals: bad batch / rect count / row pitch");
  if (nrects == 0) return RF_OK;
  if (!depth || !rects || !coefs || !out || nrects > 0x7fffffff)
    return rf_set_error(RF_ERR_ARGUMENT, "rf_max_residuals: null pointer");
  const rf_device_guard guard(t->device);
  MaxResParams M;
  RectParams& P = M.base;
  P.depth = depth;
  P.mask = mask;
  P.tan_x = t->tan_x;
  P.tan_y = t->tan_y;
  P.lat_x = t->lat_x;
  P.lat_y = t->lat_y;
  P.ifx = 1.0 / t->intr.fx;
  P.ify = 1.0 / t->intr.fy;
  P.row_pitch = row_pitch;
  P.frame_stride = row_pitch * H;
  P.out_frame = (int64_t)H * W;
  P.batch = batch;
  P.H = H;
  P.W = W;
  P.dtype = dtype;
  P.formulation = formulation;
  P.rects = rects;
  P.nrects = nrects;
  P.out = nullptr;
  M.coefs = coefs;
  M.out = out;
  max_residual_kernel<<<(unsigned)nrects, RT_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(M);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return rf_set_error(RF_ERR_CUDA, cudaGetErrorString(e));
  return RF_OK;
}

rf_status rf_fit_rects(const rf_tables* t, const void* depth, int dtype, int64_t batch, int32_t H,
                       int32_t W, int64_t row_pitch, const uint8_t* mask, const rf_rect* rects,
                       int64_t nrects, int32_t formulation, rf_rect_fit* out, void* stream) {
  if (!t) return rf_set_error(RF_ERR_ARGUMENT, "rf_fit_rects: null tables");
  if (dtype != RF_DEPTH_F32_M && dtype != RF_DEPTH_U16_MM && dtype != RF_DEPTH_F64_M)
    return rf_set_error(RF_ERR_SHAPE, "rf_fit_rects: unknown depth dtype");
  if (H != t->intr.height || W != t->intr.width)
    return rf_set_error(RF_ERR_SHAPE, "rf_fit_rects: depth size does not match the camera tables");
  if (formulation < 0 || formulation >= RF_NUM_FORMULATIONS)
    return rf_set_error(RF_ERR_ARGUMENT, "rf_fit_rects: unknown formulation");
  if (batch < 0 || nrects < 0 || row_pitch < W)
    return rf_set_error(RF_ERR_ARGUMENT, "rf_fit_rects: bad batch / rect count / row pitch");
  if (nrects == 0) return RF_OK;
  if (!depth || !rects || !out || nrects > 0x7fffffff)
    return rf_set_error(RF_ERR_ARGUMENT, "rf_fit_rects: null depth / rects / out");
  const rf_device_guard guard(t->device);
  RectParams P;
  P.depth = depth;
  P.mask = mask;
  P.tan_x = t->tan_x;
  P.tan_y = t->tan_y;
  P.lat_x = t->lat_x;
  P.lat_y = t->lat_y;
  P.ifx = 1.0 / t->intr.fx;
  P.ify = 1.0 / t->intr.fy;
  P.row_pitch = row_pitch;
  P.frame_stride = row_pitch * H;
  P.out_frame = (int64_t)H * W;
  P.batch = batch;
  P.H = H;
  P.W = W;
  P.dtype = dtype;
  P.formulation = formulation;
  P.rects = rects;
  P.nrects = nrects;
  P.out = out;
  fit_rects_kernel<<<(unsigned)nrects, RT_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(P);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return rf_set_error(RF_ERR_CUDA, cudaGetErrorString(e));
  return RF_OK;
}

}  // extern "C"
