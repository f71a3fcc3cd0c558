// rf_integral.cu -- the reference's integral backend on the device (SURVEY.md 8a rows
// A5-A8 and A10, 8b "what the drop-in must export"): per-frame channel summed-area
// tables (build_*_channels / build_integral, integral.py:136-325), box sums (_box /
// box_sum, fitting.py:405-411, integral.py:152-158) and the fits of assembled scatter
// systems (fit_implicit_* / fit_explicit_*, fitting.py:264-327, 546-629).
//
// Tables are built the way numpy builds them -- each pixel's channel value with the
// reference's fp64 expression, masked to +0.0, then np.cumsum along axis 0 (one thread
// per column, sequential down the column, coalesced across the warp) and along axis 1
// (one lane per row, sequential along the row through a 32x32 shared-memory transpose so
// that the global accesses stay coalesced) -- the same additions in the same order, so
// the tables are the reference's bit for bit.
//
// The scatter fits run one thread per system.  Implicit systems use the per-pixel
// kernels' solve (rf_solve.cuh) on the Schur complement of the constant monomial, checked
// by its eigen-residual; a cyclic Jacobi (the reference's rotation rule,
// fitting.py:193-253) covers hand-made systems the pencil cannot represent (constant-
// monomial entry not positive, or the constant monomial alone as the smallest
// eigenvector) and the minimum-norm solve of rank-deficient explicit systems
// (_pinv_solve, fitting.py:313-327).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "../../include/rangefit_b200.h"
#include "rf_internal.h"
#include "rf_solve.cuh"
#include "rf_jacobi.cuh"

namespace {
using namespace rf_dev;

constexpr int SCAN_THREADS = 128;
constexpr int ROW_WARPS = 4;

struct ChanParams {
  const void* depth;
  int dtype;
  int64_t row_pitch;
  const uint8_t* mask;
  const double* tan_x;
  const double* tan_y;
  const double* lat_x;  // non-separable lattices (distortion offsets) or null
  const double* lat_y;
  const double* src;  // generic channel (rf_integral) when channel < 0
  int64_t src_pitch;
  int H, W, channel;
  double* table;
};

// DepthImage (synth.py:69-114): values in fp64 and validity isfinite & > 0 (& mask)
__device__ __forceinline__ bool depth_at(const ChanParams& P, int y, int x, double& z) {
  bool valid;
  const int64_t off = (int64_t)y * P.row_pitch + x;
  if (P.dtype == RF_DEPTH_U16_MM) {
    const unsigned short mm = __ldg(reinterpret_cast<const unsigned short*>(P.depth) + off);
    valid = mm > 0;
    z = __ddiv_rn((double)mm, 1000.0);  // mm.astype(float64) / 1000.0
  } else if (P.dtype == RF_DEPTH_F64_M) {
    z = __ldg(reinterpret_cast<const double*>(P.depth) + off);
    valid = z > 0.0 && z <= 1.7976931348623157e308;
  } else {
    const float zf = __ldg(reinterpret_cast<const float*>(P.depth) + off);
    valid = (zf > 0.0f) && (zf <= 3.402823466e38f);
    z = (double)zf;
  }
  if (P.mask) valid = valid && __ldg(P.mask + (int64_t)y * P.W + x) != 0;
  return valid;
}

// one pixel of one channel (integral.py:188-325): lattices first, then
// build_integral's np.where(mask, channel, 0.0)
__device__ __forceinline__ double channel_value(const ChanParams& P, int y, int x) {
  if (P.channel < 0) {
    const double v = P.src[(int64_t)y * P.src_pitch + x];
    return (P.mask && P.mask[(int64_t)y * P.W + x] == 0) ? 0.0 : v;
  }
  const double tx = rf_tan(P.tan_x, P.lat_x, P.W, x, y, true), ty = rf_tan(P.tan_y, P.lat_y, P.W, x, y, false);
  switch (P.channel) {  // camera constants: not masked
    case RF_CH_ONES: return 1.0;
    case RF_CH_TX2: return tx * tx;
    case RF_CH_TXTY: return tx * ty;
    case RF_CH_TY2: return ty * ty;
    case RF_CH_TX: return tx;
    case RF_CH_TY: return ty;
    default: break;
  }
  double zr;
  const bool valid = depth_at(P, y, x, zr);
  if (!valid) return 0.0;
  const double z = zr;                     // _masked_depth: where(valid, values, 0)
  const double iz = 1.0 / z;               // _masked_inverse_depth: 1.0 / values (IEEE)
  const double X = z * tx, Y = z * ty;     // x = z * tan_x, y = z * tan_y
  switch (P.channel) {
    case RF_CH_COUNT: return 1.0;
    case RF_CH_X2: return X * X;
    case RF_CH_XY: return X * Y;
    case RF_CH_XZ: return X * z;
    case RF_CH_X: return X;
    case RF_CH_Y2: return Y * Y;
    case RF_CH_YZ: return Y * z;
    case RF_CH_Y: return Y;
    case RF_CH_Z2: return z * z;
    case RF_CH_Z: return z;
    case RF_CH_TX_OVER_Z: return tx * iz;
    case RF_CH_TY_OVER_Z: return ty * iz;
    case RF_CH_INV_Z: return iz;
    case RF_CH_INV_Z2: return iz * iz;
    case RF_CH_M_TX2: return tx * tx;
    case RF_CH_M_TXTY: return tx * ty;
    case RF_CH_M_TY2: return ty * ty;
    case RF_CH_M_TX: return tx;
    case RF_CH_M_TY: return ty;
    default: return 0.0;
  }
}

// np.cumsum(channel, axis=0) into table[1:, 1:]; zeroes row 0
__global__ void __launch_bounds__(SCAN_THREADS) column_scan_kernel(const ChanParams P) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t W1 = P.W + 1;
  if (x == 0) P.table[0] = 0.0;
  if (x >= P.W) return;
  P.table[x + 1] = 0.0;
  double acc = 0.0;
  for (int y = 0; y < P.H; ++y) {
    const double v = channel_value(P, y, x);
    acc = y == 0 ? v : acc + v;  // cumsum[0] = a[0], then sequential adds
    P.table[(int64_t)(y + 1) * W1 + x + 1] = acc;
  }
}

// np.cumsum(..., axis=1) in place on table[1:, 1:]; zeroes column 0.  One warp owns 32
// rows; each 32x32 chunk is transposed through shared memory so that lane l scans row l.
__global__ void __launch_bounds__(ROW_WARPS * 32) row_scan_kernel(double* table, int H, int W) {
  __shared__ double tile[ROW_WARPS][32][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = (blockIdx.x * ROW_WARPS + warp) * 32;
  if (r0 >= H) return;
  const int64_t W1 = W + 1;
  double (*t)[33] = tile[warp];
  if (r0 + lane < H) table[(int64_t)(r0 + lane + 1) * W1] = 0.0;
  double carry = 0.0;
  for (int c0 = 0; c0 < W; c0 += 32) {
    for (int j = 0; j < 32; ++j) {
      const int row = r0 + j;
      if (row < H && c0 + lane < W) t[j][lane] = table[(int64_t)(row + 1) * W1 + c0 + lane + 1];
    }
    __syncwarp();
    if (r0 + lane < H) {
      const int kmax = min(32, W - c0);
      for (int k = 0; k < kmax; ++k) {
        const double v = t[lane][k];
        carry = (c0 == 0 && k == 0) ? v : carry + v;
        t[lane][k] = carry;
      }
    }
    __syncwarp();
    for (int j = 0; j < 32; ++j) {
      const int row = r0 + j;
      if (row < H && c0 + lane < W) table[(int64_t)(row + 1) * W1 + c0 + lane + 1] = t[j][lane];
    }
    __syncwarp();
  }
}

struct BoxParams {
  const double* tables[RF_MAX_BOX_CHANNELS];
  int nch, H, W;
  const rf_rect* rects;
  int64_t nrects;
  double* out;
};

__global__ void box_sums_kernel(const BoxParams P) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.nrects * P.nch) return;
  const int64_t r = i / P.nch;
  const int c = (int)(i - r * P.nch);
  const rf_rect R = P.rects[r];
  if (!(0 <= R.x0 && R.x0 <= R.x1 && R.x1 <= P.W && 0 <= R.y0 && R.y0 <= R.y1 && R.y1 <= P.H)) {
    P.out[i] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  const double* t = P.tables[c];
  const int64_t W1 = P.W + 1;
  const double a = t[(int64_t)R.y1 * W1 + R.x1], b = t[(int64_t)R.y0 * W1 + R.x1];
  const double cc = t[(int64_t)R.y1 * W1 + R.x0], d = t[(int64_t)R.y0 * W1 + R.x0];
  P.out[i] = a - b - cc + d;  // evaluated left to right, as the reference
}

struct FitParams {
  const double* matrices;
  const double* rhs;
  const double* target_sq;
  const int64_t* counts;
  int64_t n;
  int formulation;
  rf_rect_fit* out;
};

// centred monomial scatter C and mean mu from an uncentred system: the Schur complement
// of the constant monomial k (entry ns > 0) over the monomials I
__device__ __forceinline__ void centre(const double (&S)[4][4], const int (&I)[3], int k, Sym3& C,
                                       double& m0, double& m1, double& m2) {
  const double ns = S[k][k];
  m0 = S[I[0]][k] / ns;
  m1 = S[I[1]][k] / ns;
  m2 = S[I[2]][k] / ns;
  C.c00 = fma(-S[I[0]][k], m0, S[I[0]][I[0]]);
  C.c01 = fma(-S[I[0]][k], m1, S[I[0]][I[1]]);
  C.c02 = fma(-S[I[0]][k], m2, S[I[0]][I[2]]);
  C.c11 = fma(-S[I[1]][k], m1, S[I[1]][I[1]]);
  C.c12 = fma(-S[I[1]][k], m2, S[I[1]][I[2]]);
  C.c22 = fma(-S[I[2]][k], m2, S[I[2]][I[2]]);
}

__global__ void fit_scatters_kernel(const FitParams P) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  rf_rect_fit res;
  for (int k = 0; k < 4; ++k) res.coef[k] = qnan;
  for (int k = 0; k < 3; ++k) res.explicit_coef[k] = qnan;
  res.eigenvalue = res.rms = res.curvature = qnan;
  const int64_t count = P.counts[i];
  res.n_points = (int32_t)count;
  res.status = 0;
  const bool space_std = P.formulation == RF_FORM_IMPLICIT_STANDARD || P.formulation == RF_FORM_EXPLICIT_STANDARD;
  const bool explicit_fit = P.formulation >= RF_FORM_EXPLICIT_STANDARD;
  // monomial order of the reference's matrices: standard [X, Y, Z, 1] (constant at 3),
  // rgbd [tx, ty, 1, 1/Z] (constant at 2)
  const int k = space_std ? 3 : 2;
  const int I[3] = {0, 1, space_std ? 2 : 3};
  const double* M = P.matrices + 16 * i;
  if (!explicit_fit) {
    if (count < 4) {  // _require_n(n, 4)
      P.out[i] = res;
      return;
    }
    double S[4][4];
    for (int r = 0; r < 4; ++r)
      for (int c = 0; c < 4; ++c) S[r][c] = M[4 * r + c];
    const double ns = S[k][k];
    bool solved = false;
    if (ns > 0.0 && isfinite(ns)) {
      Sym3 C;
      double m0, m1, m2;
      centre(S, I, k, C, m0, m1, m2);
      WindowFit f;
      solve_window(C, m0, m1, m2, ns, f);
      double v[4];
      if (space_std) canonical4(f.u0, f.u1, f.u2, f.s, v);
      else canonical4(f.u0, f.u1, f.s, f.u2, v);
      // Data scatters always pass; a hand-made system whose smallest eigenvector is the
      // constant monomial alone (mean 0, lam = n: no pencil solution) does not.
      double r2 = 0.0, s2 = 0.0;
      for (int a = 0; a < 4; ++a) {
        double ra = -f.lam * v[a];
        for (int b = 0; b < 4; ++b) ra = fma(S[a][b], v[b], ra);
        r2 += ra * ra;
        for (int b = 0; b < 4; ++b) s2 += S[a][b] * S[a][b];
      }
      if (isfinite(r2) && r2 <= 1e-16 * s2) {
        for (int a = 0; a < 4; ++a) res.coef[a] = v[a];
        res.eigenvalue = f.lam;
        res.curvature = f.kappa;
        res.status = RF_RECT_FIT | (f.degenerate ? RF_RECT_DEGENERATE : 0);
        solved = true;
      }
    }
    if (!solved) {
      // not a data scatter: the reference's Jacobi
      const double fro = frobenius(S);
      double V[4][4];
      if (!jacobi(S, V, fro)) {
        res.status = RF_RECT_JACOBI_FAILED;
        P.out[i] = res;
        return;
      }
      int lo = 0;
      for (int r = 1; r < 4; ++r)
        if (S[r][r] < S[lo][lo]) lo = r;
      double second = INFINITY;
      for (int r = 0; r < 4; ++r)
        if (r != lo && S[r][r] < second) second = S[r][r];
      const double lam = S[lo][lo];
      canonical4(V[0][lo], V[1][lo], V[2][lo], V[3][lo], res.coef);
      res.eigenvalue = lam;
      const bool deg = fro == 0.0 || second - lam <= 1e-9 * fro;
      res.status = RF_RECT_FIT | (deg ? RF_RECT_DEGENERATE : 0);
    }
    res.rms = sqrt(fmax(res.eigenvalue, 0.0) / (double)count);
    P.out[i] = res;
    return;
  }

  // explicit (fitting.py:582-621): Cholesky with the 1e-12 trace pivot floor, else the
  // minimum-norm solution
  if (count < 3) {
    P.out[i] = res;
    return;
  }
  double A[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) A[r][c] = M[4 * r + c];
  const double b0 = P.rhs[3 * i], b1 = P.rhs[3 * i + 1], b2 = P.rhs[3 * i + 2];
  // The reference evaluates this in Python floats (no fused multiply-add): the explicit
  // _rn intrinsics keep nvcc from contracting, so a well-posed system solves to the same bits.
  const double trace = __dadd_rn(__dadd_rn(A[0][0], A[1][1]), A[2][2]);
  const double floor = __dmul_rn(1e-12, trace);
  bool deg = !isfinite(trace) || trace <= 0.0;
  double l00 = 0, l10 = 0, l20 = 0, l11 = 0, l21 = 0, l22 = 0;
  if (!deg) {
    const double p0 = A[0][0];
    deg = p0 <= floor;
    if (!deg) {
      l00 = __dsqrt_rn(p0);
      l10 = __ddiv_rn(A[1][0], l00);
      l20 = __ddiv_rn(A[2][0], l00);
      const double p1 = __dsub_rn(A[1][1], __dmul_rn(l10, l10));
      deg = p1 <= floor;
      if (!deg) {
        l11 = __dsqrt_rn(p1);
        l21 = __ddiv_rn(__dsub_rn(A[2][1], __dmul_rn(l20, l10)), l11);
        const double p2 = __dsub_rn(__dsub_rn(A[2][2], __dmul_rn(l20, l20)), __dmul_rn(l21, l21));
        deg = p2 <= floor;
        if (!deg) l22 = __dsqrt_rn(p2);
      }
    }
  }
  double x0, x1, x2;
  if (!deg) {  // solve_cholesky3 (fitting.py:296-305)
    const double y0 = __ddiv_rn(b0, l00);
    const double y1 = __ddiv_rn(__dsub_rn(b1, __dmul_rn(l10, y0)), l11);
    const double y2 = __ddiv_rn(__dsub_rn(__dsub_rn(b2, __dmul_rn(l20, y0)), __dmul_rn(l21, y1)), l22);
    x2 = __ddiv_rn(y2, l22);
    x1 = __ddiv_rn(__dsub_rn(y1, __dmul_rn(l21, x2)), l11);
    x0 = __ddiv_rn(__dsub_rn(__dsub_rn(y0, __dmul_rn(l10, x1)), __dmul_rn(l20, x2)), l00);
  } else {  // _pinv_solve (fitting.py:313-327)
    double E[3][3], V[3][3];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) E[r][c] = A[r][c];
    if (!isfinite(trace) || !jacobi(E, V, frobenius(E))) {
      res.status = RF_RECT_JACOBI_FAILED;
      P.out[i] = res;
      return;
    }
    const double tol = __dmul_rn(1e-12, fmax(trace, 0.0));
    x0 = x1 = x2 = 0.0;
    for (int e = 0; e < 3; ++e) {
      const double lam = E[e][e];
      if (lam > tol) {
        const double dot = __dadd_rn(__dadd_rn(__dmul_rn(V[0][e], b0), __dmul_rn(V[1][e], b1)), __dmul_rn(V[2][e], b2));
        const double w = __ddiv_rn(dot, lam);
        x0 = __dadd_rn(x0, __dmul_rn(V[0][e], w));
        x1 = __dadd_rn(x1, __dmul_rn(V[1][e], w));
        x2 = __dadd_rn(x2, __dmul_rn(V[2][e], w));
      }
    }
  }
  res.explicit_coef[0] = x0;
  res.explicit_coef[1] = x1;
  res.explicit_coef[2] = x2;
  // explicit_to_implicit (fitting.py:729-739)
  if (space_std) canonical4(x0, x1, -1.0, x2, res.coef);
  else canonical4(x0, x1, x2, -1.0, res.coef);
  const double tq = P.target_sq ? P.target_sq[i] : qnan;
  if (isfinite(tq)) {
    res.rms = sqrt(fmax(tq - (x0 * b0 + x1 * b1 + x2 * b2), 0.0) / (double)count);
    // curvature of the full monomial scatter: standard [X, Y, Z, 1], rgbd [tx, ty, 1, 1/Z]
    double S[4][4];
    if (space_std) {
      const double v[4][4] = {{A[0][0], A[0][1], b0, A[0][2]},
                              {A[0][1], A[1][1], b1, A[1][2]},
                              {b0, b1, tq, b2},
                              {A[0][2], A[1][2], b2, A[2][2]}};
      for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) S[r][c] = v[r][c];
    } else {
      const double v[4][4] = {{A[0][0], A[0][1], A[0][2], b0},
                              {A[0][1], A[1][1], A[1][2], b1},
                              {A[0][2], A[1][2], A[2][2], b2},
                              {b0, b1, b2, tq}};
      for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) S[r][c] = v[r][c];
    }
    if (S[k][k] > 0.0) {
      Sym3 C;
      double m0, m1, m2;
      centre(S, I, k, C, m0, m1, m2);
      res.curvature = curvature_only(C);
    }
  }
  res.status = RF_RECT_FIT | (deg ? RF_RECT_DEGENERATE : 0);
  P.out[i] = res;
}

}  // namespace

extern "C" {

rf_status rf_build_channel(const rf_tables* t, const void* depth, int dtype, int64_t row_pitch,
                           const uint8_t* mask, int32_t channel, double* table, void* stream) {
  if (!t || !table) return rf_set_error(RF_ERR_ARGUMENT, "rf_build_channel: null tables or table");
  if (channel < 0 || channel >= RF_NUM_CHANNELS)
    return rf_set_error(RF_ERR_ARGUMENT, "rf_build_channel: unknown channel id");
  const bool constant = channel == RF_CH_ONES || (channel >= RF_CH_TX2 && channel <= RF_CH_TY);
  if (!constant) {
    if (!depth) return rf_set_error(RF_ERR_ARGUMENT, "rf_build_channel: null depth");
    if (dtype != RF_DEPTH_F32_M && dtype != RF_DEPTH_U16_MM && dtype != RF_DEPTH_F64_M)
      return rf_set_error(RF_ERR_SHAPE, "rf_build_channel: unknown depth dtype");
    if (row_pitch < t->intr.width) return rf_set_error(RF_ERR_SHAPE, "rf_build_channel: row_pitch < width");
  }
  const rf_device_guard guard(t->device);
  ChanParams P{};
  P.depth = depth;
  P.dtype = dtype;
  P.row_pitch = row_pitch;
  P.mask = mask;
  P.tan_x = t->tan_x;
  P.tan_y = t->tan_y;
  P.lat_x = t->lat_x;
  P.lat_y = t->lat_y;
  P.H = t->intr.height;
  P.W = t->intr.width;
  P.channel = channel;
  P.table = table;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  column_scan_kernel<<<(P.W + SCAN_THREADS - 1) / SCAN_THREADS, SCAN_THREADS, 0, s>>>(P);
  row_scan_kernel<<<(P.H + 32 * ROW_WARPS - 1) / (32 * ROW_WARPS), 32 * ROW_WARPS, 0, s>>>(table, P.H, P.W);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return rf_set_error(RF_ERR_CUDA, cudaGetErrorString(e));
  return RF_OK;
}

rf_status rf_integral(const double* src, int64_t src_pitch, const uint8_t* mask, int32_t H, int32_t W,
                      double* table, void* stream) {
  if (!src || !table) return rf_set_error(RF_ERR_ARGUMENT, "rf_integral: null pointer");
  if (H <= 0 || W <= 0 || src_pitch < W) return rf_set_error(RF_ERR_SHAPE, "rf_integral: bad shape");
  ChanParams P{};
  P.src = src;
  P.src_pitch = src_pitch;
  P.mask = mask;
  P.H = H;
  P.W = W;
  P.channel = -1;
  P.table = table;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  column_scan_kernel<<<(W + SCAN_THREADS - 1) / SCAN_THREADS, SCAN_THREADS, 0, s>>>(P);
  row_scan_kernel<<<(H + 32 * ROW_WARPS - 1) / (32 * ROW_WARPS), 32 * ROW_WARPS, 0, s>>>(table, H, W);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return rf_set_error(RF_ERR_CUDA, cudaGetErrorString(e));
  return RF_OK;
}

rf_status rf_box_sums(const double* const* tables, int32_t nch, int32_t H, int32_t W, const rf_rect* rects,
                      int64_t nrects, double* out, void* stream) {
  if (nrects < 0 || nch < 0) return rf_set_error(RF_ERR_ARGUMENT, "rf_box_sums: negative count");
  if (nrects == 0 || nch == 0) return RF_OK;
  if (!tables || !rects || !out) return rf_set_error(RF_ERR_ARGUMENT, "rf_box_sums: null pointer");
  if (nch > RF_MAX_BOX_CHANNELS) return rf_set_error(RF_ERR_ARGUMENT, "rf_box_sums: too many channels");
  if (H <= 0 || W <= 0) return rf_set_error(RF_ERR_SHAPE, "rf_box_sums: bad shape");
  BoxParams P{};
  for (int c = 0; c < nch; ++c) {
    if (!tables[c]) return rf_set_error(RF_ERR_ARGUMENT, "rf_box_sums: null table");
    P.tables[c] = tables[c];
  }
  P.nch = nch;
  P.H = H;
  P.W = W;
  P.rects = rects;
  P.nrects = nrects;
  P.out = out;
  const int64_t total = nrects * nch;
  box_sums_kernel<<<(unsigned)((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(P);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return rf_set_error(RF_ERR_CUDA, cudaGetErrorString(e));
  return RF_OK;
}

rf_status rf_fit_scatters(const double* matrices, const double* rhs, const double* target_sq,
                          const int64_t* counts, int64_t n, int32_t formulation, rf_rect_fit* out,
                          void* stream) {
  if (n < 0) return rf_set_error(RF_ERR_ARGUMENT, "rf_fit_scatters: negative count");
  if (formulation < 0 || formulation >= RF_NUM_FORMULATIONS)
    return rf_set_error(RF_ERR_ARGUMENT, "rf_fit_scatters: unknown formulation");
  if (n == 0) return RF_OK;
  if (!matrices || !counts || !out) return rf_set_error(RF_ERR_ARGUMENT, "rf_fit_scatters: null pointer");
  if (formulation >= RF_FORM_EXPLICIT_STANDARD && !rhs)
    return rf_set_error(RF_ERR_ARGUMENT, "rf_fit_scatters: explicit systems need a right-hand side");
  FitParams P{matrices, rhs, target_sq, counts, n, formulation, out};
  fit_scatters_kernel<<<(unsigned)((n + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(P);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return rf_set_error(RF_ERR_CUDA, cudaGetErrorString(e));
  return RF_OK;
}

}  // extern "C"
