// rf_lattice.cu -- per-pixel fits for cameras with distortion lattices (CameraIntrinsics
// delta_x / delta_y, camera.py:35-75): the tan maps are not separable, so the separable tile
// kernels' exact-integer geometry (rf_fit.cu) does not apply.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/rangefit_b200.h"
#include "rf_internal.h"
#include "rf_tile.cuh"
#include "rf_solve.cuh"
#include "rf_jacobi.cuh"
#include "rf_general.cuh"
#include "rf_direct.cuh"

namespace {
using namespace rf_dev;
using namespace rf_tile;

// ------------------------------------------------------------------ distortion lattices
// Cameras with non-zero delta_* lattices (camera.py:35-75): the tan maps are not separable,
// so the tile kernels' exact-integer geometry does not apply.  Direct fallback: one thread
// per output pixel sums its clipped window directly (rf_direct.cuh).
template <int VAR, bool EXP>
__global__ void __launch_bounds__(128) fit_lattice_kernel(const KParams P, const double* lat_x,
                                                          const double* lat_y) {
  const int64_t total = P.batch * P.out_frame;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < total;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t frame = p / P.out_frame;
    const int rem = (int)(p - frame * P.out_frame);
    const int y = rem / P.W;
    fit_pixel_direct<VAR, EXP>(P, lat_x, lat_y, frame, y, rem - y * P.W);
  }
}

// Tiled variant (the default for distortion lattices): the same 64x16 persistent tiles and
// sliding window sums as the separable kernels, over the nine q-moments of rf_general.cuh
// about the tile's first pixel (plain sums: the tan offsets are inside q).  The column pass
// reads depth and lattices straight from global memory (L1/L2-resident; converted twice per
// element, once entering and once leaving the window), so shared memory holds only the
// column sums and two CTAs fit per SM for radii up to 7.
constexpr int NQ = 9;  // q0, q1, q2, q0q0, q0q1, q0q2, q1q1, q1q2, q2q2

size_t lattice_smem_bytes(int r) {
  const size_t vrs = 4 * (size_t)vq_of(TW + 2 * r);
  return sizeof(double) * NQ * TH * vrs + sizeof(int) * TH * vrs + 16;
}

template <int VAR, bool EXP>
__global__ void __launch_bounds__(NTHREADS, 2) fit_lattice_tile_kernel(const KParams P, const double* lat_x,
                                                                       const double* lat_y) {
  extern __shared__ __align__(16) unsigned char smem_l[];
  const int r = P.r;
  const int HW_ = TW + 2 * r;
  const int VQ = vq_of(HW_), VRS = 4 * VQ;
  double* vd = reinterpret_cast<double*>(smem_l);          // [NQ][TH][VRS]
  int* vc = reinterpret_cast<int*>(vd + NQ * TH * VRS);    // [TH][VRS] valid counts
  const bool std_space = VAR == VAR_STD;
  const int tid = threadIdx.x;
  const int ntx = (P.W + TW - 1) / TW, nty = (P.H + TH - 1) / TH;
  const int64_t total = (int64_t)ntx * nty * P.batch;
  // high word of the largest |q_i| that has left the tile's column sums, double-buffered by
  // tile parity (the sliding-sum guard, fit_tile_kernel)
  __shared__ unsigned s_dmax[2];
  if (tid == 0) s_dmax[0] = s_dmax[1] = 0u;
  __syncthreads();
  int it = 0;
  for (int64_t t = blockIdx.x; t < total; t += gridDim.x, ++it) {
    const TileGeom g = tile_of(t, ntx, nty);
    const int64_t frame = g.frame;
    const int x0 = g.x0, y0 = g.y0;
    const double txr = __ldg(lat_x + (int64_t)y0 * P.W + x0), tyr = __ldg(lat_y + (int64_t)y0 * P.W + x0);
    // q of image pixel (y, x); false when outside the frame or invalid
    auto qof = [&](int y, int x, double& q0, double& q1, double& q2) -> bool {
      if (y < 0 || y >= P.H || x < 0 || x >= P.W) return false;
      const int64_t off = frame * P.frame_stride + (int64_t)y * P.row_pitch + x;
      double z;
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
      if (P.mask) valid = valid && __ldg(P.mask + frame * P.out_frame + (int64_t)y * P.W + x) != 0;
      if (!valid) return false;
      const int64_t li = (int64_t)y * P.W + x;
      const double dtx = __ldg(lat_x + li) - txr, dty = __ldg(lat_y + li) - tyr;
      q0 = std_space ? z * dtx : dtx;
      q1 = std_space ? z * dty : dty;
      q2 = std_space ? z : 1.0 / z;
      return true;
    };

    // ---- column sums (running, over row segments; all threads busy)
    const int parts = max(1, min(NTHREADS / HW_, TH));
    int dm = 0;
    {
      const int col = tid % HW_, part = tid / HW_;
      if (part < parts) {
        const int o0 = (part * TH) / parts, o1 = ((part + 1) * TH) / parts;
        const int x = x0 - r + col;
        double a[NQ];
        int cnt = 0;
#pragma unroll
        for (int k = 0; k < NQ; ++k) a[k] = 0.0;
        auto add = [&](int ii, double sg) {  // halo row ii = image row y0 - r + ii
          double q0, q1, q2;
          if (!qof(y0 - r + ii, x, q0, q1, q2)) return;
          const double s0 = sg * q0, s1 = sg * q1, s2 = sg * q2;
          if (sg < 0.0)
            dm = max(dm, max(__double2hiint(q0) & 0x7fffffff,
                             max(__double2hiint(q1) & 0x7fffffff, __double2hiint(q2) & 0x7fffffff)));
          a[0] += s0;
          a[1] += s1;
          a[2] += s2;
          a[3] = fma(s0, q0, a[3]);
          a[4] = fma(s0, q1, a[4]);
          a[5] = fma(s0, q2, a[5]);
          a[6] = fma(s1, q1, a[6]);
          a[7] = fma(s1, q2, a[7]);
          a[8] = fma(s2, q2, a[8]);
          cnt += sg > 0.0 ? 1 : -1;
        };
        for (int ii = o0; ii < o0 + 2 * r; ++ii) add(ii, 1.0);
        const int cpos = (col & 3) * VQ + (col >> 2);
        for (int o = o0; o < o1; ++o) {
          add(o + 2 * r, 1.0);
#pragma unroll
          for (int k = 0; k < NQ; ++k) vd[(k * TH + o) * VRS + cpos] = a[k];
          vc[o * VRS + cpos] = cnt;
          add(o, -1.0);
        }
      }
    }
    {
      const unsigned b = __reduce_max_sync(0xffffffffu, (unsigned)dm);  // dm >= 0
      if ((tid & 31) == 0) atomicMax(&s_dmax[it & 1], b);
    }
    __syncthreads();

    // ---- row sums + per-pixel solve (4 consecutive pixels per thread)
    {
      const int orow = tid / (TW / KSEG);
      const int xs = (tid % (TW / KSEG)) * KSEG;
      const int gy = y0 + orow, gxs = x0 + xs;
      if (gy < P.H && gxs < P.W) {
        const double* vrow = vd + orow * VRS;
        const int* crow = vc + orow * VRS;
        const int vstride = TH * VRS;
        const int vbase = xs >> 2;
        double h[NQ];
        int hc = 0;
#pragma unroll
        for (int k = 0; k < NQ; ++k) h[k] = 0.0;
        auto accum = [&](int k, double sg) {
          const int c = vbase + (k & 3) * VQ + (k >> 2);
#pragma unroll
          for (int m = 0; m < NQ; ++m) h[m] = fma(sg, vrow[m * vstride + c], h[m]);
          hc += sg > 0.0 ? crow[c] : -crow[c];
        };
        for (int k = 0; k <= 2 * r; ++k) accum(k, 1.0);
        const float qn = __int_as_float(0x7fc00000);
        if (tid == 0) s_dmax[(it + 1) & 1] = 0u;  // read by the previous tile, written by the next
        for (int j = 0; j < KSEG; ++j) {
          if (j > 0) {
            accum(j + 2 * r, 1.0);
            accum(j - 1, -1.0);
          }
          const int gx = gxs + j;
          if (gx >= P.W) break;
          double c0, c1, c2;
          const uint8_t vbit = qof(gy, gx, c0, c1, c2) ? RF_PIX_INPUT_VALID : 0;
          uint8_t st = vbit, stx = vbit;
          float nx = qn, ny = qn, nz = qn, off = qn, res = qn, cur = qn;
          float ex = qn, ey = qn, ez = qn, eo = qn, eres = qn, ecur = qn;
          if (vbit && hc >= (EXP ? 3 : 4)) {
            QMoments m;
            m.n = (double)hc;
            m.s0 = h[0]; m.s1 = h[1]; m.s2 = h[2];
            m.s00 = h[3]; m.s01 = h[4]; m.s02 = h[5]; m.s11 = h[6]; m.s12 = h[7]; m.s22 = h[8];
            Sym3 C;
            double mu0, mu1, mu2;
            q_to_scatter(std_space, m, txr, tyr, C, mu0, mu1, mu2);
            const double nd = m.n;
            float kap = 0.0f;
            if (P.do_imp && hc >= 4) {
              WindowFit f;
              solve_window(C, mu0, mu1, mu2, nd, f);
              if (std_space) finish_plane(f.u0, f.u1, f.u2, f.s, nx, ny, nz, off);
              else finish_plane(f.u0, f.u1, f.s, f.u2, nx, ny, nz, off);
              res = fsqrt(fmaxf((float)(f.lam / nd), 0.0f));
              cur = kap = f.kappa;
              st |= RF_PIX_FIT | (f.degenerate ? RF_PIX_DEGENERATE : 0);
            }
            if (EXP && P.do_exp) {
              if (!(P.do_imp && hc >= 4)) kap = curvature_only(C);
              ExplicitFit e;
              explicit_fit_robust(C, mu0, mu1, mu2, nd, e);
              if (std_space) finish_plane(e.a, e.b, -1.0, e.c, ex, ey, ez, eo);
              else finish_plane(e.a, e.b, e.c, -1.0, ex, ey, ez, eo);
              eres = fsqrt(fmaxf((float)(e.ss / nd), 0.0f));
              ecur = kap;
              stx |= RF_PIX_FIT | (e.degenerate ? RF_PIX_DEGENERATE : 0);
            }
          }
          const int64_t p = frame * P.out_frame + (int64_t)gy * P.W + gx;
          if (P.do_imp) store_fit(P.imp, p, nx, ny, nz, off, res, cur, st);
          if (EXP && P.do_exp) store_fit(P.exp, p, ex, ey, ez, eo, eres, ecur, stx);
        }
        {
          // sliding-sum guard (fit_tile_kernel, rf_fit.cu): departed mass of the segment's
          // window sums -- 3 leading columns' sums of q_i^2 and the (o - o0) x (2r + 4)
          // samples that left the column sums (each <= 3 x the tile's largest departed |q_i|^2) --
          // against each window's centre-column sums, in exponent steps on high words
          auto colq = [&](int c) {  // largest high word of the column's sums of q0^2, q1^2, q2^2
            const int cp = (c & 3) * VQ + (c >> 2);
            const int* w = reinterpret_cast<const int*>(vrow + cp);
            return max(w[2 * 3 * vstride + 1], max(w[2 * 6 * vstride + 1], w[2 * 8 * vstride + 1]));
          };
          int te = (max(colq(xs), max(colq(xs + 1), colq(xs + 2))) >> 20) - 1023 + 4;  // x 9
          const int seg = ((orow + 1) * parts + TH - 1) / TH - 1;
          const int rows = (orow - (seg * TH) / parts) * (2 * r + KSEG);
          if (rows > 0) te = max(te, 2 * ((int)(s_dmax[it & 1] >> 20) - 1023) + 2 + 32 - __clz(rows)) + 1;
          te -= 20;  // / 2^20
          const int thr = te < -1022 ? 0 : te > 1023 ? 0x7ff00000 : (te + 1023) << 20;
          int wmin = 0x7fffffff;
          for (int j = 0; j < KSEG; ++j) {
            const int c = xs + j + r;
            wmin = min(wmin, crow[(c & 3) * VQ + (c >> 2)] > 0 ? colq(c) : 0x7fffffff);  // exact count
          }
          // rare (never on realistic scenes): refit the segment from direct window sums here
          if (wmin < thr)
            for (int j = 0; j < KSEG && gxs + j < P.W; ++j) fit_pixel_direct<VAR, EXP>(P, lat_x, lat_y, frame, gy, gxs + j);
        }
      }
    }
    __syncthreads();  // vd / vc are rewritten by the next tile
  }
}

template <int VAR>
cudaError_t launch_lattice_var(const KParams& P, const double* lat_x, const double* lat_y, cudaStream_t s) {
  int dev = 0, sms = 148, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t sm = lattice_smem_bytes(P.r);
  if (getenv("RF_LATTICE_DIRECT") == nullptr && sm <= (size_t)optin) {
    auto kern = P.do_exp ? fit_lattice_tile_kernel<VAR, true> : fit_lattice_tile_kernel<VAR, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTHREADS, sm);
    if (per_sm < 1) per_sm = 1;
    const int64_t tiles = (int64_t)((P.W + TW - 1) / TW) * ((P.H + TH - 1) / TH) * P.batch;
    const int64_t grid = tiles < (int64_t)sms * per_sm ? tiles : (int64_t)sms * per_sm;
    kern<<<(unsigned)grid, NTHREADS, sm, s>>>(P, lat_x, lat_y);
    return cudaGetLastError();
  }
  const int64_t total = P.batch * P.out_frame;
  const int64_t want = (total + 127) / 128;
  const int64_t grid = want < (int64_t)sms * 16 ? want : (int64_t)sms * 16;
  if (P.do_exp) fit_lattice_kernel<VAR, true><<<(unsigned)grid, 128, 0, s>>>(P, lat_x, lat_y);
  else fit_lattice_kernel<VAR, false><<<(unsigned)grid, 128, 0, s>>>(P, lat_x, lat_y);
  return cudaGetLastError();
}

}  // namespace

namespace rf_tile {
cudaError_t launch_lattice(int var, const KParams& P, const double* lat_x, const double* lat_y,
                           cudaStream_t s) {
  return var == VAR_STD ? launch_lattice_var<VAR_STD>(P, lat_x, lat_y, s)
                        : launch_lattice_var<VAR_DF>(P, lat_x, lat_y, s);
}
}  // namespace rf_tile
