// rf_tile.cuh -- definitions shared by the per-pixel fit kernels (rf_fit.cu: separable tan
// maps; rf_lattice.cu: distortion lattices): tile geometry, kernel parameters, output planes.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rangefit_b200.h"

namespace rf_tile {

constexpr int TW = 64;       // output tile width  (pixels)
#ifndef RF_TH
#define RF_TH 16
#endif
constexpr int TH = RF_TH;    // output tile height (pixels)
constexpr int KSEG = 4;      // consecutive output pixels per thread
constexpr int NTHREADS = (TW / KSEG) * TH;  // 256
constexpr int MAX_RADIUS = 32;
#ifndef RF_ABLATE
#define RF_ABLATE 0
#endif
#ifndef RF_ROW_UNROLL
#define RF_ROW_UNROLL 1
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
  double ifx2, ify2, ifxy;  // ifx^2, ify^2, ifx ify (host-computed, IEEE identical)
  int64_t row_pitch;
  int64_t frame_stride;
  int64_t out_frame;    // H*W
  int64_t batch;
  int H, W, r, dtype;
  int do_imp, do_exp;  // implicit / explicit fit of this kernel's space requested
  OutPlanes imp, exp;  // implicit-* / explicit-* output planes of the space
  // programmatic dependent launch of the next kernel in the stream: 0 at exit, 1 at entry (the
  // first space's launch of a two-launch call: the second space shares nothing with it)
  int pdl_trigger;
};

// bytes per depth element
__host__ __device__ __forceinline__ int elem_size(int dtype) {
  return dtype == RF_DEPTH_U16_MM ? 2 : dtype == RF_DEPTH_F64_M ? 8 : 4;
}

// residue-major column stride of the column-sum buffers (VQ = 4 mod 8 spreads the banks)
__host__ __device__ __forceinline__ int vq_of(int hw) {
  int q = (hw + 3) / 4;
  return q + ((4 - q % 8) + 8) % 8;
}

struct TileGeom {
  int64_t frame;
  int x0, y0;
};

__device__ __forceinline__ TileGeom tile_of(int64_t t, int ntx, int nty) {
  TileGeom g;
  const int64_t per_frame = (int64_t)ntx * nty;
  int rem;
  if ((uint64_t)t <= 0xffffffffull && per_frame <= 0xffffffffll) {
    // every BASELINE batch (C4: 2.1 M tiles): 32-bit division, not the 64-bit routine that
    // all threads would otherwise run once per tile
    const unsigned tt = (unsigned)t, pf = (unsigned)per_frame;
    const unsigned f = tt / pf;
    g.frame = f;
    rem = (int)(tt - f * pf);
  } else {
    g.frame = t / per_frame;
    rem = (int)(t - g.frame * per_frame);
  }
  const int ty = (int)((unsigned)rem / (unsigned)ntx);
  g.y0 = ty * TH;
  g.x0 = (rem - ty * ntx) * TW;
  return g;
}

// The tiles a persistent CTA visits, t = t0, t0 + step, ...: the (frame, tile row, tile
// column) decomposition is advanced by the step's own decomposition with one carry per
// digit, so no division runs per tile (two divisions once per CTA)
struct TileIter {
  int64_t frame, dframe;
  int tx, ty, dtx, dty, ntx, nty;
  __device__ __forceinline__ TileIter(int64_t t0, int64_t step, int ntx_, int nty_) : ntx(ntx_), nty(nty_) {
    const TileGeom a = tile_of(t0, ntx, nty), d = tile_of(step, ntx, nty);
    frame = a.frame, ty = a.y0 / TH, tx = a.x0 / TW;
    dframe = d.frame, dty = d.y0 / TH, dtx = d.x0 / TW;
  }
  __device__ __forceinline__ TileGeom geom() const { return TileGeom{frame, tx * TW, ty * TH}; }
  __device__ __forceinline__ void advance() {
    tx += dtx;
    int cy = dty;
    if (tx >= ntx) tx -= ntx, ++cy;
    ty += cy;
    int64_t cf = dframe;
    if (ty >= nty) ty -= nty, ++cf;
    frame += cf;
  }
};

// launch the per-pixel fits of one space on cameras with distortion lattices (rf_lattice.cu)
cudaError_t launch_lattice(int var, const KParams& P, const double* lat_x, const double* lat_y,
                           cudaStream_t s);

}  // namespace rf_tile
