// rf_fit.cu -- C ABI (host side) for the per-pixel windowed implicit
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
#include <stdarg.h>

#include <mutex>
#include <type_traits>

#include "../../include/rangefit_b200.h"
#include "rf_internal.h"

#include "rf_tile.cuh"
#include "rf_solve.cuh"
#include "rf_invn.cuh"
#include "rf_jacobi.cuh"
#include "rf_general.cuh"
#include "rf_direct.cuh"

#include "rf_tile_kernel.cuh"

namespace rf_fitk {
// the kernel translation units (rf_fit_k1/k2/k3.cu)
cudaError_t launch_radius_sp1(const KParams& Ps, const KParams& Pd, const CUtensorMap& tmap, bool tma, size_t sm,
                              int64_t tiles, int sms, cudaStream_t s, bool pdl, bool three);
cudaError_t launch_radius_sp2(const KParams& Ps, const KParams& Pd, const CUtensorMap& tmap, bool tma, size_t sm,
                              int64_t tiles, int sms, cudaStream_t s, bool pdl, bool three);
cudaError_t launch_radius_sp3(const KParams& Ps, const KParams& Pd, const CUtensorMap& tmap, bool tma, size_t sm,
                              int64_t tiles, int sms, cudaStream_t s, bool pdl, bool three);
#ifdef RF_COUNT_SLOW
int read_slow_counts_sp1(unsigned long long* out, int reset);
int read_slow_counts_sp2(unsigned long long* out, int reset);
int read_slow_counts_sp3(unsigned long long* out, int reset);
#endif
}  // namespace rf_fitk

namespace {
using namespace rf_dev;
using namespace rf_tile;
using namespace rf_fitk;

// ------------------------------------------------------------------ tables
__global__ void tan_table_kernel(double* tx, double* ty, int W, int H, double fx, double fy,
                                 double cx, double cy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  // compute_tan_maps (camera.py:131-134) with delta = 0: ((col + 0.0) - cx) / fx
  if (i < W) tx[i] = __ddiv_rn(((double)i + 0.0) - cx, fx);
  if (i < H) ty[i] = __ddiv_rn(((double)i + 0.0) - cy, fy);
}

thread_local char g_err[512] = "";

__attribute__((format(printf, 2, 3))) rf_status fail(rf_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

// dynamic shared memory of fit_tile_kernel<SP, tma, r> (the kernel's own layout)
bool compiled_radius(int r) { return r == 1 || r == 2 || r == 3 || r == 4 || r == 5 || r == 7 || r == 15; }
size_t smem_bytes(int sp, int r, bool tma, int esz, bool exp = false, int minb = RF_MIN_BLOCKS) {
  // r = 15 with the standard space and a non-float32 input runs the generic-radius kernel
  const bool generic15 = r == 15 && (sp & 1) && esz != 4;
  const int hw = TW + 2 * r, hh = TH + 2 * r, hwp = (hw + 16 / esz - 1 + 7) & ~7;
  const int nvd = (sp & 1) ? 5 : 3;
  const int nsp = (sp & 1) + ((sp >> 1) & 1);
  const bool rt = tma && compiled_radius(r) && !generic15;  // the kernel's RT > 0
  const bool noprim = rt && noprim_radius(r);          // the kernel's ZF (RT == r): float Z tile
  const int psp = nsp - ((sp & 1) && noprim ? 1 : 0);  // spaces with an fp64 tile
  const bool dbuf = rt && r <= 3 && sp != 3 && (minb < 3 || TH <= 8);  // the kernel's DBUF
  const size_t raw = tma ? (((size_t)hh * hwp * esz + 127) & ~(size_t)127) : 0;
  const size_t vrs = 4 * (size_t)(noprim ? (hw + 3) / 4 : vq_of(hw));
  const size_t counts = ((rt ? sizeof(int) : sizeof(int2)) * (size_t)TH * vrs + 7) & ~(size_t)7;
  return raw + ((sp & 1) && noprim ? (((size_t)hh * hw + 1) / 2) * sizeof(double) : 0) +
         sizeof(double) * ((dbuf ? 2 : 1) * (size_t)psp * hh * hw + (size_t)nvd * TH * vrs) + counts +
         2 * sizeof(uint64_t) + 128 /* base align */ + (exp ? (size_t)28 * sizeof(float) * NTHREADS : 0);
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
  const int esz = elem_size(dtype);
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
  const CUtensorMapDataType dt = esz == 2   ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                 : esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                            : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const CUresult res = fn(m, dt, 3,
                          const_cast<void*>(depth), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS;
}

// per-device attributes, queried once
struct DeviceInfo {
  int sms = 0, smem_optin = 0, smem_sm = 0;
};
DeviceInfo g_dev_info[64];
std::mutex g_dev_mu;
DeviceInfo device_info(int dev) {
  DeviceInfo d;
  if (dev >= 0 && dev < 64) {
    std::lock_guard<std::mutex> lock(g_dev_mu);
    if (g_dev_info[dev].sms == 0) {
      cudaDeviceGetAttribute(&g_dev_info[dev].sms, cudaDevAttrMultiProcessorCount, dev);
      cudaDeviceGetAttribute(&g_dev_info[dev].smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      cudaDeviceGetAttribute(&g_dev_info[dev].smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    }
    d = g_dev_info[dev];
  } else {
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&d.smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  }
  return d;
}

// How rf_fit_pixels launches (both rf_fit_pixels and rf_launches_per_call use it).
struct LaunchPlan {
  bool fused;  // both spaces in one SP = 3 launch
  bool three;  // one launch per space at three CTAs per SM (small radii, one wave of tiles)
};
LaunchPlan plan_launches(int sp_all, int r, bool tma, int esz, bool want_exp, int64_t tiles, const DeviceInfo& di) {
  LaunchPlan lp{false, false};
  if (sp_all != 3) return lp;
  lp.three = tma && r >= 1 && r <= 3 && !want_exp && tiles <= (int64_t)3 * di.sms &&
             3 * (smem_bytes(1, r, true, esz, false, 3) + 1024) <= (size_t)di.smem_sm && getenv("RF_NO_THREE") == nullptr;
  // Both spaces in one launch (one read and conversion of the input, one launch) for small
  // batches -- at most four waves of tiles, where the launch count and tail waves dominate --
  // when two such CTAs still fit per SM.  Large batches run one launch per space (disparity
  // form first): measured on C2 (64 frames, w5) the fused kernel's doubled instruction
  // footprint costs more in instruction-fetch stalls (11.6% vs 3.5% of warp samples) than the
  // shared halo saves (1.20-1.23 vs 1.15 ms per step).
  lp.fused = !lp.three && 2 * (smem_bytes(3, r, tma, esz, want_exp) + 1024) <= (size_t)di.smem_sm &&
             (tiles <= (int64_t)4 * 2 * di.sms || getenv("RF_FUSE") != nullptr) && getenv("RF_NO_FUSE") == nullptr;
  return lp;
}

}  // namespace

rf_status rf_set_error(rf_status s, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return s;
}

extern "C" {

int32_t rf_abi_version(void) { return RF_ABI_VERSION; }

#ifdef RF_COUNT_SLOW
// experiment builds only: windows per space (0 standard, 1 rgbd) that left the fast solve
int32_t rf_debug_slow_counts(unsigned long long* out, int reset) {
  for (int i = 0; i < 256; ++i) out[i] = 0;
  return read_slow_counts_sp1(out, reset) | read_slow_counts_sp2(out, reset) | read_slow_counts_sp3(out, reset);
}
#endif

const char* rf_last_error(void) { return g_err; }

int32_t rf_launches_per_call(int32_t formulation_mask, int32_t window, int32_t dtype, int64_t batch,
                             int32_t height, int32_t width) {
  // rf_fit_pixels' launch plan for separable tables on the current device (TMA path)
  const bool want_std = (formulation_mask & (RF_IMPLICIT_STANDARD | RF_EXPLICIT_STANDARD)) != 0;
  const bool want_df = (formulation_mask & (RF_IMPLICIT_RGBD | RF_EXPLICIT_RGBD)) != 0;
  if (!(want_std && want_df)) return (want_std || want_df) ? 1 : 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const DeviceInfo di = device_info(dev);
  const bool want_exp = (formulation_mask & (RF_EXPLICIT_STANDARD | RF_EXPLICIT_RGBD)) != 0;
  const int64_t tiles = (int64_t)((width + TW - 1) / TW) * ((height + TH - 1) / TH) * batch;
  return plan_launches(3, window / 2, true, elem_size(dtype), want_exp, tiles, di).fused ? 1 : 2;
}

rf_status rf_tables_create(const rf_intrinsics* in, const double* delta_x, const double* delta_y,
                           int device, rf_tables** out) {
  if (!in || !out) return fail(RF_ERR_ARGUMENT, "rf_tables_create: null argument");
  *out = nullptr;
  // CameraIntrinsics.__post_init__ (camera.py:54-63)
  if (!(in->fx > 0) || !(in->fy > 0))
    return fail(RF_ERR_ARGUMENT, "focal lengths must be positive");
  if (in->width <= 0 || in->height <= 0) return fail(RF_ERR_ARGUMENT, "image size must be positive");
  if (!(in->cx >= 0 && in->cx < in->width && in->cy >= 0 && in->cy < in->height))
    return fail(RF_ERR_ARGUMENT, "principal point outside the image");
  const int64_t n = (int64_t)in->width * in->height;
  bool separable = true;
  for (int64_t i = 0; delta_x && i < n && separable; ++i) separable = delta_x[i] == 0.0;
  for (int64_t i = 0; delta_y && i < n && separable; ++i) separable = delta_y[i] == 0.0;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(RF_ERR_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
  rf_tables* t = new rf_tables();
  t->intr = *in;
  t->device = device;
  if (!separable) {
    // compute_tan_maps (camera.py:131-134): ((x + delta_x) - cx) / fx, evaluated on the host
    // in the reference's operation order (plain IEEE double), then kept on the device
    double* hx = new double[n];
    double* hy = new double[n];
    for (int y = 0; y < in->height; ++y)
      for (int x = 0; x < in->width; ++x) {
        const int64_t i = (int64_t)y * in->width + x;
        hx[i] = (((double)x + (delta_x ? delta_x[i] : 0.0)) - in->cx) / in->fx;
        hy[i] = (((double)y + (delta_y ? delta_y[i] : 0.0)) - in->cy) / in->fy;
      }
    e = cudaMalloc(&t->lat_x, sizeof(double) * n);
    if (e == cudaSuccess) e = cudaMalloc(&t->lat_y, sizeof(double) * n);
    if (e == cudaSuccess) e = cudaMemcpy(t->lat_x, hx, sizeof(double) * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(t->lat_y, hy, sizeof(double) * n, cudaMemcpyHostToDevice);
    delete[] hx;
    delete[] hy;
    if (e != cudaSuccess) {
      cudaFree(t->lat_x);
      cudaFree(t->lat_y);
      cudaSetDevice(prev);
      delete t;
      return fail(RF_ERR_CUDA, "rf_tables_create: %s", cudaGetErrorString(e));
    }
  }
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
    cudaFree(t->lat_x);
    cudaFree(t->lat_y);
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
  cudaFree(t->lat_x);
  cudaFree(t->lat_y);
  delete t;
  return RF_OK;
}

rf_status rf_fit_pixels(const rf_tables* t, const void* depth, int dtype, int64_t batch,
                        int32_t H, int32_t W, int64_t row_pitch, const uint8_t* mask,
                        int32_t window, int32_t fmask, const rf_pixel_out* outs, void* stream) {
  if (!t) return fail(RF_ERR_ARGUMENT, "rf_fit_pixels: null tables");
  if (!depth && batch != 0) return fail(RF_ERR_ARGUMENT, "rf_fit_pixels: null depth");
  if (dtype != RF_DEPTH_F32_M && dtype != RF_DEPTH_U16_MM && dtype != RF_DEPTH_F64_M)
    return fail(RF_ERR_SHAPE, "unknown depth dtype %d", dtype);
  if (H != t->intr.height || W != t->intr.width)
    return fail(RF_ERR_SHAPE, "depth %dx%d does not match the camera tables", W, H);
  if (batch < 0) return fail(RF_ERR_ARGUMENT, "batch %lld is negative", (long long)batch);
  if (row_pitch < W) return fail(RF_ERR_ARGUMENT, "row_pitch %lld < width", (long long)row_pitch);
  if (window < 1 || (window & 1) == 0 || window / 2 > MAX_RADIUS)
    return fail(RF_ERR_ARGUMENT, "window must be odd and in [1, %d], got %d", 2 * MAX_RADIUS + 1, window);
  if ((fmask & ~RF_ALL_FORMULATIONS) != 0 || fmask == 0)
    return fail(RF_ERR_ARGUMENT, "formulation_mask %d invalid", fmask);
  if (batch == 0) return RF_OK;
  if (!outs) return fail(RF_ERR_ARGUMENT, "rf_fit_pixels: null output array");
  for (int f = 0; f < RF_NUM_FORMULATIONS; ++f) {
    if (!(fmask & (1 << f))) continue;
    const rf_pixel_out& o = outs[f];
    if (!o.normal || !o.offset || !o.residual || !o.curvature || !o.status)
      return fail(RF_ERR_ARGUMENT, "formulation %d requested without output buffers", f);
  }
  const rf_device_guard guard(t->device);
  const int r = window / 2;
  const int64_t tiles = (int64_t)((W + TW - 1) / TW) * ((H + TH - 1) / TH) * batch;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const DeviceInfo di = device_info(t->device);
  const int esz = elem_size(dtype);
  const bool want_std = (fmask & (RF_IMPLICIT_STANDARD | RF_EXPLICIT_STANDARD)) != 0;
  const bool want_df = (fmask & (RF_IMPLICIT_RGBD | RF_EXPLICIT_RGBD)) != 0;
  // the two spaces' parameters: same input and geometry, their own outputs
  KParams Pv[2];
  for (int var = 0; var < 2; ++var) {
    const int fi = var == VAR_STD ? RF_FORM_IMPLICIT_STANDARD : RF_FORM_IMPLICIT_RGBD;
    const int fe = var == VAR_STD ? RF_FORM_EXPLICIT_STANDARD : RF_FORM_EXPLICIT_RGBD;
    KParams& P = Pv[var];
    memset(&P, 0, sizeof(P));
    P.depth = depth;
    P.mask = mask;
    P.tan_x = t->tan_x;
    P.tan_y = t->tan_y;
    P.ifx = 1.0 / t->intr.fx;
    P.ify = 1.0 / t->intr.fy;
    P.ifx2 = P.ifx * P.ifx;
    P.ify2 = P.ify * P.ify;
    P.ifxy = P.ifx * P.ify;
    P.row_pitch = row_pitch;
    P.frame_stride = row_pitch * H;
    P.out_frame = (int64_t)H * W;
    P.H = H;
    P.W = W;
    P.r = r;
    P.dtype = dtype;
    P.batch = batch;
    P.do_imp = (fmask >> fi) & 1;
    P.do_exp = (fmask >> fe) & 1;
    if (P.do_imp) P.imp = OutPlanes{outs[fi].normal, outs[fi].offset, outs[fi].residual, outs[fi].curvature, outs[fi].status};
    if (P.do_exp) P.exp = OutPlanes{outs[fe].normal, outs[fe].offset, outs[fe].residual, outs[fe].curvature, outs[fe].status};
  }
  cudaError_t e = cudaSuccess;
  if (t->lat_x) {  // non-separable tan maps: one lattice launch per space
    if (want_df) e = launch_lattice(VAR_DF, Pv[VAR_DF], t->lat_x, t->lat_y, s);
    if (e == cudaSuccess && want_std) e = launch_lattice(VAR_STD, Pv[VAR_STD], t->lat_x, t->lat_y, s);
    return e == cudaSuccess ? RF_OK : fail(RF_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
  }
  const bool want_exp = (fmask & (RF_EXPLICIT_STANDARD | RF_EXPLICIT_RGBD)) != 0;
  // TMA when the shared-memory footprint fits the opt-in limit (large radii with wide
  // elements fall back to the LDG halo path) and the tensor map can address the input
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  const int sp_all = (want_std ? 1 : 0) | (want_df ? 2 : 0);
  const bool tma = getenv("RF_DISABLE_TMA") == nullptr &&
                   smem_bytes(sp_all, r, true, esz, want_exp) <= (size_t)di.smem_optin &&
                   make_depth_tmap(&tmap, depth, dtype, batch, H, W, row_pitch, r);
  // Both spaces in one launch (one read and conversion of the input, one launch) for small
  // batches -- at most four waves of tiles, where the launch count and tail waves dominate
  // (a single frame) -- when two such CTAs still fit per SM.  Large batches run one launch
  // per space (disparity form first): measured on C2 (64 frames, w5) the fused kernel's
  // doubled instruction footprint costs more in instruction-fetch stalls (11.6% vs 3.5% of
  // warp samples) than the shared halo saves (1.20-1.23 vs 1.15 ms per step).
  // One wave of tiles at small radii (a single frame): one launch per space at three CTAs per
  // SM (their smaller per-space footprint fits) so every tile has its own CTA slot.
  const LaunchPlan lp = plan_launches(sp_all, r, tma, esz, want_exp, tiles, di);
  const bool fused = lp.fused;
  const bool three = lp.three;
  const size_t sm_both = smem_bytes(3, r, tma, esz, want_exp);
  if (fused) {
    e = launch_radius_sp3(Pv[VAR_STD], Pv[VAR_DF], tmap, tma, sm_both, tiles, di.sms, s, false, false);
  } else {
    // Two launches (one per space): the second is a programmatic dependent launch -- it shares
    // nothing with the first (same input, its own outputs), so its CTAs take the SMs the first
    // frees as its CTAs retire (the first releases its dependents at entry).  The next call's
    // first launch is ordered normally after both.
    const bool pdl = want_df && want_std && getenv("RF_NO_PDL") == nullptr;
    if (pdl) Pv[VAR_DF].pdl_trigger = 1;
    const int minb = three ? 3 : RF_MIN_BLOCKS;
    if (want_df)
      e = launch_radius_sp2(Pv[VAR_STD], Pv[VAR_DF], tmap, tma, smem_bytes(2, r, tma, esz, Pv[VAR_DF].do_exp, minb),
                           tiles, di.sms, s, false, three);
    if (e == cudaSuccess && want_std)
      e = launch_radius_sp1(Pv[VAR_STD], Pv[VAR_DF], tmap, tma, smem_bytes(1, r, tma, esz, Pv[VAR_STD].do_exp, minb),
                           tiles, di.sms, s, pdl, three);
  }
  if (e != cudaSuccess) return fail(RF_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
  return RF_OK;
}

}  // extern "C"
