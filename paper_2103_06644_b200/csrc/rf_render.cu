// rf_render.cu -- the reference's virtual depth sensor on the device (SURVEY.md 8f row 3:
// render_scene, synth.py:137-194).  One thread per pixel: each plane's ray intersection
// Z = -d / (a tan_x + b tan_y + c) (positive, finite, inside the plane's mask rect), the
// nearest one wins (first plane on ties, as np.argmin), then the quadratic depth noise
// Z + (k Z) Z eps and the dropout draw.  The random draws come in as arrays: either the
// reference's own per-row numpy streams (generated on the host, so the frame is the
// reference's bit for bit) or device-generated ones.  The arithmetic is written with
// explicit _rn intrinsics: numpy evaluates it unfused, and so must we for identical bits.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/rangefit_b200.h"
#include "rf_internal.h"

namespace {

constexpr int MAX_PLANES = 256;

struct RenderParams {
  const double* tan_x;
  const double* tan_y;
  const double* lat_x;  // non-separable lattices (distortion offsets) or null
  const double* lat_y;
  const double* planes;  // [nplanes][4]
  const int32_t* rects;  // [nplanes][4], already normalised to [0, W] x [0, H]
  int nplanes, H, W;
  const double* eps;     // [H][W] standard normals or NULL
  const double* uni;     // [H][W] uniforms in [0, 1) or NULL
  double noise_coef, dropout;
  double* depth;
  uint8_t* valid;
  uint8_t* labels;
};

__global__ void render_kernel(const RenderParams P) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= P.W || y >= P.H) return;
  const double tx = rf_tan(P.tan_x, P.lat_x, P.W, x, y, true), ty = rf_tan(P.tan_y, P.lat_y, P.W, x, y, false);
  double best = INFINITY;
  int label = 0;  // np.argmin of an all-inf column is 0; invalid pixels are relabelled below
  for (int p = 0; p < P.nplanes; ++p) {
    const double a = P.planes[4 * p], b = P.planes[4 * p + 1], c = P.planes[4 * p + 2], d = P.planes[4 * p + 3];
    const double denom = __dadd_rn(__dadd_rn(__dmul_rn(a, tx), __dmul_rn(b, ty)), c);
    double z = denom != 0.0 ? __ddiv_rn(-d, denom) : INFINITY;
    if (!(isfinite(z) && z > 0.0)) z = INFINITY;
    const int32_t* r = P.rects + 4 * p;
    if (!(x >= r[0] && x < r[2] && y >= r[1] && y < r[3])) z = INFINITY;
    if (z < best) {
      best = z;
      label = p;
    }
  }
  bool valid = isfinite(best);
  double depth = valid ? best : 0.0;
  const int64_t i = (int64_t)y * P.W + x;
  if (P.eps || P.uni) {
    if (P.eps) depth = __dadd_rn(depth, __dmul_rn(__dmul_rn(__dmul_rn(P.noise_coef, depth), depth), P.eps[i]));
    if (P.uni && P.uni[i] < P.dropout) valid = false;
    valid = valid && depth > 0.0;
    depth = valid ? depth : 0.0;
  }
  P.depth[i] = depth;
  P.valid[i] = valid ? 1 : 0;
  P.labels[i] = valid ? (uint8_t)label : (uint8_t)255;
}

}  // namespace

extern "C" {

rf_status rf_render_planes(const rf_tables* t, const double* planes, const int32_t* rects, int32_t nplanes,
                           const double* eps, const double* uniforms, double noise_coefficient, double dropout,
                           double* depth, uint8_t* valid, uint8_t* labels, void* stream) {
  if (!t || !planes || !rects || !depth || !valid || !labels)
    return rf_set_error(RF_ERR_ARGUMENT, "rf_render_planes: null pointer");
  if (nplanes < 1 || nplanes > MAX_PLANES)
    return rf_set_error(RF_ERR_ARGUMENT, "rf_render_planes: need 1..256 planes (uint8 labels, 255 = invalid)");
  if (!(dropout >= 0.0 && dropout < 1.0)) return rf_set_error(RF_ERR_ARGUMENT, "dropout must be in [0, 1)");
  const rf_device_guard guard(t->device);
  RenderParams P{t->tan_x, t->tan_y, t->lat_x, t->lat_y, planes, rects, nplanes, t->intr.height, t->intr.width, eps, uniforms,
                 noise_coefficient, dropout, depth, valid, labels};
  const dim3 grid((unsigned)((P.W + 127) / 128), (unsigned)P.H);
  render_kernel<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(P);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return rf_set_error(RF_ERR_CUDA, cudaGetErrorString(e));
  return RF_OK;
}

}  // extern "C"
