// rf_internal.h -- definitions shared by the translation units of librangefit_b200.
#pragma once
#include "../../include/rangefit_b200.h"

// per-camera device tables (opaque in the public header); immutable after rf_tables_create,
// so one handle serves any number of concurrent streams
struct rf_tables {
  rf_intrinsics intr;
  int device;
  double* tan_x;  // [W] device: (x - cx) / fx
  double* tan_y;  // [H] device: (y - cy) / fy
  // non-zero distortion lattices (CameraIntrinsics.delta_*): the full tan lattices
  // (x + delta_x - cx) / fx and (y + delta_y - cy) / fy, [H][W] device; null when separable
  double* lat_x;
  double* lat_y;
};

// tan_x / tan_y of pixel (x, y): the lattice when the camera has distortion offsets
#ifdef __CUDACC__
__host__ __device__
#endif
inline double rf_tan(const double* table, const double* lattice, int W, int x, int y, bool along_x) {
  return lattice ? lattice[(long long)y * W + x] : table[along_x ? x : y];
}

#ifdef __CUDACC__
#include <cuda_runtime.h>
// makes the tables' device current for one entry point (restored on exit), so that a
// caller whose current device differs still launches where the tables and buffers live
struct rf_device_guard {
  int prev = -1;
  explicit rf_device_guard(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != device) cudaSetDevice(device);
    else prev = -1;
  }
  ~rf_device_guard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
#endif

// thread-local error message behind rf_last_error()
rf_status rf_set_error(rf_status s, const char* msg);
