// rf_internal.h -- definitions shared by the translation units of librangefit_b200.
#pragma once
#include "../../include/rangefit_b200.h"

// per-camera device tables (opaque in the public header)
struct rf_tables {
  rf_intrinsics intr;
  int device;
  double* tan_x;  // [W] device
  double* tan_y;  // [H] device
};

// thread-local error message behind rf_last_error()
rf_status rf_set_error(rf_status s, const char* msg);
