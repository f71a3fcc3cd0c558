/*
 * rangefit_b200.h -- C ABI of the sm_100a per-pixel windowed plane-fit path.
 *
 * This is the drop-in boundary for the reference package `rangefit`
 * (arxiv/paper_2103_06644, /root/reference/pkg/src/rangefit).  The reference is
 * pure Python/numpy and has no FFI; its plugin point is the `backend` string of
 * `fit_rect` (fitting.py:757-786) and its per-window pipeline is
 *   compute_tan_maps (camera.py:124-135)
 *   -> build_{rgbd,standard}_implicit_channels (integral.py:217-263)
 *   -> scatter_from_integrals (fitting.py:420-533)
 *   -> fit_implicit_{rgbd,standard} (fitting.py:546-579)
 *   -> canonicalize_implicit (fitting.py:76-94).
 * Each entry point below names the reference interface it replaces.  The
 * Python host layer (paper_2103_06644_b200/) binds these with ctypes; see
 * INTEGRATION.md for the binding a maintainer adds on the reference side.
 *
 * Conventions: no C++ exceptions cross this boundary; every call returns an
 * rf_status; rf_last_error() returns a thread-local message.  All device
 * buffers are caller-owned.  Calls are stream-ordered and asynchronous.
 */
#ifndef RANGEFIT_B200_H
#define RANGEFIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RF_ABI_VERSION 4

typedef enum rf_status {
  RF_OK = 0,
  RF_ERR_ARGUMENT = 1,    /* bad argument (reference: ValueError)              */
  RF_ERR_SHAPE = 2,       /* shape / dtype mismatch (reference: ValueError)    */
  RF_ERR_CUDA = 3,        /* CUDA runtime error                                */
  RF_ERR_UNSUPPORTED = 4  /* valid reference input this path does not support  */
} rf_status;

/* depth element types (reference DepthImage, synth.py:69-114) */
typedef enum rf_depth_dtype {
  RF_DEPTH_F32_M = 0,   /* float32 metres; valid = isfinite & > 0 (synth.py:84)     */
  RF_DEPTH_U16_MM = 1,  /* uint16 millimetres; Z = mm / 1000.0, valid = mm > 0
                           (DepthImage.from_millimeters, synth.py:111-114)         */
  RF_DEPTH_F64_M = 2    /* float64 metres (DepthImage.values as held by the reference,
                           the loss-free RF64 files); valid = isfinite & > 0         */
} rf_depth_dtype;

/* formulation ids = positions in the reference's FORMULATIONS tuple (fitting.py:45-49) */
#define RF_FORM_IMPLICIT_STANDARD 0 /* "implicit-standard": smallest eigvec of [X,Y,Z,1] scatter */
#define RF_FORM_IMPLICIT_RGBD 1     /* "implicit-rgbd" (disparity form): [tx, ty, 1, 1/Z]       */
#define RF_FORM_EXPLICIT_STANDARD 2 /* "explicit-standard": Z = aX + bY + c                     */
#define RF_FORM_EXPLICIT_RGBD 3     /* "explicit-rgbd": 1/Z = a tx + b ty + c                    */
#define RF_NUM_FORMULATIONS 4
/* formulation mask bits (1 << id) */
#define RF_IMPLICIT_STANDARD (1 << RF_FORM_IMPLICIT_STANDARD)
#define RF_IMPLICIT_RGBD (1 << RF_FORM_IMPLICIT_RGBD)
#define RF_EXPLICIT_STANDARD (1 << RF_FORM_EXPLICIT_STANDARD)
#define RF_EXPLICIT_RGBD (1 << RF_FORM_EXPLICIT_RGBD)
#define RF_ALL_FORMULATIONS 15

/* status bits of the per-pixel status byte */
#define RF_PIX_INPUT_VALID 1u  /* centre pixel valid (DepthImage.valid)               */
#define RF_PIX_FIT 2u          /* centre valid and window holds >= MIN_SAMPLES
                                  (4 implicit, 3 explicit; fitting.py:55-60)          */
#define RF_PIX_DEGENERATE 4u   /* FitResult.degenerate (fitting.py:553-554 implicit,
                                  Cholesky pivot failure fitting.py:584-589 explicit)  */

/* Pinhole intrinsics (reference CameraIntrinsics, camera.py:35-75). */
typedef struct rf_intrinsics {
  double fx, fy, cx, cy;
  int32_t width, height;
} rf_intrinsics;

/* Per-camera device tables (reference TanAngleMaps, camera.py:78-96): the
 * separable tan lattices tan_x[x] = (x - cx)/fx, tan_y[y] = (y - cy)/fy. */
typedef struct rf_tables rf_tables;

/* Caller-owned device output planes for one formulation, each [batch, H, W]
 * (normal is [batch, H, W, 3], xyz interleaved).  Pixels whose status lacks
 * RF_PIX_FIT hold NaN in every float plane.  Explicit fits are reported in
 * implicit form (explicit_to_implicit, fitting.py:729-739) and their residual is
 * the rms of the explicit objective (fitting.py:590-597). */
typedef struct rf_pixel_out {
  float* normal;     /* unit normal (a,b,c)/|(a,b,c)|, canonical sign (fitting.py:76-94) */
  float* offset;     /* d/|(a,b,c)|: n.X + offset = 0                                    */
  float* residual;   /* FitResult.rms_residual = sqrt(max(lambda,0)/n) (fitting.py:556)  */
  float* curvature;  /* lambda_min(C3)/trace(C3) of the centred monomial scatter         */
  uint8_t* status;   /* RF_PIX_* bits                                                    */
} rf_pixel_out;

/* Replaces compute_tan_maps (camera.py:124-135) + the camera-constant channel
 * stack build_constant_channels (integral.py:193-199), once per camera.
 * delta_x / delta_y (H*W float64 host arrays, CameraIntrinsics.delta_*) may be NULL
 * (zero).  Zero lattices keep the separable tables the tile kernels need; non-zero
 * lattices are stored whole ((x + delta_x - cx) / fx, ...) and every kernel reads them
 * per pixel (the per-pixel fits then sum each window directly, slower but exact).
 * Validation mirrors CameraIntrinsics.__post_init__. */
rf_status rf_tables_create(const rf_intrinsics* intrinsics, const double* delta_x,
                           const double* delta_y, int device, rf_tables** out);
rf_status rf_tables_destroy(rf_tables* tables);

/* Replaces, for every pixel of a batch of frames, the reference pipeline
 *   fit_rect(depth, maps, Rect(max(x-r,0), max(y-r,0), min(x+r+1,W), min(y+r+1,H)),
 *            formulation, backend)            (fitting.py:757-786)
 * with window = 2r+1, for each formulation whose bit is set in formulation_mask.
 * depth: device pointer to batch frames of H rows, each row_pitch elements apart
 * (frame stride = H*row_pitch).  mask: optional device uint8 [batch,H,W]
 * (DepthImage(values, valid=mask), synth.py:88-94) or NULL.  outs: array of
 * RF_NUM_FORMULATIONS output sets indexed by RF_FORM_*; only the requested entries
 * are read.  The implicit and explicit fits of one space share one pass over its window
 * moments; small batches fit both spaces in one launch (rf_launches_per_call).  The tables
 * are immutable: any number of streams may share one handle concurrently.
 * stream: a cudaStream_t (NULL = legacy default). */
rf_status rf_fit_pixels(const rf_tables* tables, const void* depth, int dtype, int64_t batch,
                        int32_t height, int32_t width, int64_t row_pitch, const uint8_t* mask,
                        int32_t window, int32_t formulation_mask, const rf_pixel_out* outs,
                        void* stream);

/* One half-open pixel rectangle of one frame (reference Rect, integral.py:50-66). */
typedef struct rf_rect {
  int32_t frame, x0, y0, x1, y1;
} rf_rect;

/* rect status bits */
#define RF_RECT_FIT 2u            /* n_points >= MIN_SAMPLES (else InsufficientSamplesError) */
#define RF_RECT_DEGENERATE 4u     /* FitResult.degenerate                                    */
#define RF_RECT_OUT_OF_BOUNDS 16u /* _check_rect failed (integral.py:131-133, ValueError)    */

/* Per-rect result (reference FitResult, fitting.py:158-174), fp64. */
typedef struct rf_rect_fit {
  double coef[4];          /* canonical implicit (a,b,c,d) (ImplicitPlane / explicit_to_implicit) */
  double explicit_coef[3]; /* ExplicitPlane.coefficients for explicit formulations, else NaN   */
  double eigenvalue;       /* smallest scatter eigenvalue (implicit), else NaN                */
  double rms;              /* FitResult.rms_residual                                           */
  double curvature;        /* SURVEY.md A17 extension                                          */
  int32_t n_points;        /* valid samples in the rect                                        */
  int32_t status;          /* RF_RECT_* bits                                                   */
} rf_rect_fit;

/* Replaces fit_rect(depth, maps, rect, formulation, backend) (fitting.py:757-786)
 * for a device list of rects of a [batch, H, W] depth tensor; one formulation
 * (RF_FORM_*) per call; `out` is a device array of nrects results.  Sums are
 * direct over each rect (the naive backend's numerics, fitting.py:339-402). */
rf_status rf_fit_rects(const rf_tables* tables, const void* depth, int dtype, int64_t batch,
                       int32_t height, int32_t width, int64_t row_pitch, const uint8_t* mask,
                       const rf_rect* rects, int64_t nrects, int32_t formulation,
                       rf_rect_fit* out, void* stream);

/* Replaces segment.py's _max_residual (segment.py:306-325) for a device list of rects and
 * planes: out[r] = max |objective| over the rect's valid pixels (0 for none), with coefs
 * [nrects][4] = the canonical implicit coefficients (implicit formulations) or the
 * ExplicitPlane (a, b, c) (explicit; 4th entry unused). */
rf_status rf_max_residuals(const rf_tables* tables, const void* depth, int dtype, int64_t batch,
                           int32_t height, int32_t width, int64_t row_pitch, const uint8_t* mask,
                           const rf_rect* rects, int64_t nrects, int32_t formulation, const double* coefs,
                           double* out, void* stream);

/* Number of kernel launches rf_fit_pixels issues on the current device for a formulation
 * mask, window, depth dtype and batch shape with separable tables: one tile kernel for both
 * spaces on small batches (up to four waves of tiles) when two of its CTAs fit per SM, else
 * one per space. */
int32_t rf_launches_per_call(int32_t formulation_mask, int32_t window, int32_t dtype, int64_t batch,
                             int32_t height, int32_t width);

/* Thread-local message describing the last non-RF_OK status. */
const char* rf_last_error(void);

/* ---- the reference's integral backend on the device (8b) ----
 * Channels of the reference's ChannelStacks (integral.py:36-47, 188-325).  Depth-derived
 * channels are masked by validity (0 where invalid); the constant tan monomials are not. */
typedef enum rf_channel {
  RF_CH_COUNT = 0,      /* validity as 0/1 (the per-frame "count" channel)            */
  RF_CH_ONES = 1,       /* every pixel (the constant stack's count)                  */
  RF_CH_X2 = 2, RF_CH_XY = 3, RF_CH_XZ = 4, RF_CH_X = 5, RF_CH_Y2 = 6, RF_CH_YZ = 7,
  RF_CH_Y = 8, RF_CH_Z2 = 9, RF_CH_Z = 10,            /* X = Z tan_x, Y = Z tan_y   */
  RF_CH_TX_OVER_Z = 11, RF_CH_TY_OVER_Z = 12, RF_CH_INV_Z = 13, RF_CH_INV_Z2 = 14,
  RF_CH_TX2 = 15, RF_CH_TXTY = 16, RF_CH_TY2 = 17, RF_CH_TX = 18, RF_CH_TY = 19,
  RF_CH_M_TX2 = 20, RF_CH_M_TXTY = 21, RF_CH_M_TY2 = 22, RF_CH_M_TX = 23, RF_CH_M_TY = 24
} rf_channel;
#define RF_NUM_CHANNELS 25
#define RF_MAX_BOX_CHANNELS 32

/* Replaces build_integral(channel(depth), valid) (integral.py:136-149) for one channel of
 * one frame: table is a device [height+1][width+1] fp64 array (row 0 and column 0 zero).
 * The additions are numpy's (cumsum down each column, then along each row, sequential), so
 * the table equals the reference's bit for bit.  mask: optional device uint8 [H][W]. */
rf_status rf_build_channel(const rf_tables* tables, const void* depth, int dtype, int64_t row_pitch,
                           const uint8_t* mask, int32_t channel, double* table, void* stream);

/* build_integral(src, mask) (integral.py:136-149) for an arbitrary fp64 device channel
 * [height][src_pitch]; mask optional. */
rf_status rf_integral(const double* src, int64_t src_pitch, const uint8_t* mask, int32_t height,
                      int32_t width, double* table, void* stream);

/* _box / box_sum (fitting.py:405-411, integral.py:152-158) of nch tables (a HOST array of
 * device table pointers, each [height+1][width+1]) over nrects device rects (the frame field
 * is ignored): out[r][c] = t[y1,x1] - t[y0,x1] - t[y1,x0] + t[y0,x0], evaluated in that
 * order.  Out-of-bounds rects give NaN (callers check bounds, integral.py:131-133). */
rf_status rf_box_sums(const double* const* tables, int32_t nch, int32_t height, int32_t width,
                      const rf_rect* rects, int64_t nrects, double* out, void* stream);

#define RF_RECT_JACOBI_FAILED 8u  /* jacobi_eigh did not converge (DegenerateFitError)  */

/* Replaces FIT_BY_FORMULATION[formulation](scatter) (fitting.py:546-629) for n assembled
 * systems, all device arrays: matrices [n][16] (row-major 4x4 Scatter4.matrix; explicit: the
 * 3x3 Scatter3.matrix in the top-left, row stride 4), rhs [n][3] (explicit only, else NULL),
 * target_sq [n] (explicit, NaN = absent; may be NULL), counts [n] (Scatter*.n).
 * Implicit: the smallest eigenpair through the same solve as the per-pixel kernels (Schur
 * complement on the constant monomial; cyclic Jacobi when that entry is not positive).
 * Explicit: the reference's Cholesky (pivot floor 1e-12 trace) or, when rank-deficient, the
 * minimum-norm solution from a cyclic Jacobi (fitting.py:264-327).  Results as rf_rect_fit
 * (rms NaN where the reference returns None). */
rf_status rf_fit_scatters(const double* matrices, const double* rhs, const double* target_sq,
                          const int64_t* counts, int64_t n, int32_t formulation, rf_rect_fit* out,
                          void* stream);

/* ---- the reference's virtual depth sensor (render_scene, synth.py:137-194) ----
 * One frame of the camera in `tables`: planes [nplanes][4] (unit-normal a,b,c,d), rects
 * [nplanes][4] half-open pixel bounds already clipped to the frame (the whole frame for
 * planes without a mask rect); eps [H][W] standard normals (NULL = no noise), uniforms
 * [H][W] in [0,1) (NULL = no dropout): nearest positive intersection, Z += k Z^2 eps,
 * dropout, validity Z > 0.  Outputs depth fp64 [H][W] (0 where invalid), valid and labels
 * uint8 [H][W] (plane index, 255 = invalid).  All arrays are device memory. */
rf_status rf_render_planes(const rf_tables* tables, const double* planes, const int32_t* rects, int32_t nplanes,
                           const double* eps, const double* uniforms, double noise_coefficient, double dropout,
                           double* depth, uint8_t* valid, uint8_t* labels, void* stream);

/* RF_ABI_VERSION of the loaded library. */
int32_t rf_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RANGEFIT_B200_H */
