/*
 * rf_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference
 * per-window implicit plane fit (arxiv/paper_2103_06644, package `rangefit`),
 * used as the parity checker for the sm_100a kernels and as the timed CPU
 * baseline in bench.py.  Nothing in the product path links or calls this file.
 *
 * Parity is pinned against the reference itself: tests/golden/make_golden.py
 * runs the reference's own `fit_rect` per pixel and tests/test_oracle.py checks
 * this restatement against those vectors.
 *
 * What is restated (reference = /root/reference/pkg/src/rangefit/):
 *   - naive backend: gather_window_samples + accumulate_scatter_naive
 *       fitting.py:339-402  (standard samples (Z*tx, Z*ty, Z); rgbd samples
 *       (tx, ty, Z) with one 1/Z per sample, fitting.py:361; monomials
 *       [X,Y,Z,1] / [tx,ty,1,1/Z], fitting.py:364-369)
 *   - integral backend: build_integral (cumsum axis 0 then axis 1,
 *       integral.py:136-149), stack builders integral.py:188-263, constant
 *       stack integral.py:193-199, box sums fitting.py:405-411 and
 *       scatter_from_integrals fitting.py:420-521 (constant tan block iff
 *       n == rect.area, masked tan channels otherwise, fitting.py:482-504)
 *   - cyclic Jacobi: jacobi_eigh fitting.py:193-253 (same rotation formulas,
 *       thresholds 1e-13*||A||_F, 50 sweeps, theta > 1e8 shortcut)
 *   - _fit_implicit fitting.py:546-559 (argsort, gap, degenerate flag with
 *       _EIGEN_TIE_REL = 1e-9, rms = sqrt(max(lam,0)/n))
 *   - canonicalize_implicit fitting.py:76-94 (order (c,b,a,d), eps 1e-9)
 *   - explicit fits: the normal equations read from the same space's scatter
 *       (accumulate_scatter_naive / scatter_from_integrals, fitting.py:370-381,
 *       464-476, 523-533), cholesky3 + solve_cholesky3 or _pinv_solve,
 *       _fit_explicit and explicit_to_implicit (fitting.py:264-322, 582-599,
 *       729-739), MIN_SAMPLES 3
 * Per-pixel extensions (not in the reference):
 *   - window of pixel (x,y): Rect(max(x-r,0), max(y-r,0), min(x+r+1,W),
 *     min(y+r+1,H)) -- clipped like the segmenter's border tiles
 *     (segment.py:287-292)
 *   - status bit0 = centre pixel valid, bit1 = bit0 && n >= MIN_SAMPLES (4),
 *     bit2 = degenerate, bit3 = reference solver raised DegenerateFitError
 *   - unit normal (a,b,c)/|(a,b,c)|, offset d/|(a,b,c)|, residual = rms,
 *     curvature = lambda_min(C3)/trace(C3), C3 = S[I,I] - S[I,k]S[I,k]^T/n,
 *     I=(0,1,2),k=3 for standard and I=(0,1,3),k=2 for rgbd.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>
#include <unistd.h>

#define RFO_STANDARD 0          /* implicit-standard */
#define RFO_RGBD 1              /* implicit-rgbd (disparity form) */
#define RFO_EXPLICIT_STANDARD 2 /* explicit-standard */
#define RFO_EXPLICIT_RGBD 3     /* explicit-rgbd */
#define RFO_SPACE(f) ((f) == RFO_STANDARD || (f) == RFO_EXPLICIT_STANDARD ? RFO_STANDARD : RFO_RGBD)
#define RFO_NAIVE 0
#define RFO_INTEGRAL 1

static const double CANONICAL_EPS = 1e-9;  /* fitting.py:65 */
static const double EIGEN_TIE_REL = 1e-9;  /* fitting.py:69 */
static const double PIVOT_REL = 1e-12;     /* fitting.py:71 */

/* ---- jacobi_eigh, fitting.py:193-253 (returns 0 ok, -1 not converged) ---- */
static int jacobi_eigh(int n, const double* m, double* values, double* vectors) {
  double a[16], v[16];
  double fro2 = 0.0;
  for (int i = 0; i < n * n; ++i) { a[i] = m[i]; fro2 += m[i] * m[i]; }
  double fro = sqrt(fro2);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) v[i * n + j] = (i == j) ? 1.0 : 0.0;
  if (fro == 0.0) {
    for (int i = 0; i < n; ++i) values[i] = 0.0;
    memcpy(vectors, v, sizeof(double) * n * n);
    return 0;
  }
  const double threshold = 1e-13 * fro;
  for (int sweep = 0; sweep < 50; ++sweep) {
    double off2 = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off2 += a[p * n + q] * a[p * n + q];
    if (sqrt(2.0 * off2) <= threshold) {
      for (int i = 0; i < n; ++i) values[i] = a[i * n + i];
      memcpy(vectors, v, sizeof(double) * n * n);
      return 0;
    }
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        double apq = a[p * n + q];
        if (apq == 0.0) continue;
        double theta = 0.5 * (a[q * n + q] - a[p * n + p]) / apq;
        double t;
        if (fabs(theta) > 1e8) t = 0.5 / theta;
        else if (theta >= 0.0) t = 1.0 / (theta + sqrt(1.0 + theta * theta));
        else t = -1.0 / (-theta + sqrt(1.0 + theta * theta));
        double c = 1.0 / sqrt(1.0 + t * t);
        double s = t * c;
        double app = a[p * n + p], aqq = a[q * n + q];
        a[p * n + p] = app - t * apq;
        a[q * n + q] = aqq + t * apq;
        a[p * n + q] = a[q * n + p] = 0.0;
        for (int k = 0; k < n; ++k) {
          if (k == p || k == q) continue;
          double akp = a[k * n + p], akq = a[k * n + q];
          a[k * n + p] = a[p * n + k] = c * akp - s * akq;
          a[k * n + q] = a[q * n + k] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          double vkp = v[k * n + p], vkq = v[k * n + q];
          v[k * n + p] = c * vkp - s * vkq;
          v[k * n + q] = s * vkp + c * vkq;
        }
      }
    }
  }
  double off2 = 0.0;
  for (int p = 0; p < n; ++p)
    for (int q = p + 1; q < n; ++q) off2 += a[p * n + q] * a[p * n + q];
  for (int i = 0; i < n; ++i) values[i] = a[i * n + i];
  memcpy(vectors, v, sizeof(double) * n * n);
  return sqrt(2.0 * off2) > threshold ? -1 : 0;
}

/* stable ascending argsort of <= 4 values (insertion sort) */
static void argsort(int n, const double* vals, int* order) {
  for (int i = 0; i < n; ++i) order[i] = i;
  for (int i = 1; i < n; ++i) {
    int k = order[i], j = i - 1;
    while (j >= 0 && vals[order[j]] > vals[k]) { order[j + 1] = order[j]; --j; }
    order[j + 1] = k;
  }
}

/* canonicalize_implicit, fitting.py:76-94 */
static void canonicalize(const double* coef, double* out) {
  double norm = sqrt(coef[0] * coef[0] + coef[1] * coef[1] + coef[2] * coef[2] + coef[3] * coef[3]);
  double unit[4];
  for (int i = 0; i < 4; ++i) unit[i] = coef[i] / norm;
  static const int order[4] = {2, 1, 0, 3};
  double sign = 1.0;
  for (int k = 0; k < 4; ++k) {
    if (fabs(unit[order[k]]) > CANONICAL_EPS) { sign = unit[order[k]] > 0 ? 1.0 : -1.0; break; }
  }
  for (int i = 0; i < 4; ++i) out[i] = sign * unit[i];
}

typedef struct {
  double coef[4];   /* canonical unit 4-vector (a,b,c,d) */
  double lam;       /* smallest eigenvalue */
  double rms;
  double curvature;
  double scale;     /* ||S||_F / n, sets the rounding floor of lambda */
  double curv_cond; /* sum of the uncentred diagonal / trace(C3): rounding amplification of kappa */
  int degenerate;
  int failed;
} fit_out;

static double curvature_of(const double* S, int space, double* cond);

/* _fit_implicit fitting.py:546-559 plus the A17 curvature extension */
static void fit_scatter(const double* S, int n, int formulation, fit_out* o) {
  double vals[4], vecs[16];
  o->failed = jacobi_eigh(4, S, vals, vecs) != 0;
  int order[4];
  argsort(4, vals, order);
  int sm = order[0];
  double lam = vals[sm];
  double fro2 = 0.0;
  for (int i = 0; i < 16; ++i) fro2 += S[i] * S[i];
  double fro = sqrt(fro2);
  double gap = vals[order[1]] - lam;
  o->degenerate = (fro == 0.0) || (gap <= EIGEN_TIE_REL * fro);
  o->scale = fro / (double)n;
  double v[4] = {vecs[0 * 4 + sm], vecs[1 * 4 + sm], vecs[2 * 4 + sm], vecs[3 * 4 + sm]};
  canonicalize(v, o->coef);
  o->lam = lam;
  o->rms = sqrt((lam > 0.0 ? lam : 0.0) / (double)n);
  /* curvature: centred 3x3 block of the non-constant monomials */
  o->curvature = curvature_of(S, formulation, &o->curv_cond);
}

/* curvature (A17) from an implicit 4x4 scatter of the formulation's space; *cond receives
 * the rounding amplification sum_i S[I_i][I_i] / trace(C3) of the centring (test metric) */
static double curvature_of(const double* S, int space, double* cond) {
  int I[3], k;
  if (space == RFO_STANDARD) { I[0] = 0; I[1] = 1; I[2] = 2; k = 3; }
  else { I[0] = 0; I[1] = 1; I[2] = 3; k = 2; }
  double nn = S[k * 4 + k];
  double C3[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      C3[i * 3 + j] = S[I[i] * 4 + I[j]] - S[I[i] * 4 + k] * S[I[j] * 4 + k] / nn;
  double cv[3], cvec[9];
  jacobi_eigh(3, C3, cv, cvec);
  double mn = cv[0];
  if (cv[1] < mn) mn = cv[1];
  if (cv[2] < mn) mn = cv[2];
  double tr = C3[0] + C3[4] + C3[8];
  if (cond) *cond = tr > 0.0 ? (S[I[0] * 4 + I[0]] + S[I[1] * 4 + I[1]] + S[I[2] * 4 + I[2]]) / tr : INFINITY;
  return tr > 0.0 ? mn / tr : 0.0;
}

/* cholesky3 fitting.py:264-293; returns 0, or -1 for DegenerateFitError */
static int cholesky3(const double* s, double* L) {
  double trace = s[0] + s[4] + s[8];
  double floor = PIVOT_REL * trace;
  if (!isfinite(trace) || trace <= 0.0) return -1;
  double p0 = s[0];
  if (p0 <= floor) return -1;
  double l00 = sqrt(p0), l10 = s[3] / l00, l20 = s[6] / l00;
  double p1 = s[4] - l10 * l10;
  if (p1 <= floor) return -1;
  double l11 = sqrt(p1), l21 = (s[7] - l20 * l10) / l11;
  double p2 = s[8] - l20 * l20 - l21 * l21;
  if (p2 <= floor) return -1;
  double l22 = sqrt(p2);
  L[0] = l00; L[1] = l10; L[2] = l11; L[3] = l20; L[4] = l21; L[5] = l22;
  return 0;
}

/* _fit_explicit fitting.py:582-599 (+ explicit_to_implicit :729-739, A17 curvature).
 * S: the implicit 4x4 scatter of the same space, from which the explicit normal
 * equations are read: standard M = S[{0,1,3}], rhs = S[{0,1,3},2], target Z;
 * rgbd M = S[{0,1,2}], rhs = S[{0,1,2},3], target 1/Z. */
static void fit_explicit(const double* S, int n, int space, fit_out* o) {
  int I[3], tcol;
  if (space == RFO_STANDARD) { I[0] = 0; I[1] = 1; I[2] = 3; tcol = 2; }
  else { I[0] = 0; I[1] = 1; I[2] = 2; tcol = 3; }
  double M[9], rhs[3];
  for (int i = 0; i < 3; ++i) {
    rhs[i] = S[I[i] * 4 + tcol];
    for (int j = 0; j < 3; ++j) M[i * 3 + j] = S[I[i] * 4 + I[j]];
  }
  double target_sq = S[tcol * 4 + tcol];
  double L[6], alpha[3];
  o->failed = 0;
  if (cholesky3(M, L) == 0) {
    /* solve_cholesky3 fitting.py:296-305 */
    double y0 = rhs[0] / L[0];
    double y1 = (rhs[1] - L[1] * y0) / L[2];
    double y2 = (rhs[2] - L[3] * y0 - L[4] * y1) / L[5];
    alpha[2] = y2 / L[5];
    alpha[1] = (y1 - L[4] * alpha[2]) / L[2];
    alpha[0] = (y0 - L[1] * alpha[1] - L[3] * alpha[2]) / L[0];
    o->degenerate = 0;
  } else {
    /* _pinv_solve fitting.py:313-322 */
    double vals[3], vecs[9];
    jacobi_eigh(3, M, vals, vecs);
    double tr = M[0] + M[4] + M[8];
    double tol = PIVOT_REL * (tr > 0.0 ? tr : 0.0);
    alpha[0] = alpha[1] = alpha[2] = 0.0;
    for (int i = 0; i < 3; ++i) {
      if (vals[i] > tol) {
        double ub = vecs[0 * 3 + i] * rhs[0] + vecs[1 * 3 + i] * rhs[1] + vecs[2 * 3 + i] * rhs[2];
        for (int k = 0; k < 3; ++k) alpha[k] += vecs[k * 3 + i] * (ub / vals[i]);
      }
    }
    o->degenerate = 1;
  }
  double sq = target_sq - (alpha[0] * rhs[0] + alpha[1] * rhs[1] + alpha[2] * rhs[2]);
  o->rms = sqrt((sq > 0.0 ? sq : 0.0) / (double)n);
  o->lam = sq;
  double imp[4];
  if (space == RFO_STANDARD) { imp[0] = alpha[0]; imp[1] = alpha[1]; imp[2] = -1.0; imp[3] = alpha[2]; }
  else { imp[0] = alpha[0]; imp[1] = alpha[1]; imp[2] = alpha[2]; imp[3] = -1.0; }
  canonicalize(imp, o->coef);
  double fro2 = 0.0;
  for (int i = 0; i < 16; ++i) fro2 += S[i] * S[i];
  o->scale = sqrt(fro2) / (double)n;
  o->curvature = curvature_of(S, space, &o->curv_cond);
}

/* ---- naive scatter: gather_window_samples + accumulate_scatter_naive ---- */
static int naive_scatter(const double* depth, const uint8_t* valid, const double* tan_x,
                         const double* tan_y, int W, int x0, int y0, int x1, int y1,
                         int formulation, double* S) {
  double acc[16];
  memset(acc, 0, sizeof(acc));
  int n = 0;
  for (int y = y0; y < y1; ++y) {
    for (int x = x0; x < x1; ++x) {
      int64_t i = (int64_t)y * W + x;
      if (!valid[i]) continue;
      double z = depth[i], tx = tan_x[i], ty = tan_y[i];
      double m[4];
      if (formulation == RFO_STANDARD) { m[0] = z * tx; m[1] = z * ty; m[2] = z; m[3] = 1.0; }
      else { m[0] = tx; m[1] = ty; m[2] = 1.0; m[3] = 1.0 / z; }
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) acc[a * 4 + b] += m[a] * m[b];
      ++n;
    }
  }
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) S[a * 4 + b] = (acc[a * 4 + b] + acc[b * 4 + a]) * 0.5;
  return n;
}

/* ---- integral backend: per-frame summed-area tables ---- */
typedef struct {
  int H, W, nch;
  double* t; /* nch x (H+1) x (W+1) */
} sat_stack;

/* build_integral: table[1:,1:] = cumsum(cumsum(src, axis=0), axis=1) */
static void build_integral_into(double* table, const double* src, int H, int W) {
  int64_t TW = W + 1;
  for (int x = 0; x <= W; ++x) table[x] = 0.0;
  for (int y = 0; y < H; ++y) {
    table[(int64_t)(y + 1) * TW] = 0.0;
    for (int x = 0; x < W; ++x) table[(int64_t)(y + 1) * TW + x + 1] = src[(int64_t)y * W + x];
  }
  /* cumsum over axis 0 (down the columns), sequential like numpy */
  for (int y = 1; y < H; ++y)
    for (int x = 0; x < W; ++x)
      table[(int64_t)(y + 1) * TW + x + 1] += table[(int64_t)y * TW + x + 1];
  /* cumsum over axis 1 (along the rows) */
  for (int y = 0; y < H; ++y)
    for (int x = 1; x < W; ++x)
      table[(int64_t)(y + 1) * TW + x + 1] += table[(int64_t)(y + 1) * TW + x];
}

static double box(const double* t, int W, int x0, int y0, int x1, int y1) {
  int64_t TW = W + 1;
  return t[(int64_t)y1 * TW + x1] - t[(int64_t)y0 * TW + x1] - t[(int64_t)y1 * TW + x0] +
         t[(int64_t)y0 * TW + x0];
}

/* channel index layout of the oracle's SAT stack */
enum { CH_COUNT = 0, CH_ST_X2, CH_ST_XY, CH_ST_XZ, CH_ST_X, CH_ST_Y2, CH_ST_YZ, CH_ST_Y, CH_ST_Z2, CH_ST_Z,
       CH_ST_END };
enum { CHD_COUNT = 0, CHD_TXW, CHD_TYW, CHD_W, CHD_W2, CHD_MTX2, CHD_MTXTY, CHD_MTY2, CHD_MTX, CHD_MTY,
       CHD_CTX2, CHD_CTXTY, CHD_CTY2, CHD_CTX, CHD_CTY, CHD_END };

static int build_stack(const double* depth, const uint8_t* valid, const double* tan_x,
                       const double* tan_y, int H, int W, int formulation, sat_stack* st) {
  int64_t N = (int64_t)H * W;
  int64_t TS = (int64_t)(H + 1) * (W + 1);
  st->H = H; st->W = W;
  st->nch = formulation == RFO_STANDARD ? CH_ST_END : CHD_END;
  st->t = (double*)malloc(sizeof(double) * TS * st->nch);
  double* src = (double*)malloc(sizeof(double) * N);
  if (!st->t || !src) { free(st->t); free(src); return -1; }
  /* count = mask as float64 (integral.py:176) */
  for (int64_t i = 0; i < N; ++i) src[i] = valid[i] ? 1.0 : 0.0;
  build_integral_into(st->t, src, H, W);
  if (formulation == RFO_STANDARD) {
    /* build_standard_implicit_channels, integral.py:217-237 */
    for (int c = CH_ST_X2; c < CH_ST_END; ++c) {
      for (int64_t i = 0; i < N; ++i) {
        double z = valid[i] ? depth[i] : 0.0;
        double x = z * tan_x[i], y = z * tan_y[i], val;
        switch (c) {
          case CH_ST_X2: val = x * x; break;
          case CH_ST_XY: val = x * y; break;
          case CH_ST_XZ: val = x * z; break;
          case CH_ST_X: val = x; break;
          case CH_ST_Y2: val = y * y; break;
          case CH_ST_YZ: val = y * z; break;
          case CH_ST_Y: val = y; break;
          case CH_ST_Z2: val = z * z; break;
          default: val = z; break;
        }
        src[i] = valid[i] ? val : 0.0;
      }
      build_integral_into(st->t + TS * c, src, H, W);
    }
  } else {
    /* build_rgbd_implicit_channels integral.py:240-263 + constant stack :193-199 */
    for (int c = CHD_TXW; c < CHD_END; ++c) {
      for (int64_t i = 0; i < N; ++i) {
        double w = valid[i] ? 1.0 / depth[i] : 0.0;
        double tx = tan_x[i], ty = tan_y[i], val;
        int masked = 1;
        switch (c) {
          case CHD_TXW: val = tx * w; break;
          case CHD_TYW: val = ty * w; break;
          case CHD_W: val = w; break;
          case CHD_W2: val = w * w; break;
          case CHD_MTX2: case CHD_CTX2: val = tx * tx; masked = c == CHD_MTX2; break;
          case CHD_MTXTY: case CHD_CTXTY: val = tx * ty; masked = c == CHD_MTXTY; break;
          case CHD_MTY2: case CHD_CTY2: val = ty * ty; masked = c == CHD_MTY2; break;
          case CHD_MTX: case CHD_CTX: val = tx; masked = c == CHD_MTX; break;
          default: val = ty; masked = c == CHD_MTY; break;
        }
        src[i] = (!masked || valid[i]) ? val : 0.0;
      }
      build_integral_into(st->t + TS * c, src, H, W);
    }
  }
  free(src);
  return 0;
}

/* scatter_from_integrals, fitting.py:420-521 */
static int integral_scatter(const sat_stack* st, int x0, int y0, int x1, int y1, int formulation,
                            int min_samples, double* S) {
  int64_t TS = (int64_t)(st->H + 1) * (st->W + 1);
  int W = st->W;
#define BOX(c) box(st->t + TS * (c), W, x0, y0, x1, y1)
  int n = (int)llround(BOX(0));
  if (n < min_samples) return n;
  if (formulation == RFO_STANDARD) {
    double sx2 = BOX(CH_ST_X2), sxy = BOX(CH_ST_XY), sxz = BOX(CH_ST_XZ), sx = BOX(CH_ST_X);
    double sy2 = BOX(CH_ST_Y2), syz = BOX(CH_ST_YZ), sy = BOX(CH_ST_Y), sz2 = BOX(CH_ST_Z2),
           sz = BOX(CH_ST_Z);
    double m[16] = {sx2, sxy, sxz, sx, sxy, sy2, syz, sy, sxz, syz, sz2, sz, sx, sy, sz, (double)n};
    memcpy(S, m, sizeof(m));
  } else {
    double stx2, stxty, sty2, stx, sty;
    if (n == (x1 - x0) * (y1 - y0)) {
      stx2 = BOX(CHD_CTX2); stxty = BOX(CHD_CTXTY); sty2 = BOX(CHD_CTY2); stx = BOX(CHD_CTX);
      sty = BOX(CHD_CTY);
    } else {
      stx2 = BOX(CHD_MTX2); stxty = BOX(CHD_MTXTY); sty2 = BOX(CHD_MTY2); stx = BOX(CHD_MTX);
      sty = BOX(CHD_MTY);
    }
    double stxz = BOX(CHD_TXW), styz = BOX(CHD_TYW), sinv = BOX(CHD_W), sinv2 = BOX(CHD_W2);
    double m[16] = {stx2, stxty, stx, stxz, stxty, sty2, sty, styz,
                    stx, sty, (double)n, sinv, stxz, styz, sinv, sinv2};
    memcpy(S, m, sizeof(m));
  }
#undef BOX
  return n;
}

/*
 * Per-pixel driver.  depth: H*W fp64 values (DepthImage.values); valid: H*W
 * bytes (DepthImage.valid); tan_x/tan_y: H*W fp64 (TanAngleMaps).  pix: optional
 * list of npix flat indices (NULL = every pixel, npix = H*W).  Outputs are
 * indexed by list position.  coef (4 per pixel) and lam are optional.
 * nthreads <= 0 uses every online core.  Returns 0, or -1 on bad arguments /
 * allocation failure.
 */
typedef struct {
  const double *depth, *tan_x, *tan_y;
  const uint8_t* valid;
  int H, W, r, formulation, backend;
  const sat_stack* st;
  const int64_t* pix;
  int64_t npix;
  float *normal, *offset, *residual, *curvature;
  uint8_t* status;
  double *coef, *lam, *scale, *curv_cond;
  atomic_llong next;
} job_t;

static void fit_one(job_t* J, int64_t k) {
  int W = J->W, H = J->H, r = J->r;
  int64_t idx = J->pix ? J->pix[k] : k;
  int y = (int)(idx / W), x = (int)(idx % W);
  int x0 = x - r < 0 ? 0 : x - r, y0 = y - r < 0 ? 0 : y - r;
  int x1 = x + r + 1 > W ? W : x + r + 1, y1 = y + r + 1 > H ? H : y + r + 1;
  uint8_t s = J->valid[idx] ? 1 : 0;
  double S[16];
  int n = 0;
  const int space = RFO_SPACE(J->formulation);
  const int explicit_fit = J->formulation >= RFO_EXPLICIT_STANDARD;
  const int min_samples = explicit_fit ? 3 : 4; /* MIN_SAMPLES fitting.py:55-60 */
  if (s) {
    n = J->backend == RFO_INTEGRAL
            ? integral_scatter(J->st, x0, y0, x1, y1, space, min_samples, S)
            : naive_scatter(J->depth, J->valid, J->tan_x, J->tan_y, W, x0, y0, x1, y1, space, S);
  }
  if (s && n >= min_samples) {
    fit_out o;
    if (explicit_fit) fit_explicit(S, n, space, &o);
    else fit_scatter(S, n, space, &o);
    if (o.failed) {
      s |= 8;
    } else {
      s |= 2;
      if (o.degenerate) s |= 4;
      double nn = sqrt(o.coef[0] * o.coef[0] + o.coef[1] * o.coef[1] + o.coef[2] * o.coef[2]);
      J->normal[3 * k + 0] = (float)(o.coef[0] / nn);
      J->normal[3 * k + 1] = (float)(o.coef[1] / nn);
      J->normal[3 * k + 2] = (float)(o.coef[2] / nn);
      J->offset[k] = (float)(o.coef[3] / nn);
      J->residual[k] = (float)o.rms;
      J->curvature[k] = (float)o.curvature;
      if (J->coef) memcpy(J->coef + 4 * k, o.coef, sizeof(o.coef));
      if (J->lam) J->lam[k] = o.lam;
      if (J->scale) J->scale[k] = o.scale;
      if (J->curv_cond) J->curv_cond[k] = o.curv_cond;
    }
  }
  if (!(s & 2)) {
    J->normal[3 * k + 0] = J->normal[3 * k + 1] = J->normal[3 * k + 2] = NAN;
    J->offset[k] = J->residual[k] = J->curvature[k] = NAN;
    if (J->coef) J->coef[4 * k] = J->coef[4 * k + 1] = J->coef[4 * k + 2] = J->coef[4 * k + 3] = NAN;
    if (J->lam) J->lam[k] = NAN;
    if (J->scale) J->scale[k] = NAN;
    if (J->curv_cond) J->curv_cond[k] = NAN;
  }
  J->status[k] = s;
}

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  const int64_t chunk = 256;
  for (;;) {
    int64_t b = atomic_fetch_add(&J->next, chunk);
    if (b >= J->npix) break;
    int64_t e = b + chunk < J->npix ? b + chunk : J->npix;
    for (int64_t k = b; k < e; ++k) fit_one(J, k);
  }
  return NULL;
}

int rfo_max_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

int rfo_fit_pixels(const double* depth, const uint8_t* valid, const double* tan_x,
                   const double* tan_y, int H, int W, int window, int formulation, int backend,
                   const int64_t* pix, int64_t npix, float* normal, float* offset, float* residual,
                   float* curvature, uint8_t* status, double* coef, double* lam, double* scale,
                   double* curv_cond, int nthreads) {
  if (window < 1 || (window & 1) == 0 || H <= 0 || W <= 0) return -1;
  if (formulation < RFO_STANDARD || formulation > RFO_EXPLICIT_RGBD) return -1;
  sat_stack st;
  st.t = NULL;
  if (backend == RFO_INTEGRAL) {
    if (build_stack(depth, valid, tan_x, tan_y, H, W, RFO_SPACE(formulation), &st) != 0) return -1;
  }
  job_t J = {depth, tan_x, tan_y, valid, H, W, window / 2, formulation, backend, &st, pix, npix,
             normal, offset, residual, curvature, status, coef, lam, scale, curv_cond, 0};
  atomic_init(&J.next, 0);
  if (nthreads <= 0) nthreads = rfo_max_threads();
  if (nthreads > 256) nthreads = 256;
  if (nthreads == 1 || npix < 4096) {
    worker(&J);
  } else {
    pthread_t th[256];
    int started = 0;
    for (int i = 0; i < nthreads; ++i)
      if (pthread_create(&th[started], NULL, worker, &J) == 0) ++started;
    if (started == 0) worker(&J);
    for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
  }
  free(st.t);
  return 0;
}

/*
 * Arbitrary rects: fit_rect(depth, maps, Rect(x0, y0, x1, y1), formulation, backend)
 * (fitting.py:757-786) for each of nrects rects (int32 x0, y0, x1, y1 each) of one frame.
 * status: bit1 fitted, bit2 degenerate, bit4 out of bounds (_check_rect raises).
 */
int rfo_fit_rects(const double* depth, const uint8_t* valid, const double* tan_x,
                  const double* tan_y, int H, int W, const int32_t* rects, int64_t nrects,
                  int formulation, int backend, double* coef, double* lam, double* rms,
                  double* curvature, int32_t* npts, int32_t* status) {
  if (formulation < RFO_STANDARD || formulation > RFO_EXPLICIT_RGBD) return -1;
  const int space = RFO_SPACE(formulation);
  const int explicit_fit = formulation >= RFO_EXPLICIT_STANDARD;
  const int min_samples = explicit_fit ? 3 : 4;
  sat_stack st;
  st.t = NULL;
  if (backend == RFO_INTEGRAL && build_stack(depth, valid, tan_x, tan_y, H, W, space, &st) != 0)
    return -1;
  for (int64_t k = 0; k < nrects; ++k) {
    const int x0 = rects[4 * k], y0 = rects[4 * k + 1], x1 = rects[4 * k + 2], y1 = rects[4 * k + 3];
    for (int i = 0; i < 4; ++i) coef[4 * k + i] = NAN;
    lam[k] = rms[k] = curvature[k] = NAN;
    npts[k] = 0;
    if (!(0 <= x0 && x0 <= x1 && x1 <= W && 0 <= y0 && y0 <= y1 && y1 <= H)) {
      status[k] = 16;
      continue;
    }
    double S[16];
    int n = backend == RFO_INTEGRAL ? integral_scatter(&st, x0, y0, x1, y1, space, min_samples, S)
                                    : naive_scatter(depth, valid, tan_x, tan_y, W, x0, y0, x1, y1, space, S);
    npts[k] = n;
    if (n < min_samples) { status[k] = 0; continue; }
    fit_out o;
    if (explicit_fit) fit_explicit(S, n, space, &o);
    else fit_scatter(S, n, space, &o);
    status[k] = 2 | (o.degenerate ? 4 : 0) | (o.failed ? 8 : 0);
    memcpy(coef + 4 * k, o.coef, sizeof(o.coef));
    lam[k] = o.lam;
    rms[k] = o.rms;
    curvature[k] = o.curvature;
  }
  free(st.t);
  return 0;
}

/* Single-window fit on a caller-supplied 4x4 scatter (for unit tests of the
 * restated Jacobi / canonicalisation).  Returns 0, or -1 if not converged. */
int rfo_fit_scatter(const double* S, int n, int formulation, double* coef, double* lam,
                    double* rms, double* curvature, int* degenerate) {
  fit_out o;
  if (formulation >= RFO_EXPLICIT_STANDARD) fit_explicit(S, n, RFO_SPACE(formulation), &o);
  else fit_scatter(S, n, formulation, &o);
  memcpy(coef, o.coef, sizeof(o.coef));
  *lam = o.lam;
  *rms = o.rms;
  *curvature = o.curvature;
  *degenerate = o.degenerate;
  return o.failed ? -1 : 0;
}

int rfo_jacobi_eigh(int n, const double* m, double* values, double* vectors) {
  if (n < 1 || n > 4) return -2;
  return jacobi_eigh(n, m, values, vectors);
}

