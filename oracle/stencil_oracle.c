/*
 * stencil_oracle.c — CPU ORACLE for the PERKS stencil time loop.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this code.
 * It shares no code, header, table or helper with the CUDA path under
 * paper_2204_02064_b200/ (and neither side includes the other).
 *
 * What it computes (the plain definition; PERKS is an execution scheme that
 * "does not touch on the compute part"):
 *
 *   x^{k+1} = F(x^k)                                    (Eq. iterative)
 *   x(c)^{k+1} = sum_p w_p * x(c + d_p)^k               (Eq. iterativeStencil;
 *                                                        2d5pt: N,S,C,W,E terms)
 *
 * applied T times out of place (Jacobi: step k+1 reads only step-k values,
 * P:191).  Readings of the paper:
 *   R1 boundary: FRAME = cells within r of any face are never updated and keep
 *      their input value bit-exactly; PERIODIC = every cell updated, indices wrap.
 *   R4 layout: C order [z][y][x], x unit stride; offsets are (dx,dy,dz).
 *   R5 accumulation order = the list order of the points: the first term is a
 *      single rounded multiply, every later term one fused multiply-add
 *      (C99 fma/fmaf: one rounding).  No reassociation.
 *   R6 arithmetic in the storage dtype; the weights passed in are already
 *      rounded to that dtype by the caller.
 *   R8 T = 0 returns the input; the result is x^T for any parity of T.
 *   R9 any active extent < 2r+1 -> error ORACLE_INVALID_DOMAIN.
 *
 * Build: gcc -O2 -mfma -ffp-contract=off -fopenmp -shared -fPIC (no -ffast-math).
 * The OpenMP mode parallelises over (z,y) rows only; each cell's arithmetic is
 * independent of the schedule, so results are identical for any thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_INVALID_ARGUMENT 1
#define ORACLE_INVALID_DOMAIN 2
#define ORACLE_OOM 3

#define ORACLE_BC_FRAME 0
#define ORACLE_BC_PERIODIC 1

static int64_t wrap(int64_t i, int64_t n) {
  int64_t m = i % n;
  return m < 0 ? m + n : m;
}

static int check_args(int ndim, const int64_t ext[3], int npts,
                      const int32_t *offsets, int bc, int64_t T, int *radius) {
  if (ndim != 2 && ndim != 3) return ORACLE_INVALID_ARGUMENT;
  if (npts < 1 || !offsets || T < 0) return ORACLE_INVALID_ARGUMENT;
  if (bc != ORACLE_BC_FRAME && bc != ORACLE_BC_PERIODIC) return ORACLE_INVALID_ARGUMENT;
  if (ndim == 2 && ext[2] != 1) return ORACLE_INVALID_DOMAIN;
  int r = 0;
  for (int p = 0; p < npts; p++) {
    for (int a = 0; a < 3; a++) {
      int d = offsets[3 * p + a];
      if (a >= ndim && d != 0) return ORACLE_INVALID_ARGUMENT;
      if (abs(d) > r) r = abs(d);
    }
  }
  for (int a = 0; a < ndim; a++)
    if (ext[a] < 2 * r + 1) return ORACLE_INVALID_DOMAIN;
  *radius = r;
  return ORACLE_OK;
}

/* One generic body per dtype, written out twice so each reads plainly. */

int oracle_stencil_f64(int ndim, const int64_t ext[3], int npts, const int32_t *offsets,
                       const double *weights, int bc, int64_t T, const double *in,
                       double *out, int nthreads) {
  int r = 0;
  int st = check_args(ndim, ext, npts, offsets, bc, T, &r);
  if (st != ORACLE_OK) return st;
  if (!in || !out || !weights) return ORACLE_INVALID_ARGUMENT;
  const int64_t nx = ext[0], ny = ext[1], nz = ext[2];
  const int64_t ncell = nx * ny * nz;
  double *a = (double *)malloc(sizeof(double) * (size_t)ncell);
  double *b = (double *)malloc(sizeof(double) * (size_t)ncell);
  if (!a || !b) { free(a); free(b); return ORACLE_OOM; }
  /* b starts as a copy too, so FRAME cells hold their input in both buffers. */
  memcpy(a, in, sizeof(double) * (size_t)ncell);
  memcpy(b, in, sizeof(double) * (size_t)ncell);
  /* the update set U: FRAME -> [r, n-r) on active axes; PERIODIC -> all */
  const int64_t zlo = (ndim == 3 && bc == ORACLE_BC_FRAME) ? r : 0;
  const int64_t zhi = (ndim == 3 && bc == ORACLE_BC_FRAME) ? nz - r : nz;
  const int64_t ylo = (bc == ORACLE_BC_FRAME) ? r : 0, yhi = (bc == ORACLE_BC_FRAME) ? ny - r : ny;
  const int64_t xlo = (bc == ORACLE_BC_FRAME) ? r : 0, xhi = (bc == ORACLE_BC_FRAME) ? nx - r : nx;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  for (int64_t k = 0; k < T; k++) {
    const int64_t nrows = (zhi - zlo) * (yhi - ylo);
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < nrows; row++) {
      const int64_t z = zlo + row / (yhi - ylo);
      const int64_t y = ylo + row % (yhi - ylo);
      for (int64_t x = xlo; x < xhi; x++) {
        double acc = 0.0;
        for (int p = 0; p < npts; p++) {
          int64_t qx = x + offsets[3 * p + 0];
          int64_t qy = y + offsets[3 * p + 1];
          int64_t qz = z + offsets[3 * p + 2];
          if (bc == ORACLE_BC_PERIODIC) {
            qx = wrap(qx, nx); qy = wrap(qy, ny); qz = wrap(qz, nz);
          }
          const double v = a[(qz * ny + qy) * nx + qx];
          if (p == 0) acc = weights[0] * v;            /* one rounding */
          else acc = fma(weights[p], v, acc);           /* one rounding */
        }
        b[(z * ny + y) * nx + x] = acc;
      }
    }
    double *t = a; a = b; b = t;
  }
  memcpy(out, a, sizeof(double) * (size_t)ncell);
  free(a); free(b);
  return ORACLE_OK;
}

int oracle_stencil_f32(int ndim, const int64_t ext[3], int npts, const int32_t *offsets,
                       const float *weights, int bc, int64_t T, const float *in,
                       float *out, int nthreads) {
  int r = 0;
  int st = check_args(ndim, ext, npts, offsets, bc, T, &r);
  if (st != ORACLE_OK) return st;
  if (!in || !out || !weights) return ORACLE_INVALID_ARGUMENT;
  const int64_t nx = ext[0], ny = ext[1], nz = ext[2];
  const int64_t ncell = nx * ny * nz;
  float *a = (float *)malloc(sizeof(float) * (size_t)ncell);
  float *b = (float *)malloc(sizeof(float) * (size_t)ncell);
  if (!a || !b) { free(a); free(b); return ORACLE_OOM; }
  memcpy(a, in, sizeof(float) * (size_t)ncell);
  memcpy(b, in, sizeof(float) * (size_t)ncell);
  const int64_t zlo = (ndim == 3 && bc == ORACLE_BC_FRAME) ? r : 0;
  const int64_t zhi = (ndim == 3 && bc == ORACLE_BC_FRAME) ? nz - r : nz;
  const int64_t ylo = (bc == ORACLE_BC_FRAME) ? r : 0, yhi = (bc == ORACLE_BC_FRAME) ? ny - r : ny;
  const int64_t xlo = (bc == ORACLE_BC_FRAME) ? r : 0, xhi = (bc == ORACLE_BC_FRAME) ? nx - r : nx;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  for (int64_t k = 0; k < T; k++) {
    const int64_t nrows = (zhi - zlo) * (yhi - ylo);
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < nrows; row++) {
      const int64_t z = zlo + row / (yhi - ylo);
      const int64_t y = ylo + row % (yhi - ylo);
      for (int64_t x = xlo; x < xhi; x++) {
        float acc = 0.0f;
        for (int p = 0; p < npts; p++) {
          int64_t qx = x + offsets[3 * p + 0];
          int64_t qy = y + offsets[3 * p + 1];
          int64_t qz = z + offsets[3 * p + 2];
          if (bc == ORACLE_BC_PERIODIC) {
            qx = wrap(qx, nx); qy = wrap(qy, ny); qz = wrap(qz, nz);
          }
          const float v = a[(qz * ny + qy) * nx + qx];
          if (p == 0) acc = weights[0] * v;
          else acc = fmaf(weights[p], v, acc);
        }
        b[(z * ny + y) * nx + x] = acc;
      }
    }
    float *t = a; a = b; b = t;
  }
  memcpy(out, a, sizeof(float) * (size_t)ncell);
  free(a); free(b);
  return ORACLE_OK;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
