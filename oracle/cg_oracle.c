/*
 * cg_oracle.c — CPU ORACLE for the PERKS conjugate-gradient solver (NEXT-3).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this code.
 * It shares no code, header, table or helper with the CUDA path under
 * paper_2204_02064_b200/ (and neither side includes the other).
 *
 * What it computes (the plain definitions, in the paper's order and notation):
 *
 *   SpMV  y = A x, A in CSR ("A is stored in CSR format, includes value,
 *         column_indices and compressed row_offsets"):
 *           y_i = sum_{k = row_off[i]}^{row_off[i+1]-1} val[k] * x[col[k]]
 *         summed left to right in storage order, acc starting at +0, one fused
 *         multiply-add (one rounding) per term, in the storage dtype.
 *         (Merge-based SpMV, is an execution scheme for the same
 *         sum; reading RC1.)
 *
 *   CG    Algorithm "Conjugate Gradient Solver":
 *           x_0 = 0; r_0 = b; p_0 = b
 *           while k < k_max:
 *             alpha_k   = <r_k,r_k> / <p_k, A p_k>
 *             x_{k+1}   = x_k + alpha_k p_k
 *             r_{k+1}   = r_k - alpha_k A p_k
 *             beta_k    = <r_{k+1},r_{k+1}> / <r_k,r_k>
 *             p_{k+1}   = r_{k+1} + beta_k p_k
 *             stop when <r_{k+1},r_{k+1}> <= tol*tol
 *         Readings (RC2-RC4):
 *           RC2 the stopping test is evaluated before each iteration (so b = 0
 *               takes 0 iterations instead of dividing 0 by 0); tol = 0 runs
 *               k_max iterations unless <r,r> reaches exactly 0.
 *           RC3 vectors and matrix in the storage dtype T; every inner product
 *               <u,v> accumulated in double, left to right, one fma per term
 *               on the double-converted operands; alpha, beta and <r,r> kept in
 *               double; each vector update is one fma in T with the scalar
 *               rounded to T once:  x = fma((T)alpha, p, x),
 *               r = fma(-(T)alpha, q, r),  p = fma((T)beta, p, r).
 *           RC4 <p, A p> <= 0 with <r,r> > 0 means A is not positive definite:
 *               error ORACLE_NOT_SPD (the iteration count so far is returned).
 *
 * Build: gcc -O2 -mfma -ffp-contract=off -fopenmp -shared -fPIC (no -ffast-math).
 * Single-threaded except the SpMV row loop (rows are independent; per-row
 * arithmetic does not depend on the schedule, so results are identical for any
 * thread count).  Inner products are sequential.
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
#define ORACLE_OOM 3
#define ORACLE_NOT_SPD 4

static int check_csr(int64_t n, const int64_t *row_off, const int32_t *col) {
  if (n < 0 || !row_off || (n > 0 && !col)) return ORACLE_INVALID_ARGUMENT;
  if (row_off[0] != 0) return ORACLE_INVALID_ARGUMENT;
  for (int64_t i = 0; i < n; i++) {
    if (row_off[i + 1] < row_off[i]) return ORACLE_INVALID_ARGUMENT;
    for (int64_t k = row_off[i]; k < row_off[i + 1]; k++)
      if (col[k] < 0 || col[k] >= n) return ORACLE_INVALID_ARGUMENT;
  }
  return ORACLE_OK;
}

/* ------------------------------------------------------------------ SpMV */

static void spmv_f64(int64_t n, const int64_t *row_off, const int32_t *col,
                     const double *val, const double *x, double *y) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; i++) {
    double acc = 0.0;
    for (int64_t k = row_off[i]; k < row_off[i + 1]; k++)
      acc = fma(val[k], x[col[k]], acc);
    y[i] = acc;
  }
}

static void spmv_f32(int64_t n, const int64_t *row_off, const int32_t *col,
                     const float *val, const float *x, float *y) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; i++) {
    float acc = 0.0f;
    for (int64_t k = row_off[i]; k < row_off[i + 1]; k++)
      acc = fmaf(val[k], x[col[k]], acc);
    y[i] = acc;
  }
}

int oracle_csr_spmv_f64(int64_t n, const int64_t *row_off, const int32_t *col,
                        const double *val, const double *x, double *y, int nthreads) {
  int st = check_csr(n, row_off, col);
  if (st) return st;
  if (n > 0 && (!x || !y || (row_off[n] > 0 && !val))) return ORACLE_INVALID_ARGUMENT;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  spmv_f64(n, row_off, col, val, x, y);
  return ORACLE_OK;
}

int oracle_csr_spmv_f32(int64_t n, const int64_t *row_off, const int32_t *col,
                        const float *val, const float *x, float *y, int nthreads) {
  int st = check_csr(n, row_off, col);
  if (st) return st;
  if (n > 0 && (!x || !y || (row_off[n] > 0 && !val))) return ORACLE_INVALID_ARGUMENT;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  spmv_f32(n, row_off, col, val, x, y);
  return ORACLE_OK;
}

/* ------------------------------------------------------------- inner products
 * RC3: accumulated in double, left to right, one fma per term. */

static double dot_f64(int64_t n, const double *u, const double *v) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; i++) acc = fma(u[i], v[i], acc);
  return acc;
}

static double dot_f32(int64_t n, const float *u, const float *v) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; i++) acc = fma((double)u[i], (double)v[i], acc);
  return acc;
}

/* ------------------------------------------------------------------- CG
 * Algorithm P:244-258 (see header).  x_out: n values (x_k on return);
 * rr_hist (nullable): k_max+1 doubles, rr_hist[k] = <r_k,r_k> for k = 0..iters,
 * the rest left untouched; iters: iterations performed. */

int oracle_cg_f64(int64_t n, const int64_t *row_off, const int32_t *col,
                  const double *val, const double *b, int64_t kmax, double tol,
                  double *x_out, double *rr_hist, int64_t *iters, int nthreads) {
  int st = check_csr(n, row_off, col);
  if (st) return st;
  if (kmax < 0 || !(tol >= 0.0) || !x_out || !iters || (n > 0 && !b))
    return ORACLE_INVALID_ARGUMENT;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  double *x = x_out;
  double *r = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double *p = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double *q = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  if (!r || !p || !q) { free(r); free(p); free(q); return ORACLE_OOM; }
  for (int64_t i = 0; i < n; i++) { x[i] = 0.0; r[i] = b[i]; p[i] = b[i]; }  /* x0=0, r0=p0=b */
  double rr = dot_f64(n, r, r);
  if (rr_hist) rr_hist[0] = rr;
  int64_t k = 0;
  st = ORACLE_OK;
  while (k < kmax) {
    if (rr <= tol * tol) break;                                   /* RC2 */
    spmv_f64(n, row_off, col, val, p, q);                         /* q = A p_k */
    const double pAp = dot_f64(n, p, q);
    if (!(pAp > 0.0)) { st = ORACLE_NOT_SPD; break; }             /* RC4 */
    const double alpha = rr / pAp;
    const double a = alpha;                                       /* (T)alpha, T = double */
    for (int64_t i = 0; i < n; i++) x[i] = fma(a, p[i], x[i]);    /* x_{k+1} */
    for (int64_t i = 0; i < n; i++) r[i] = fma(-a, q[i], r[i]);   /* r_{k+1} */
    const double rr_new = dot_f64(n, r, r);
    const double beta = rr_new / rr;
    for (int64_t i = 0; i < n; i++) p[i] = fma(beta, p[i], r[i]); /* p_{k+1} */
    rr = rr_new;
    k++;
    if (rr_hist) rr_hist[k] = rr;
  }
  *iters = k;
  free(r); free(p); free(q);
  return st;
}

int oracle_cg_f32(int64_t n, const int64_t *row_off, const int32_t *col,
                  const float *val, const float *b, int64_t kmax, double tol,
                  float *x_out, double *rr_hist, int64_t *iters, int nthreads) {
  int st = check_csr(n, row_off, col);
  if (st) return st;
  if (kmax < 0 || !(tol >= 0.0) || !x_out || !iters || (n > 0 && !b))
    return ORACLE_INVALID_ARGUMENT;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  float *x = x_out;
  float *r = (float *)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  float *p = (float *)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  float *q = (float *)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  if (!r || !p || !q) { free(r); free(p); free(q); return ORACLE_OOM; }
  for (int64_t i = 0; i < n; i++) { x[i] = 0.0f; r[i] = b[i]; p[i] = b[i]; }
  double rr = dot_f32(n, r, r);
  if (rr_hist) rr_hist[0] = rr;
  int64_t k = 0;
  st = ORACLE_OK;
  while (k < kmax) {
    if (rr <= tol * tol) break;
    spmv_f32(n, row_off, col, val, p, q);
    const double pAp = dot_f32(n, p, q);
    if (!(pAp > 0.0)) { st = ORACLE_NOT_SPD; break; }
    const double alpha = rr / pAp;
    const float a = (float)alpha;                                 /* rounded to T once */
    for (int64_t i = 0; i < n; i++) x[i] = fmaf(a, p[i], x[i]);
    for (int64_t i = 0; i < n; i++) r[i] = fmaf(-a, q[i], r[i]);
    const double rr_new = dot_f32(n, r, r);
    const double beta = rr_new / rr;
    const float bt = (float)beta;
    for (int64_t i = 0; i < n; i++) p[i] = fmaf(bt, p[i], r[i]);
    rr = rr_new;
    k++;
    if (rr_hist) rr_hist[k] = rr;
  }
  *iters = k;
  free(r); free(p); free(q);
  return st;
}
