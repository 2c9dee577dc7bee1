/*
 * perks_cg.h — C ABI of the PERKS conjugate-gradient solver, part of
 * libperks_stencil.so.
 *
 * What the library computes (PAPER.md = /root/reference/PAPER.md, arXiv 2204.02064):
 *   the conjugate-gradient Algorithm "Conjugate Gradient Solver" on a symmetric
 *   positive-definite matrix A in CSR (value, column_indices, row_offsets):
 *       x_0 = 0, r_0 = p_0 = b;  alpha_k = <r_k,r_k>/<p_k,A p_k>;  x_{k+1} = x_k + alpha_k p_k;
 *       r_{k+1} = r_k - alpha_k A p_k;  beta_k = <r_{k+1},r_{k+1}>/<r_k,r_k>;
 *       p_{k+1} = r_{k+1} + beta_k p_k;  stop when <r,r> <= tol^2 (tested before each
 *       iteration, reading RC2) or after k_max iterations.
 *   Arithmetic (reading RC3): matrix and vectors in the storage dtype; inner products
 *   accumulated in double; alpha, beta, <r,r> in double; each vector update one fma in the
 *   dtype with the scalar rounded to the dtype once.
 * How (the execution variants, as for the stencil library):
 *   PERKS_HOSTLOOP   (a) two kernel launches per iteration (SpMV + <p,Ap>; updates + <r,r>);
 *   PERKS_PERSISTENT (b) one cooperative launch, the iteration loop inside the kernel with two
 *                        device-wide barriers per iteration, nothing cached explicitly
 *                        (the paper's IMP policy);
 *   PERKS_PERKS      (c) (b) plus the cache policy: VEC keeps each CTA's own rows of r, x, p
 *                        and A p in shared memory, MAT keeps the CTA's matrix tiles resident in
 *                        Tensor Memory and shared memory across iterations, MIX both
 *                        (P:1749-1766).
 * SpMV is merge-based: each CTA owns a row-aligned share of the merge path of
 * (row ends, nonzeros) (the "TB-level search", done once at create and kept in device memory);
 * inside a CTA the share's nonzeros are cut into tiles of NT*IPT items, each thread owning IPT
 * consecutive items (the "thread-level search", also done once at create: the library stores
 * the matrix in this thread-interleaved item layout, with row-end marks and per-thread headers).
 * MAT keeps the first tiles of each CTA in Tensor Memory and shared memory across iterations.
 * All variants and policies use the same partition and the same reduction order, so they are
 * bit-identical to one another (checked by the tests); against the oracle they agree within the
 * rounding bound of a reordered sum (RC1).
 *
 * Conventions: as perks_stencil.h (extern "C", perks_status returns, stream-ordered and
 * asynchronous, the caller owns every device buffer it passes; the library owns its copy of
 * the matrix and the partition).
 */
#ifndef PERKS_CG_H
#define PERKS_CG_H

#include <stddef.h>
#include <stdint.h>

#include "perks_stencil.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PERKS_CG_AUTO = 0, /* MIX                                                                   */
  PERKS_CG_IMP = 1,  /* nothing cached explicitly (L2 only)                                   */
  PERKS_CG_VEC = 2,  /* own rows of r, x, p, Ap in shared memory                              */
  PERKS_CG_MAT = 3,  /* matrix tiles resident in Tensor Memory + shared memory, rest streamed */
  PERKS_CG_MIX = 4   /* VEC + MAT                                                            */
} perks_cg_policy;

/* CSR matrix (host arrays, copied at create; the caller may free them afterwards).
 *   row_offsets: n_rows+1 non-decreasing int64, row_offsets[0] = 0, row_offsets[n_rows] = nnz;
 *   col_indices: nnz int32 in [0, n_rows); values: nnz doubles, rounded ONCE to dtype at create.
 * Square only (CG).  Symmetry and definiteness are not checked here: a breakdown
 * (<p, A p> <= 0) is reported by solve through d_info[1] = 1. */
typedef struct {
  int64_t n_rows;
  int64_t nnz;
  const int64_t *row_offsets;
  const int32_t *col_indices;
  const double *values;
  perks_dtype dtype;
} perks_csr_desc;

typedef struct perks_cg_s *perks_cg_t;

typedef struct {
  int32_t variant;            /* resolved variant                                             */
  int32_t policy;             /* resolved cache policy (never PERKS_CG_AUTO)                  */
  int32_t grid;               /* CTAs (the merge-path partition count)                        */
  int32_t block;              /* threads per CTA                                              */
  int32_t items_per_thread;   /* merge-path items per thread per tile (IPT)                   */
  int32_t tiles;              /* tiles over all CTAs                                          */
  int32_t smem_per_cta;       /* dynamic shared memory bytes                                  */
  int32_t regs_per_thread;
  int64_t cached_nnz_smem;    /* item slots (nonzeros) resident in shared memory (MAT)        */
  int64_t cached_rows_smem;   /* vector rows resident in shared memory (VEC; r, x, p, Ap each) */
  int64_t n_rows, nnz;
  double dram_bytes_per_iter; /* modelled DRAM bytes per iteration (CG rows)    */
  double unfused_bytes_per_iter; /* algorithmic bytes of one unfused iteration (the metric)   */
  size_t workspace_bytes;
  char kernel_name[64];
  int64_t cached_nnz_tmem;    /* item slots resident in Tensor Memory across iterations (MAT) */
  int32_t tmem_tiles_per_cta; /* resident tiles per CTA: Tensor Memory, shared memory          */
  int32_t smem_tiles_per_cta;
} perks_cg_info;

/* Validates the CSR (INVALID_ARGUMENT on bad offsets or column indices; UNSUPPORTED when nnz or
 * n_rows exceed 2^31-1), copies it to the device, and computes the merge-path partition. */
perks_status perks_cg_create(const perks_csr_desc *desc, int device, perks_cg_t *out);

/* Device workspace for solve/spmv (256-B aligned, caller-allocated): r, two p buffers, A p,
 * reduction slots and barrier words. */
perks_status perks_cg_workspace_bytes(perks_cg_t h, size_t *bytes);

/* y = A x with the merge-based SpMV kernel (one launch).  d_x, d_y: device, n_rows values of
 * the handle's dtype, not overlapping. */
perks_status perks_cg_spmv(perks_cg_t h, const void *d_x, void *d_y, void *d_workspace,
                           size_t workspace_bytes, void *stream);

/* Run CG from x_0 = 0 for at most k_max iterations (tol = 0: exactly k_max unless <r,r> hits 0).
 *   d_b: device, n_rows values (read only);  d_x: device, n_rows values (x_k on completion);
 *   d_rr_history: device, nullable, k_max+1 doubles: [k] = <r_k,r_k> for k = 0..iterations
 *   (entries past the last iteration are not written);
 *   d_info: device, nullable, 2 int64: [0] = iterations performed, [1] = 0 ok / 1 breakdown.
 * Asynchronous like perks_stencil_run; persistent variants must not overlap on one device. */
perks_status perks_cg_solve(perks_cg_t h, perks_variant variant, perks_cg_policy policy,
                            const void *d_b, void *d_x, int64_t k_max, double tol,
                            double *d_rr_history, int64_t *d_info, void *d_workspace,
                            size_t workspace_bytes, void *stream);

/* End-to-end: host b in, host x (and nullable host history / info) out: copies b to device
 * scratch, solves, copies back, synchronises.  Blocking.  The device scratch and a private stream
 * are kept in the handle across calls (grown on demand, freed by destroy); calls on one handle
 * are serialised. */
perks_status perks_cg_solve_host(perks_cg_t h, perks_variant variant, perks_cg_policy policy,
                                 const void *h_b, void *h_x, int64_t k_max, double tol,
                                 double *h_rr_history, int64_t *h_info);

perks_status perks_cg_query(perks_cg_t h, perks_variant variant, perks_cg_policy policy,
                            perks_cg_info *info);

/* The CTA-level (TB-level) merge-path partition: first row of each CTA, grid+1 values
 * (row-aligned; the last is n_rows).  cap = capacity of h_rows in elements. */
perks_status perks_cg_partition(perks_cg_t h, int64_t *h_rows, int32_t cap);

perks_status perks_cg_destroy(perks_cg_t h);

#ifdef __cplusplus
}
#endif
#endif /* PERKS_CG_H */
