// cg.cu — PERKS conjugate gradient (include/perks/perks_cg.h).
//
// The paper's second case study: CG (Algorithm) with a
// merge-based SpMV, run (a) as a host loop of kernels, (b) as one persistent
// kernel with device-wide barriers, (c) as PERKS with the cache policies IMP / VEC / MAT / MIX
// (P:1749-1766).  B200 design (DESIGN.md §5 "CG"):
//
//   * Partition.  Merge path of (row ends, nonzeros) (length n + nnz).  CTA c owns a row-aligned
//     share [R_c, R_{c+1}) (the CTA-level search, done once on the host at create and kept in
//     device memory — "We save the search result of thread block workloads in global memory",
//     P:1123).  Row-aligned shares need no cross-CTA carry, so A p for a CTA's own rows is
//     complete inside the CTA and never leaves the SM.  The share is cut into tiles of NT*IPT
//     path items (tile start coordinates also precomputed).
//   * Tile = three contiguous CSR ranges (row offsets, column indices, values) moved into shared
//     memory by 1D bulk copies (cp.async.bulk, mbarrier completion), double buffered; MAT keeps
//     the first tiles of each CTA resident in shared memory for the whole solve instead.
//   * SpMV of a tile: phase 1, coalesced over the tile's nonzeros, prod[k] = val[k] * p[col[k]]
//     (independent gathers, full memory-level parallelism); phase 2, each thread finds its slice
//     of the tile's merge path by a binary search in shared memory (the "thread-level search",
//     P:1123) and sums products row by row; rows split between threads (or tiles) are combined
//     from the per-thread carries in thread order — a fixed order, so every launch, variant and
//     policy produces the same bits.
//   * Two device-wide barriers per iteration instead of three: p_k of OTHER CTAs' rows is never
//     read from memory during the SpMV; it is recomputed at the gather as fma(beta, p_{k-1}, r_k)
//     from the published r_k and p_{k-1} (the owner computes its own rows with the same fma, so
//     the values are identical).  p is double-buffered by iteration parity.
//   * Inner products: per-thread fma chains in double over the CTA's own rows, a fixed
//     xor-butterfly per warp and across warps, one partial per CTA in a slot; after the barrier
//     every CTA sums the slots in the same fixed order (no atomics; deterministic).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/perks/perks_cg.h"
#include "internal.h"
#include "stream3d.cuh"

namespace perks {
namespace cg {

constexpr int NT = 512;       // threads per CTA (16 warps; one CTA per SM)
constexpr int IPT = 6;        // merge-path items per thread per tile
constexpr int TILE = NT * IPT;
constexpr int kSmemMax = 227 * 1024;

// ------------------------------------------------------------------ tile geometry (host+device)
// A tile covers path items [(i0,k0), (i1,k1)): rows_t = i1 - i0 completions, nnz_t = k1 - k0.
// Shared-memory image: row_off[i0 - sro .. i1] | col[k0 - sc .. k1) | val[k0 - sv .. k1), each
// part a 16-byte multiple starting 16-byte aligned (bulk copies need 16-B aligned addresses and
// sizes); the shifts s* (< 16 bytes) absorb the misalignment of the global source.
__host__ __device__ inline int a16(long long b) { return (int)((b + 15) & ~15ll); }
template <typename T> struct TileGeo {
  int sro, sc, sv;          // element shifts
  int ro_b, col_b, val_b;   // copy bytes (16-multiples; 0 if nothing to copy)
  __host__ __device__ TileGeo(int i0, int rows_t, int k0, int nnz_t) {
    sro = i0 & 3;
    sc = k0 & 3;
    sv = k0 & (16 / (int)sizeof(T) - 1);
    ro_b = a16((long long)(rows_t + 1 + sro) * 4);
    col_b = nnz_t ? a16((long long)(nnz_t + sc) * 4) : 0;
    val_b = nnz_t ? a16((long long)(nnz_t + sv) * (int)sizeof(T)) : 0;
  }
  __host__ __device__ int bytes() const { return ro_b + col_b + val_b; }
};
// Upper bound of any tile's image (rows_t + nnz_t <= TILE).
template <typename T> constexpr int tile_max_bytes() {
  return ((TILE + 1 + 3) * 4 + 15) / 16 * 16 + ((TILE + 3) * 4 + 15) / 16 * 16 +
         ((TILE + 16 / (int)sizeof(T) - 1) * (int)sizeof(T) + 15) / 16 * 16;
}

template <typename T> struct Params {
  int n, G;
  const int *row_off;     // n+1 (+pad)
  const int *col;         // nnz (+pad)
  const T *val;           // nnz (+pad)
  const int2 *coords;     // tile start coordinates (row, nnz); CTA c: coords[ctile[c] .. ctile[c+1]-1]
  const int *ctile;       //   (its last entry is the CTA's end coordinate)
  const int *crow;        // G+1 row boundaries
  const T *b;
  T *x;                   // output
  T *r, *p0, *p1, *q;     // workspace vectors (global)
  const T *xin;           // spmv: input vector (output in q)
  double *slots;          // 2*G partial sums
  double *scal;           // host loop: <r,r> by iteration parity [2]
  long long *state;       // host loop: [0] done, [1] iterations, [2] status
  unsigned *bar;          // grid barrier words
  double *hist;           // nullable, kmax+1
  long long *info;        // nullable, 2
  long long kmax;
  double tol2;
  int rows_max;           // max own rows over CTAs (VEC arrays)
  int res_budget;         // bytes of resident-tile region (MAT); 0 = stream everything
  int stream;             // 1 if this launch streams tiles (double buffer present)
};

// Dynamic shared memory layout.
struct Smem {
  static constexpr int RED = 0;                       // 32 doubles
  static constexpr int MBAR = RED + 32 * 8;           // 3 mbarriers (2 stream + 1 resident)
  static constexpr int TCAR = MBAR + 32;              // tile carries [2]: valid + value (16 B each)
  static constexpr int BCAST = TCAR + 32;             // reduction broadcasts [4] (doubles)
  static constexpr int CROW = BCAST + 32;             // NT ints
  static constexpr int CVAL = CROW + NT * 4;          // NT doubles (T)
  static constexpr int PROD = CVAL + NT * 8;          // TILE values
  template <typename T> static constexpr int vec_off() { return PROD + TILE * (int)sizeof(T); }
};
template <typename T> inline int smem_bytes(int vec_rows, bool stream, int res_budget) {
  int b = Smem::vec_off<T>() + 4 * a16((long long)vec_rows * (int)sizeof(T));
  if (stream) b += 2 * tile_max_bytes<T>();
  return b + res_budget;
}

// ------------------------------------------------------------------------ reductions
PERKS_DEVINL double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // identical in every lane (IEEE addition is commutative)
}
// Sum of one double per thread, fixed order; every thread gets the same value.
PERKS_DEVINL double block_sum(double v, double *s_red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) s_red[w] = v;
  __syncthreads();
  double t = lane < NT / 32 ? s_red[lane] : 0.0;
  t = warp_sum(t);
  __syncthreads();
  return t;
}
// Sum of the G slot partials (written by other CTAs before a grid barrier), fixed order.  One
// warp reads the slots (all loads in flight together; lane l sums slots l, l+32, ... in order),
// reduces, and broadcasts through shared memory — every thread gets the same value.
constexpr int kMaxG = 256;
PERKS_DEVINL double slots_sum(const double *slots, int G, double *s_bc) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double v[kMaxG / 32];
#pragma unroll
    for (int j = 0; j < kMaxG / 32; ++j) v[j] = lane + 32 * j < G ? __ldcg(slots + lane + 32 * j) : 0.0;
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < kMaxG / 32; ++j) t += v[j];
    t = warp_sum(t);
    if (lane == 0) *s_bc = t;
  }
  __syncthreads();
  return *s_bc;
}

// ------------------------------------------------------------------------ tile pipeline
template <typename T> struct TileView {
  const int *ro;   // ro[m] = row_off[i0 + m], m = 0..rows_t
  const int *col;  // col[e] = col[k0 + e]
  const T *val;
  int i0, k0, rows_t, nnz_t;
};

template <typename T>
PERKS_DEVINL TileView<T> tile_view(unsigned char *base, int i0, int k0, int rows_t, int nnz_t) {
  const TileGeo<T> g(i0, rows_t, k0, nnz_t);
  TileView<T> v;
  v.ro = reinterpret_cast<const int *>(base) + g.sro;
  v.col = reinterpret_cast<const int *>(base + g.ro_b) + g.sc;
  v.val = reinterpret_cast<const T *>(base + g.ro_b + g.col_b) + g.sv;
  v.i0 = i0; v.k0 = k0; v.rows_t = rows_t; v.nnz_t = nnz_t;
  return v;
}

// One thread: bulk copies of a tile image into `dst`, completing on `mb` (expect_tx included).
template <typename T>
PERKS_DEVINL void issue_tile(const Params<T> &P, unsigned char *dst, int i0, int k0, int rows_t, int nnz_t,
                             uint64_t *mb, bool arm = true) {
  const TileGeo<T> g(i0, rows_t, k0, nnz_t);
  if (arm) mbar_arrive_tx(mb, (unsigned)g.bytes());
  bulk_load(dst, P.row_off + (i0 - g.sro), (unsigned)g.ro_b, mb);
  if (nnz_t) {
    bulk_load(dst + g.ro_b, P.col + (k0 - g.sc), (unsigned)g.col_b, mb);
    bulk_load(dst + g.ro_b + g.col_b, P.val + (k0 - g.sv), (unsigned)g.val_b, mb);
  }
}

// Tile carry between consecutive tiles of one CTA (the partial sum of the row a tile ends in).
template <typename T> struct TileCarry {
  int valid;
  int pad;
  T val;
};

// SpMV of one tile (see the header comment).  gather(j) returns the vector value at column j;
// qstore(row, v) stores a completed row.  Ends with __syncthreads.
// The tile carry is double buffered by tile parity (read tc[par], write tc[par ^ 1]) so the
// writer of the next carry never races the readers of this one.
template <typename T, class Gather, class QStore>
PERKS_DEVINL void tile_spmv(const TileView<T> &t, unsigned char *smem, int par, bool last, Gather gather,
                            QStore qstore) {
  T *s_prod = reinterpret_cast<T *>(smem + Smem::PROD);
  int *s_crow = reinterpret_cast<int *>(smem + Smem::CROW);
  T *s_cval = reinterpret_cast<T *>(smem + Smem::CVAL);
  const TileCarry<T> *tc = reinterpret_cast<TileCarry<T> *>(smem + Smem::TCAR) + par;
  TileCarry<T> *tn = reinterpret_cast<TileCarry<T> *>(smem + Smem::TCAR) + (par ^ 1);
  const int tid = threadIdx.x;
  // phase 1: products, coalesced over the nonzeros; all IPT gathers of a thread in flight at once
  {
    int cj[IPT];
    T vj[IPT], gj[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const int e = tid + j * NT;
      cj[j] = e < t.nnz_t ? t.col[e] : -1;
      vj[j] = e < t.nnz_t ? t.val[e] : T(0);
    }
#pragma unroll
    for (int j = 0; j < IPT; ++j) gj[j] = cj[j] >= 0 ? gather(cj[j]) : T(0);
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const int e = tid + j * NT;
      if (e < t.nnz_t) s_prod[e] = mul_rn(vj[j], gj[j]);
    }
  }
  __syncthreads();
  // phase 2: thread-level merge-path search + row sums
  const int items = t.rows_t + t.nnz_t;
  const int ipt = (items + NT - 1) / NT;
  int d = min(tid * ipt, items);
  const int dend = min(d + ipt, items);
  int lo = max(0, d - t.nnz_t), hi = min(d, t.rows_t);
  while (lo < hi) {  // rows completed before diagonal d: row m ends (ro[m+1]-k0) at or before nnz d-1-m
    const int mid = (lo + hi) >> 1;
    if (t.ro[mid + 1] - t.k0 <= d - 1 - mid) lo = mid + 1;
    else hi = mid;
  }
  int i = lo, k = d - lo;
  bool pending = (k + t.k0 > t.ro[i]);  // row i0+i already has terms before this thread's slice
  T acc = T(0), sval = T(0);
  int srow = -1;
  for (; d < dend; ++d) {
    if (i < t.rows_t && k + t.k0 >= t.ro[i + 1]) {  // row i complete
      if (pending) { srow = i; sval = acc; pending = false; }
      else qstore(t.i0 + i, acc);
      acc = T(0);
      ++i;
    } else {
      acc = acc + s_prod[k];
      ++k;
    }
  }
  s_crow[tid] = i;
  s_cval[tid] = acc;
  __syncthreads();
  if (srow >= 0) {  // first completed row of a slice that started mid-row: carries in thread order
    int t0 = tid;
    while (t0 > 0 && s_crow[t0 - 1] == srow) --t0;
    bool have = false;
    T v = T(0);
    if (t0 == 0 && srow == 0 && tc->valid) { v = tc->val; have = true; }
    for (int u = t0; u < tid; ++u) { v = have ? v + s_cval[u] : s_cval[u]; have = true; }
    v = have ? v + sval : sval;
    qstore(t.i0 + srow, v);
  }
  if (!last && tid == NT - 1) {  // carry into the next tile: the partial sum of row i0 + rows_t
                                 // (the CTA's last tile ends on a row boundary: no carry)
    int t0 = NT;
    while (t0 > 0 && s_crow[t0 - 1] == t.rows_t) --t0;
    bool have = false;
    T v = T(0);
    if (t0 == 0 && t.rows_t == 0 && tc->valid) { v = tc->val; have = true; }
    for (int u = t0; u < NT; ++u) { v = have ? v + s_cval[u] : s_cval[u]; have = true; }
    tn->val = v;
    tn->valid = have ? 1 : 0;
  }
  __syncthreads();
}

// Streams / resident tiles of CTA c through tile_spmv.  State of the double buffer lives in the
// caller (u = next stream sequence number to consume; persistent launches wrap around so the
// first tiles of the next iteration are in flight across the barrier).
template <typename T> struct Pipe {
  int tb, nt;        // first coordinate index, tile count
  int mres;          // resident tiles
  int ns;            // streamed tiles
  long long u;       // next streamed sequence number to consume
  long long issued;  // streamed sequence numbers issued
  unsigned char *sbuf;  // stream buffer b at sbuf + b * sstride
  int sstride;
  unsigned char *res;
};

template <typename T>
PERKS_DEVINL void pipe_issue_next(const Params<T> &P, Pipe<T> &pp, uint64_t *mbar, bool wrap) {
  // thread 0 only: keep two streamed tiles in flight
  while (pp.ns > 0 && pp.issued < pp.u + 2 && (wrap || pp.issued < pp.ns)) {
    const int m = pp.mres + (int)(pp.issued % pp.ns);
    const int2 a = P.coords[pp.tb + m], e = P.coords[pp.tb + m + 1];
    const int buf = (int)(pp.issued & 1);
    issue_tile<T>(P, pp.sbuf + buf * pp.sstride, a.x, a.y, e.x - a.x, e.y - a.y, mbar + buf);
    ++pp.issued;
  }
}

template <typename T, class Gather, class QStore>
PERKS_DEVINL void spmv_cta(const Params<T> &P, Pipe<T> &pp, unsigned char *smem, bool wrap, Gather gather,
                           QStore qstore) {
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + Smem::MBAR);
  TileCarry<T> *tc = reinterpret_cast<TileCarry<T> *>(smem + Smem::TCAR);
  if (threadIdx.x == 0) tc->valid = 0;  // CTA shares start on a row boundary
  __syncthreads();
  int roff = 0;
  for (int m = 0; m < pp.nt; ++m) {
    const int2 a = P.coords[pp.tb + m], e = P.coords[pp.tb + m + 1];
    const int rows_t = e.x - a.x, nnz_t = e.y - a.y;
    unsigned char *img;
    if (m < pp.mres) {
      img = pp.res + roff;
      roff += TileGeo<T>(a.x, rows_t, a.y, nnz_t).bytes();
    } else {
      const int buf = (int)(pp.u & 1);
      mbar_wait(mbar + buf, (unsigned)((pp.u >> 1) & 1));
      img = pp.sbuf + buf * pp.sstride;
    }
    tile_spmv<T>(tile_view<T>(img, a.x, a.y, rows_t, nnz_t), smem, m & 1, m == pp.nt - 1, gather, qstore);
    if (m >= pp.mres) {
      ++pp.u;
      if (threadIdx.x == 0) pipe_issue_next<T>(P, pp, mbar, wrap);
    }
  }
}

template <typename T>
PERKS_DEVINL void pipe_init(const Params<T> &P, Pipe<T> &pp, unsigned char *smem, int vec_rows, bool wrap) {
  const int c = blockIdx.x;
  pp.tb = P.ctile[c];
  pp.nt = P.ctile[c + 1] - pp.tb - 1;
  unsigned char *p = smem + Smem::vec_off<T>() + 4 * a16((long long)vec_rows * (int)sizeof(T));
  pp.sbuf = p;
  pp.sstride = P.stream ? tile_max_bytes<T>() : 0;
  pp.res = p + (P.stream ? 2 * tile_max_bytes<T>() : 0);
  // resident tiles: the first tiles of the CTA while their images fit the budget
  int used = 0, mres = 0;
  for (int m = 0; m < pp.nt; ++m) {
    const int2 a = P.coords[pp.tb + m], e = P.coords[pp.tb + m + 1];
    const int bts = TileGeo<T>(a.x, e.x - a.x, a.y, e.y - a.y).bytes();
    if (used + bts > P.res_budget) break;
    used += bts;
    ++mres;
  }
  pp.mres = mres;
  pp.ns = pp.nt - mres;
  pp.u = 0;
  pp.issued = 0;
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + Smem::MBAR);
  if (threadIdx.x == 0) {
    mbar_init(mbar + 0, 1);
    mbar_init(mbar + 1, 1);
    mbar_init(mbar + 2, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mres > 0) {  // resident tiles: one mbarrier phase for all of them
      mbar_arrive_tx(mbar + 2, (unsigned)used);
      int off = 0;
      for (int m = 0; m < mres; ++m) {
        const int2 a = P.coords[pp.tb + m], e = P.coords[pp.tb + m + 1];
        issue_tile<T>(P, pp.res + off, a.x, a.y, e.x - a.x, e.y - a.y, mbar + 2, false);
        off += TileGeo<T>(a.x, e.x - a.x, a.y, e.y - a.y).bytes();
      }
    }
    pipe_issue_next<T>(P, pp, mbar, wrap);
  }
  if (mres > 0) mbar_wait(mbar + 2, 0);
}

// Before exit: every issued bulk copy must have landed (thread 0 waits on the outstanding ones).
template <typename T> PERKS_DEVINL void pipe_drain(Pipe<T> &pp, unsigned char *smem) {
  uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + Smem::MBAR);
  if (threadIdx.x == 0)
    for (long long v = pp.u; v < pp.issued; ++v) mbar_wait(mbar + (v & 1), (unsigned)((v >> 1) & 1));
  __syncthreads();
}

// ------------------------------------------------------------------------ CG building blocks
// Vector access for the CTA's own rows: shared memory under VEC, global otherwise.
template <typename T, bool VEC> struct Own {
  T *s_r, *s_x, *s_p, *s_q;
  int R0, rows;
};

template <typename T, bool VEC>
PERKS_DEVINL Own<T, VEC> own_view(const Params<T> &P, unsigned char *smem) {
  Own<T, VEC> o;
  o.R0 = P.crow[blockIdx.x];
  o.rows = P.crow[blockIdx.x + 1] - o.R0;
  const int vb = a16((long long)P.rows_max * (int)sizeof(T));
  unsigned char *v = smem + Smem::vec_off<T>();
  o.s_r = reinterpret_cast<T *>(v);
  o.s_x = reinterpret_cast<T *>(v + vb);
  o.s_p = reinterpret_cast<T *>(v + 2 * vb);
  o.s_q = reinterpret_cast<T *>(v + 3 * vb);
  return o;
}

// x_0 = 0, r_0 = b (published for the gathers); returns this thread's part of <r_0, r_0>.
template <typename T, bool VEC> PERKS_DEVINL double cg_prologue(const Params<T> &P, const Own<T, VEC> &o) {
  double acc = 0.0;
  for (int j = threadIdx.x; j < o.rows; j += NT) {
    const int i = o.R0 + j;
    const T bi = P.b[i];
    if (VEC) { o.s_x[j] = T(0); o.s_r[j] = bi; }
    else P.x[i] = T(0);
    P.r[i] = bi;
    acc = fma_rn((double)bi, (double)bi, acc);
  }
  return acc;
}

// Own-row passes visit rows j = tid, tid+NT, ... in that order (the order of every per-thread
// inner-product chain); U rows per batch so their loads are in flight together.
constexpr int U = 4;

// p_k (own rows): p_0 = r_0; p_k = fma(beta, p_{k-1}, r_k); published into pcur.
template <typename T, bool VEC>
PERKS_DEVINL void cg_p_update(const Params<T> &P, const Own<T, VEC> &o, bool first, T beta, const T *pprev, T *pcur) {
  for (int j0 = threadIdx.x; j0 < o.rows; j0 += U * NT) {
    T r[U], pp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * NT, i = o.R0 + j;
      const bool ok = j < o.rows;
      r[u] = ok ? (VEC ? o.s_r[j] : __ldcg(P.r + i)) : T(0);
      pp[u] = ok && !first ? (VEC ? o.s_p[j] : __ldcg(pprev + i)) : T(0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * NT;
      if (j < o.rows) {
        const T p = first ? r[u] : fma_rn(beta, pp[u], r[u]);
        if (VEC) o.s_p[j] = p;
        pcur[o.R0 + j] = p;
      }
    }
  }
}

// This thread's part of <p_k, A p_k>.
template <typename T, bool VEC> PERKS_DEVINL double cg_pap(const Params<T> &P, const Own<T, VEC> &o, const T *pcur) {
  double acc = 0.0;
  for (int j0 = threadIdx.x; j0 < o.rows; j0 += U * NT) {
    T p[U], q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * NT, i = o.R0 + j;
      const bool ok = j < o.rows;
      p[u] = ok ? (VEC ? o.s_p[j] : __ldcg(pcur + i)) : T(0);
      q[u] = ok ? (VEC ? o.s_q[j] : __ldcg(P.q + i)) : T(0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j0 + u * NT < o.rows) acc = fma_rn((double)p[u], (double)q[u], acc);
  }
  return acc;
}

// x_{k+1} = fma(a, p, x); r_{k+1} = fma(-a, A p, r) (published); this thread's part of <r,r>.
template <typename T, bool VEC>
PERKS_DEVINL double cg_xr_update(const Params<T> &P, const Own<T, VEC> &o, T a, const T *pcur) {
  double acc = 0.0;
  for (int j0 = threadIdx.x; j0 < o.rows; j0 += U * NT) {
    T p[U], q[U], x[U], r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * NT, i = o.R0 + j;
      const bool ok = j < o.rows;
      if (VEC) {
        p[u] = ok ? o.s_p[j] : T(0); q[u] = ok ? o.s_q[j] : T(0);
        x[u] = ok ? o.s_x[j] : T(0); r[u] = ok ? o.s_r[j] : T(0);
      } else {
        p[u] = ok ? __ldcg(pcur + i) : T(0); q[u] = ok ? __ldcg(P.q + i) : T(0);
        x[u] = ok ? __ldcg(P.x + i) : T(0); r[u] = ok ? __ldcg(P.r + i) : T(0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * NT, i = o.R0 + j;
      if (j < o.rows) {
        const T xn = fma_rn(a, p[u], x[u]);
        const T rn = fma_rn(-a, q[u], r[u]);
        if (VEC) { o.s_x[j] = xn; o.s_r[j] = rn; }
        else P.x[i] = xn;
        P.r[i] = rn;
        acc = fma_rn((double)rn, (double)rn, acc);
      }
    }
  }
  return acc;
}

// The SpMV A p_k of the CTA's own rows, gathers as described in the header.
template <typename T, bool VEC>
PERKS_DEVINL void cg_spmv(const Params<T> &P, const Own<T, VEC> &o, Pipe<T> &pp, unsigned char *smem, bool wrap,
                          bool first, T beta, const T *pprev, const T *pcur) {
  const int R0 = o.R0, rows = o.rows;
  const T *r = P.r;
  T *q = P.q;
  const T *sp = o.s_p;
  T *sq = o.s_q;
  auto gather = [=](int jc) -> T {
    const unsigned off = (unsigned)(jc - R0);
    if (off < (unsigned)rows) return VEC ? sp[off] : __ldcg(pcur + jc);
    return first ? __ldcg(r + jc) : fma_rn(beta, __ldcg(pprev + jc), __ldcg(r + jc));
  };
  auto qstore = [=](int row, T v) {
    if (VEC) sq[row - R0] = v;
    else q[row] = v;
  };
  spmv_cta<T>(P, pp, smem, wrap, gather, qstore);
}

// ------------------------------------------------------------------------ kernels
// (b)/(c): the whole solve in one cooperative launch.
template <typename T, bool VEC> __global__ void __launch_bounds__(NT, 1) cg_persistent_kernel(Params<T> P) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *s_red = reinterpret_cast<double *>(smem + Smem::RED);
  double *s_bc = reinterpret_cast<double *>(smem + Smem::BCAST);
  const Own<T, VEC> o = own_view<T, VEC>(P, smem);
  Pipe<T> pp;
  pipe_init<T>(P, pp, smem, VEC ? P.rows_max : 0, true);
  const int c = blockIdx.x;
  unsigned nb = 0;
  double part = block_sum(cg_prologue<T, VEC>(P, o), s_red);
  if (threadIdx.x == 0) P.slots[P.G + c] = part;
  grid_barrier(P.bar, ++nb);
  double rr = slots_sum(P.slots + P.G, P.G, s_bc);
  if (c == 0 && threadIdx.x == 0 && P.hist) P.hist[0] = rr;
  long long k = 0;
  int status = 0;
  double beta = 0.0;
  while (k < P.kmax) {
    if (!(rr > P.tol2)) break;  // reading RC2: <r_k,r_k> <= tol^2 stops before the iteration
    const bool first = (k == 0);
    T *pcur = (k & 1) ? P.p1 : P.p0;
    const T *pprev = (k & 1) ? P.p0 : P.p1;
    const T bt = (T)beta;
    cg_p_update<T, VEC>(P, o, first, bt, pprev, pcur);
    __syncthreads();
    cg_spmv<T, VEC>(P, o, pp, smem, true, first, bt, pprev, pcur);
    part = block_sum(cg_pap<T, VEC>(P, o, pcur), s_red);
    if (threadIdx.x == 0) P.slots[c] = part;
    grid_barrier(P.bar, ++nb);
    const double pap = slots_sum(P.slots, P.G, s_bc + 1);
    if (!(pap > 0.0)) { status = 1; break; }  // reading RC4: not positive definite
    const double alpha = rr / pap;
    part = block_sum(cg_xr_update<T, VEC>(P, o, (T)alpha, pcur), s_red);
    if (threadIdx.x == 0) P.slots[P.G + c] = part;
    grid_barrier(P.bar, ++nb);
    const double rr_new = slots_sum(P.slots + P.G, P.G, s_bc + 2);
    beta = rr_new / rr;
    rr = rr_new;
    ++k;
    if (c == 0 && threadIdx.x == 0 && P.hist) P.hist[k] = rr;
  }
  if (VEC)
    for (int j = threadIdx.x; j < o.rows; j += NT) P.x[o.R0 + j] = o.s_x[j];
  if (c == 0 && threadIdx.x == 0 && P.info) { P.info[0] = k; P.info[1] = status; }
  pipe_drain<T>(pp, smem);
}

// (a) host loop: prologue, then per iteration kernel A (p update, SpMV, <p,Ap>) and kernel B
// (x/r update, <r,r>), then a finishing kernel.  Same partition, same arithmetic, same order.
template <typename T> __global__ void __launch_bounds__(NT, 1) cg_hl_prologue_kernel(Params<T> P) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *s_red = reinterpret_cast<double *>(smem + Smem::RED);
  double *s_bc = reinterpret_cast<double *>(smem + Smem::BCAST);
  const Own<T, false> o = own_view<T, false>(P, smem);
  const double part = block_sum(cg_prologue<T, false>(P, o), s_red);
  if (threadIdx.x == 0) P.slots[P.G + blockIdx.x] = part;
  if (blockIdx.x == 0 && threadIdx.x == 0) { P.state[0] = 0; P.state[1] = 0; P.state[2] = 0; }
}

template <typename T> __global__ void __launch_bounds__(NT, 1) cg_hl_a_kernel(Params<T> P, long long k) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *s_red = reinterpret_cast<double *>(smem + Smem::RED);
  double *s_bc = reinterpret_cast<double *>(smem + Smem::BCAST);
  if (__ldcg(P.state) != 0) return;
  const int c = blockIdx.x;
  const double rr = slots_sum(P.slots + P.G, P.G, s_bc);  // <r_k, r_k>
  const double beta = k > 0 ? rr / __ldcg(P.scal + ((k - 1) & 1)) : 0.0;
  if (c == 0 && threadIdx.x == 0) {
    P.scal[k & 1] = rr;
    if (P.hist) P.hist[k] = rr;
  }
  if (!(rr > P.tol2)) {
    if (c == 0 && threadIdx.x == 0) { P.state[1] = k; P.state[0] = 1; }
    return;
  }
  const Own<T, false> o = own_view<T, false>(P, smem);
  Pipe<T> pp;
  pipe_init<T>(P, pp, smem, 0, false);
  const bool first = (k == 0);
  T *pcur = (k & 1) ? P.p1 : P.p0;
  const T *pprev = (k & 1) ? P.p0 : P.p1;
  const T bt = (T)beta;
  cg_p_update<T, false>(P, o, first, bt, pprev, pcur);
  __syncthreads();
  cg_spmv<T, false>(P, o, pp, smem, false, first, bt, pprev, pcur);
  const double part = block_sum(cg_pap<T, false>(P, o, pcur), s_red);
  if (threadIdx.x == 0) P.slots[c] = part;
  pipe_drain<T>(pp, smem);
}

template <typename T> __global__ void __launch_bounds__(NT, 1) cg_hl_b_kernel(Params<T> P, long long k) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *s_red = reinterpret_cast<double *>(smem + Smem::RED);
  double *s_bc = reinterpret_cast<double *>(smem + Smem::BCAST);
  if (__ldcg(P.state) != 0) return;
  const int c = blockIdx.x;
  const double pap = slots_sum(P.slots, P.G, s_bc);
  if (!(pap > 0.0)) {
    if (c == 0 && threadIdx.x == 0) { P.state[1] = k; P.state[2] = 1; P.state[0] = 1; }
    return;
  }
  const double rr = __ldcg(P.scal + (k & 1));
  const double alpha = rr / pap;
  const Own<T, false> o = own_view<T, false>(P, smem);
  T *pcur = (k & 1) ? P.p1 : P.p0;
  const double part = block_sum(cg_xr_update<T, false>(P, o, (T)alpha, pcur), s_red);
  if (threadIdx.x == 0) P.slots[P.G + c] = part;
}

template <typename T> __global__ void cg_hl_finish_kernel(Params<T> P) {
  // one warp: <r_kmax, r_kmax> (if the loop ran to k_max) and the info words
  const long long done = __ldcg(P.state);
  if (!done) {
    __shared__ double s_fin;
    const double rr = slots_sum(P.slots + P.G, P.G, &s_fin);
    if (threadIdx.x == 0 && P.hist) P.hist[P.kmax] = rr;
  }
  if (threadIdx.x == 0 && P.info) {
    P.info[0] = done ? __ldcg(P.state + 1) : P.kmax;
    P.info[1] = done ? __ldcg(P.state + 2) : 0;
  }
}

// Standalone merge-based SpMV: q = A xin.
template <typename T> __global__ void __launch_bounds__(NT, 1) cg_spmv_kernel(Params<T> P) {
  extern __shared__ __align__(128) unsigned char smem[];
  Pipe<T> pp;
  pipe_init<T>(P, pp, smem, 0, false);
  const T *xin = P.xin;
  T *y = P.q;
  auto gather = [=](int j) -> T { return __ldg(xin + j); };
  auto qstore = [=](int row, T v) { y[row] = v; };
  spmv_cta<T>(P, pp, smem, false, gather, qstore);
  pipe_drain<T>(pp, smem);
}

}  // namespace cg
}  // namespace perks

// =============================================================================== host side
using namespace perks;
using namespace perks::cg;

namespace {
perks_status cg_cuda_fail(cudaError_t e) { return perks::cuda_status(e); }
struct DevGuard {
  int prev = -1;
  bool ok = true;
  explicit DevGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DevGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};
}  // namespace

struct perks_cg_s {
  int device = 0, num_sms = 0;
  perks_dtype dtype = PERKS_F64;
  int64_t n = 0, nnz = 0;
  int G = 1;
  int rows_max = 0;
  int ntiles = 0;
  int tile_max = 0;                 // largest tile image (bytes)
  std::vector<int> h_crow;          // G+1
  std::vector<int> h_ctile;         // G+1
  std::vector<int2> h_coords;       // ntiles + G
  void *d_mem = nullptr;            // one allocation: row_off | col | val | coords | ctile | crow
  int *d_row_off = nullptr, *d_col = nullptr, *d_ctile = nullptr, *d_crow = nullptr;
  void *d_val = nullptr;
  int2 *d_coords = nullptr;
  // run_host scratch
  std::mutex mu;
  size_t elem() const { return dtype == PERKS_F64 ? 8 : 4; }
};

namespace {

// Merge-path search on the global CSR: (rows completed, nonzeros consumed) at diagonal d.
void path_coord(const std::vector<int64_t> &ro, int64_t n, int64_t nnz, int64_t d, int64_t &i, int64_t &k) {
  int64_t lo = std::max<int64_t>(0, d - nnz), hi = std::min<int64_t>(d, n);
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (ro[mid + 1] <= d - 1 - mid) lo = mid + 1;
    else hi = mid;
  }
  i = lo;
  k = d - lo;
}

struct Layout {
  size_t ws_bytes, off_r, off_p0, off_p1, off_q, off_slots, off_scal, off_state, off_bar;
};
Layout ws_layout(const perks_cg_s *h) {
  Layout L{};
  const size_t vb = align256((size_t)std::max<int64_t>(h->n, 1) * h->elem());
  size_t o = 0;
  L.off_bar = o; o += 256;
  L.off_slots = o; o += align256((size_t)2 * h->G * 8);
  L.off_scal = o; o += 256;
  L.off_state = o; o += 256;
  L.off_r = o; o += vb;
  L.off_p0 = o; o += vb;
  L.off_p1 = o; o += vb;
  L.off_q = o; o += vb;
  L.ws_bytes = o;
  return L;
}

struct CgPlan {
  int variant, policy;
  bool vec = false;
  int res_budget = 0;
  bool stream = true;
  int smem = 0;
  int64_t cached_nnz = 0, cached_rows = 0;
  double dram = 0, unfused = 0;
};

int tile_bytes_host(const perks_cg_s *h, int idx, int c) {
  const int2 a = h->h_coords[idx], e = h->h_coords[idx + 1];
  (void)c;
  return h->dtype == PERKS_F64 ? TileGeo<double>(a.x, e.x - a.x, a.y, e.y - a.y).bytes()
                               : TileGeo<float>(a.x, e.x - a.x, a.y, e.y - a.y).bytes();
}

CgPlan make_plan(const perks_cg_s *h, perks_variant v, perks_cg_policy pol) {
  CgPlan pl;
  if (v == PERKS_AUTO) v = PERKS_PERKS;
  if (pol == PERKS_CG_AUTO) pol = PERKS_CG_MIX;
  if (v == PERKS_HOSTLOOP || v == PERKS_PERSISTENT) pol = PERKS_CG_IMP;
  pl.variant = v;
  pl.policy = pol;
  const bool f64 = h->dtype == PERKS_F64;
  const int S = (int)h->elem();
  const int tmax = f64 ? tile_max_bytes<double>() : tile_max_bytes<float>();
  const int base = f64 ? Smem::vec_off<double>() : Smem::vec_off<float>();
  const int vecb = 4 * a16((long long)h->rows_max * S);
  pl.vec = (pol == PERKS_CG_VEC || pol == PERKS_CG_MIX) && base + vecb + 2 * tmax <= kSmemMax;
  const int fixed = base + (pl.vec ? vecb : 0);
  const bool mat = pol == PERKS_CG_MAT || pol == PERKS_CG_MIX;
  // resident budget: if every CTA's whole share fits without stream buffers, no streaming
  int need_max = 0;
  for (int c = 0; c < h->G; ++c) {
    int s = 0;
    for (int m = h->h_ctile[c]; m < h->h_ctile[c + 1] - 1; ++m) s += tile_bytes_host(h, m, c);
    need_max = std::max(need_max, s);
  }
  if (mat && fixed + need_max <= kSmemMax) {
    pl.res_budget = need_max;
    pl.stream = false;
  } else if (mat) {
    pl.res_budget = std::max(0, kSmemMax - fixed - 2 * tmax) & ~15;
    pl.stream = true;
  } else {
    pl.res_budget = 0;
    pl.stream = h->ntiles > 0;
  }
  pl.smem = fixed + (pl.stream ? 2 * tmax : 0) + pl.res_budget;
  // what is cached, per CTA exactly as pipe_init decides
  for (int c = 0; c < h->G; ++c) {
    int used = 0;
    for (int m = h->h_ctile[c]; m < h->h_ctile[c + 1] - 1; ++m) {
      const int b = tile_bytes_host(h, m, c);
      if (used + b > pl.res_budget) break;
      used += b;
      pl.cached_nnz += h->h_coords[m + 1].y - h->h_coords[m].y;
    }
    if (pl.vec) pl.cached_rows += h->h_crow[c + 1] - h->h_crow[c];
  }
  // bytes per iteration.  Unfused (the metric): A once (values, columns, row offsets), the
  // gathered p once per row, and the vector passes of Algorithm: p update (r, p
  // read, p written), <p,Ap> (p, q read), x update (x, p read, x written), r update (r, q
  // read, r written), <r,r> (r read) = 13 vector accesses per row, and A p written once.
  const double n = (double)h->n, nnz = (double)h->nnz;
  pl.unfused = nnz * (S + 4) + (n + 1) * 4 + n * S * (1 + 13 + 1);
  // modelled DRAM: uncached matrix + the vectors that leave the SM (r and p published, read
  // back by the gathers through L2: counted once), plus own-row vector traffic without VEC.
  const double mat_b = (nnz - (double)pl.cached_nnz) * (S + 4) + (n + 1) * 4;
  const double vec_b = pl.vec ? n * S * 2 : n * S * (2 + 9);
  pl.dram = mat_b + vec_b;
  return pl;
}

template <typename T> Params<T> make_params(perks_cg_s *h, void *ws, const CgPlan &pl) {
  const Layout L = ws_layout(h);
  unsigned char *w = static_cast<unsigned char *>(ws);
  Params<T> P{};
  P.n = (int)h->n;
  P.G = h->G;
  P.row_off = h->d_row_off;
  P.col = h->d_col;
  P.val = static_cast<const T *>(h->d_val);
  P.coords = h->d_coords;
  P.ctile = h->d_ctile;
  P.crow = h->d_crow;
  P.r = reinterpret_cast<T *>(w + L.off_r);
  P.p0 = reinterpret_cast<T *>(w + L.off_p0);
  P.p1 = reinterpret_cast<T *>(w + L.off_p1);
  P.q = reinterpret_cast<T *>(w + L.off_q);
  P.slots = reinterpret_cast<double *>(w + L.off_slots);
  P.scal = reinterpret_cast<double *>(w + L.off_scal);
  P.state = reinterpret_cast<long long *>(w + L.off_state);
  P.bar = reinterpret_cast<unsigned *>(w + L.off_bar);
  P.rows_max = h->rows_max;
  P.res_budget = pl.res_budget;
  P.stream = pl.stream ? 1 : 0;
  return P;
}

template <typename T>
cudaError_t launch_solve(perks_cg_s *h, const CgPlan &pl, const void *b, void *x, int64_t kmax, double tol,
                         double *hist, int64_t *info, void *ws, cudaStream_t s) {
  Params<T> P = make_params<T>(h, ws, pl);
  P.b = static_cast<const T *>(b);
  P.x = static_cast<T *>(x);
  P.hist = hist;
  P.info = reinterpret_cast<long long *>(info);
  P.kmax = kmax;
  P.tol2 = tol * tol;
  cudaError_t e;
  if (pl.variant == PERKS_HOSTLOOP) {
    const int smem = smem_bytes<T>(0, P.stream, 0);
    void (*ka)(Params<T>, long long) = cg_hl_a_kernel<T>;
    void (*pk)(Params<T>) = cg_hl_prologue_kernel<T>;
    void (*kb)(Params<T>, long long) = cg_hl_b_kernel<T>;
    if ((e = cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess) return e;
    pk<<<h->G, NT, smem, s>>>(P);
    for (long long k = 0; k < kmax; ++k) {
      ka<<<h->G, NT, smem, s>>>(P, k);
      kb<<<h->G, NT, smem, s>>>(P, k);
    }
    cg_hl_finish_kernel<T><<<1, 32, 0, s>>>(P);
    return cudaGetLastError();
  }
  if ((e = reset_grid_barrier(P.bar, s)) != cudaSuccess) return e;
  void *kfn = pl.vec ? (void *)cg_persistent_kernel<T, true> : (void *)cg_persistent_kernel<T, false>;
  if ((e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem)) != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(h->G);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = (size_t)pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  void *args[] = {&P};
  return cudaLaunchKernelExC(&cfg, kfn, args);
}

template <typename T> cudaError_t launch_spmv(perks_cg_s *h, const void *xin, void *y, void *ws, cudaStream_t s) {
  CgPlan pl = make_plan(h, PERKS_HOSTLOOP, PERKS_CG_IMP);
  Params<T> P = make_params<T>(h, ws, pl);
  P.xin = static_cast<const T *>(xin);
  P.q = static_cast<T *>(y);
  const int smem = smem_bytes<T>(0, P.stream, 0);
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(cg_spmv_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess)
    return e;
  cg_spmv_kernel<T><<<h->G, NT, smem, s>>>(P);
  return cudaGetLastError();
}

bool overlaps(const void *a, size_t na, const void *b, size_t nb) {
  const char *x = static_cast<const char *>(a), *y = static_cast<const char *>(b);
  return x < y + nb && y < x + na;
}

}  // namespace

extern "C" {

perks_status perks_cg_create(const perks_csr_desc *d, int device, perks_cg_t *out) {
  if (!d || !out) return PERKS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (d->dtype != PERKS_F32 && d->dtype != PERKS_F64) return PERKS_ERR_INVALID_ARGUMENT;
  if (d->n_rows < 0 || d->nnz < 0 || !d->row_offsets) return PERKS_ERR_INVALID_ARGUMENT;
  if (d->nnz > 0 && (!d->col_indices || !d->values)) return PERKS_ERR_INVALID_ARGUMENT;
  if (d->n_rows >= INT_MAX / 2 || d->nnz >= INT_MAX / 2 || d->n_rows + d->nnz >= INT_MAX / 2)
    return PERKS_ERR_UNSUPPORTED;
  const int64_t n = d->n_rows, nnz = d->nnz;
  if (d->row_offsets[0] != 0 || d->row_offsets[n] != nnz) return PERKS_ERR_INVALID_ARGUMENT;
  for (int64_t i = 0; i < n; ++i)
    if (d->row_offsets[i + 1] < d->row_offsets[i]) return PERKS_ERR_INVALID_ARGUMENT;
  for (int64_t k = 0; k < nnz; ++k)
    if (d->col_indices[k] < 0 || d->col_indices[k] >= n) return PERKS_ERR_INVALID_ARGUMENT;
  DevGuard g(device);
  if (!g.ok) return cg_cuda_fail(cudaGetLastError());
  perks_cg_s *h = new (std::nothrow) perks_cg_s;
  if (!h) return PERKS_ERR_OOM;
  h->device = device;
  h->dtype = d->dtype;
  h->n = n;
  h->nnz = nnz;
  cudaError_t e = cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) { delete h; return cg_cuda_fail(e); }
  h->num_sms = env_int("PERKS_NUM_SMS", h->num_sms);
  // CTA-level (TB-level) merge-path partition, row aligned; then tiles of TILE path items.
  const int64_t L = n + nnz;
  h->G = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(h->num_sms, kMaxG), (L + 1023) / 1024));
  std::vector<int64_t> ro(d->row_offsets, d->row_offsets + n + 1);
  h->h_crow.resize(h->G + 1);
  for (int c = 0; c <= h->G; ++c) {
    int64_t i, k;
    path_coord(ro, n, nnz, L * c / h->G, i, k);
    h->h_crow[c] = (int)(c == h->G ? n : i);
  }
  for (int c = 0; c < h->G; ++c) h->rows_max = std::max(h->rows_max, h->h_crow[c + 1] - h->h_crow[c]);
  h->h_ctile.resize(h->G + 1);
  for (int c = 0; c < h->G; ++c) {
    h->h_ctile[c] = (int)h->h_coords.size();
    const int64_t R0 = h->h_crow[c], R1 = h->h_crow[c + 1];
    const int64_t P0 = R0 + ro[R0], P1 = R1 + ro[R1];
    for (int64_t dd = P0; dd < P1; dd += TILE) {
      int64_t i, k;
      path_coord(ro, n, nnz, dd, i, k);
      h->h_coords.push_back(make_int2((int)i, (int)k));
    }
    h->h_coords.push_back(make_int2((int)R1, (int)ro[R1]));
  }
  h->h_ctile[h->G] = (int)h->h_coords.size();
  h->ntiles = (int)h->h_coords.size() - h->G;
  // device copy: row_off | col | val | coords | ctile | crow (each 256-B aligned, padded so the
  // 16-byte-rounded bulk copies never read past an allocation)
  const size_t S = h->elem();
  const size_t b_ro = align256((n + 1) * 4 + 64), b_col = align256(nnz * 4 + 64), b_val = align256(nnz * S + 64);
  const size_t b_co = align256(h->h_coords.size() * 8), b_ct = align256((h->G + 1) * 4), b_cr = b_ct;
  e = cudaMalloc(&h->d_mem, b_ro + b_col + b_val + b_co + b_ct + b_cr);
  if (e != cudaSuccess) { delete h; return cg_cuda_fail(e); }
  char *m = static_cast<char *>(h->d_mem);
  h->d_row_off = reinterpret_cast<int *>(m);
  h->d_col = reinterpret_cast<int *>(m + b_ro);
  h->d_val = m + b_ro + b_col;
  h->d_coords = reinterpret_cast<int2 *>(m + b_ro + b_col + b_val);
  h->d_ctile = reinterpret_cast<int *>(m + b_ro + b_col + b_val + b_co);
  h->d_crow = reinterpret_cast<int *>(m + b_ro + b_col + b_val + b_co + b_ct);
  std::vector<int> ro32(n + 1);
  for (int64_t i = 0; i <= n; ++i) ro32[i] = (int)ro[i];
  std::vector<unsigned char> vals(nnz * S + 1);
  for (int64_t k = 0; k < nnz; ++k) {
    if (h->dtype == PERKS_F64) {
      const double v = d->values[k];
      std::memcpy(vals.data() + k * 8, &v, 8);
    } else {
      const float v = (float)d->values[k];  // rounded once (reading RC3)
      std::memcpy(vals.data() + k * 4, &v, 4);
    }
  }
  if ((e = cudaMemset(h->d_mem, 0, b_ro + b_col + b_val)) != cudaSuccess ||
      (e = cudaMemcpy(h->d_row_off, ro32.data(), (n + 1) * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (nnz && (e = cudaMemcpy(h->d_col, d->col_indices, nnz * 4, cudaMemcpyHostToDevice)) != cudaSuccess) ||
      (nnz && (e = cudaMemcpy(h->d_val, vals.data(), nnz * S, cudaMemcpyHostToDevice)) != cudaSuccess) ||
      (e = cudaMemcpy(h->d_coords, h->h_coords.data(), h->h_coords.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(h->d_ctile, h->h_ctile.data(), (h->G + 1) * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(h->d_crow, h->h_crow.data(), (h->G + 1) * 4, cudaMemcpyHostToDevice)) != cudaSuccess) {
    cudaFree(h->d_mem);
    delete h;
    return cg_cuda_fail(e);
  }
  *out = h;
  return PERKS_OK;
}

perks_status perks_cg_workspace_bytes(perks_cg_t h, size_t *bytes) {
  if (!h || !bytes) return PERKS_ERR_INVALID_ARGUMENT;
  *bytes = ws_layout(h).ws_bytes;
  return PERKS_OK;
}

static perks_status check_ws(perks_cg_t h, void *ws, size_t wsb) {
  if (!ws || ((uintptr_t)ws & 255) || wsb < ws_layout(h).ws_bytes) return PERKS_ERR_WORKSPACE;
  return PERKS_OK;
}

perks_status perks_cg_spmv(perks_cg_t h, const void *d_x, void *d_y, void *ws, size_t wsb, void *stream) {
  if (!h || (h->n > 0 && (!d_x || !d_y))) return PERKS_ERR_INVALID_ARGUMENT;
  if (perks_status st = check_ws(h, ws, wsb)) return st;
  if (h->n == 0) return PERKS_OK;
  if (overlaps(d_x, h->n * h->elem(), d_y, h->n * h->elem())) return PERKS_ERR_ALIAS;
  DevGuard g(h->device);
  if (!g.ok) return cg_cuda_fail(cudaGetLastError());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const cudaError_t e = h->dtype == PERKS_F64 ? launch_spmv<double>(h, d_x, d_y, ws, s)
                                              : launch_spmv<float>(h, d_x, d_y, ws, s);
  return e == cudaSuccess ? PERKS_OK : cg_cuda_fail(e);
}

perks_status perks_cg_solve(perks_cg_t h, perks_variant v, perks_cg_policy pol, const void *d_b, void *d_x,
                            int64_t kmax, double tol, double *d_hist, int64_t *d_info, void *ws, size_t wsb,
                            void *stream) {
  if (!h || kmax < 0 || !(tol >= 0.0) || (h->n > 0 && (!d_b || !d_x))) return PERKS_ERR_INVALID_ARGUMENT;
  if ((int)v < PERKS_AUTO || (int)v > PERKS_PERKS || (int)pol < PERKS_CG_AUTO || (int)pol > PERKS_CG_MIX)
    return PERKS_ERR_INVALID_ARGUMENT;
  if (perks_status st = check_ws(h, ws, wsb)) return st;
  if (h->n > 0 && overlaps(d_b, h->n * h->elem(), d_x, h->n * h->elem())) return PERKS_ERR_ALIAS;
  DevGuard g(h->device);
  if (!g.ok) return cg_cuda_fail(cudaGetLastError());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const CgPlan pl = make_plan(h, v, pol);
  if (pl.smem > kSmemMax) return PERKS_ERR_UNSUPPORTED;
  const cudaError_t e = h->dtype == PERKS_F64
                            ? launch_solve<double>(h, pl, d_b, d_x, kmax, tol, d_hist, d_info, ws, s)
                            : launch_solve<float>(h, pl, d_b, d_x, kmax, tol, d_hist, d_info, ws, s);
  return e == cudaSuccess ? PERKS_OK : cg_cuda_fail(e);
}

perks_status perks_cg_solve_host(perks_cg_t h, perks_variant v, perks_cg_policy pol, const void *h_b, void *h_x,
                                 int64_t kmax, double tol, double *h_hist, int64_t *h_info) {
  if (!h || (h->n > 0 && (!h_b || !h_x)) || kmax < 0) return PERKS_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lk(h->mu);
  DevGuard g(h->device);
  if (!g.ok) return cg_cuda_fail(cudaGetLastError());
  const size_t vb = (size_t)std::max<int64_t>(h->n, 1) * h->elem();
  const size_t wsb = ws_layout(h).ws_bytes;
  const size_t hb = (size_t)(kmax + 1) * 8;
  char *buf = nullptr;
  const size_t ob_b = 0, ob_x = align256(vb), ob_h = 2 * align256(vb), ob_i = ob_h + align256(hb),
               ob_w = ob_i + 256, total = ob_w + wsb;
  cudaError_t e = cudaMalloc(&buf, total);
  if (e != cudaSuccess) return cg_cuda_fail(e);
  cudaStream_t s = nullptr;
  perks_status st = PERKS_OK;
  if ((e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) != cudaSuccess) { cudaFree(buf); return cg_cuda_fail(e); }
  if (h->n > 0) e = cudaMemcpyAsync(buf + ob_b, h_b, h->n * h->elem(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    st = perks_cg_solve(h, v, pol, buf + ob_b, buf + ob_x, kmax, tol, reinterpret_cast<double *>(buf + ob_h),
                        reinterpret_cast<int64_t *>(buf + ob_i), buf + ob_w, wsb, s);
    if (st == PERKS_OK) {
      if (h->n > 0) e = cudaMemcpyAsync(h_x, buf + ob_x, h->n * h->elem(), cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess && h_hist) e = cudaMemcpyAsync(h_hist, buf + ob_h, hb, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess && h_info) e = cudaMemcpyAsync(h_info, buf + ob_i, 16, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    }
  }
  cudaStreamDestroy(s);
  cudaFree(buf);
  if (st != PERKS_OK) return st;
  return e == cudaSuccess ? PERKS_OK : cg_cuda_fail(e);
}

perks_status perks_cg_query(perks_cg_t h, perks_variant v, perks_cg_policy pol, perks_cg_info *info) {
  if (!h || !info) return PERKS_ERR_INVALID_ARGUMENT;
  if ((int)v < PERKS_AUTO || (int)v > PERKS_PERKS || (int)pol < PERKS_CG_AUTO || (int)pol > PERKS_CG_MIX)
    return PERKS_ERR_INVALID_ARGUMENT;
  const CgPlan pl = make_plan(h, v, pol);
  std::memset(info, 0, sizeof(*info));
  info->variant = pl.variant;
  info->policy = pl.policy;
  info->grid = h->G;
  info->block = NT;
  info->items_per_thread = IPT;
  info->tiles = h->ntiles;
  info->smem_per_cta = pl.variant == PERKS_HOSTLOOP ? (h->dtype == PERKS_F64 ? smem_bytes<double>(0, true, 0)
                                                                             : smem_bytes<float>(0, true, 0))
                                                    : pl.smem;
  DevGuard g(h->device);
  cudaFuncAttributes fa{};
  const void *kfn = h->dtype == PERKS_F64
                        ? (pl.variant == PERKS_HOSTLOOP ? (const void *)cg_hl_a_kernel<double>
                           : pl.vec                     ? (const void *)cg_persistent_kernel<double, true>
                                                        : (const void *)cg_persistent_kernel<double, false>)
                        : (pl.variant == PERKS_HOSTLOOP ? (const void *)cg_hl_a_kernel<float>
                           : pl.vec                     ? (const void *)cg_persistent_kernel<float, true>
                                                        : (const void *)cg_persistent_kernel<float, false>);
  if (g.ok && cudaFuncGetAttributes(&fa, kfn) == cudaSuccess) info->regs_per_thread = fa.numRegs;
  else cudaGetLastError();
  info->cached_nnz_smem = pl.cached_nnz;
  info->cached_rows_smem = pl.cached_rows;
  info->n_rows = h->n;
  info->nnz = h->nnz;
  info->dram_bytes_per_iter = pl.dram;
  info->unfused_bytes_per_iter = pl.unfused;
  info->workspace_bytes = ws_layout(h).ws_bytes;
  static const char *pn[] = {"auto", "imp", "vec", "mat", "mix"};
  std::snprintf(info->kernel_name, sizeof(info->kernel_name), "cg_%s_%s_%s",
                pl.variant == PERKS_HOSTLOOP ? "hostloop" : pl.variant == PERKS_PERSISTENT ? "persistent" : "perks",
                pn[pl.policy], h->dtype == PERKS_F64 ? "f64" : "f32");
  return PERKS_OK;
}

perks_status perks_cg_partition(perks_cg_t h, int64_t *rows, int32_t cap) {
  if (!h || !rows || cap < h->G + 1) return PERKS_ERR_INVALID_ARGUMENT;
  for (int c = 0; c <= h->G; ++c) rows[c] = h->h_crow[c];
  return PERKS_OK;
}

perks_status perks_cg_destroy(perks_cg_t h) {
  if (!h) return PERKS_ERR_INVALID_ARGUMENT;
  {
    DevGuard g(h->device);
    cudaFree(h->d_mem);
  }
  delete h;
  return PERKS_OK;
}

}  // extern "C"
