// cg.cu — PERKS conjugate gradient (include/perks/perks_cg.h).
//
// The paper's second case study: CG (Algorithm) with a
// merge-based SpMV, run (a) as a host loop of kernels, (b) as one persistent
// kernel with device-wide barriers, (c) as PERKS with the cache policies IMP / VEC / MAT / MIX
// (P:1749-1766).  B200 design (DESIGN.md §5 "CG"):
//
//   * Partition (the paper's "TB-level search", saved once because "the matrix is static
//     throughout the entire iteration").  CTA c owns a row-aligned share [R_c, R_{c+1})
//     of the merge path of (row ends, nonzeros), so A p of its own rows is complete inside the
//     CTA and never leaves the SM.
//   * Thread-level work (the "thread-level search", also static, so done once at create): the
//     share is a sequence of ITEMS — each nonzero of each row in storage order, an empty row
//     contributing one zero item — cut into tiles of NT*IPT items, thread t of a tile owning IPT
//     consecutive items.  Each item stores (value, column | END) where END marks the last item
//     of a row; each thread has a header (its first row | OPEN, OPEN = that row began in an
//     earlier thread).  Items are stored thread-interleaved ([e*NT + t]) so every warp load is
//     coalesced.  This is the merge path with its search results precomputed: no per-iteration
//     search, no row-offset reads, and the per-thread walk is a fully unrolled chain over
//     registers: acc = fma(val, p[col], acc), a row ends -> store (bit-identical to the oracle's
//     row sum unless the row is split between threads).
//   * Rows split between threads or tiles: the thread whose first row is OPEN combines the
//     partial sums of the preceding threads (and the previous tile's carry) in thread order —
//     a fixed order, so every launch, variant and policy produces the same bits.
//   * Where the items live across iterations (MAT / MIX): the first tiles of each CTA in Tensor
//     Memory (each thread's items in its own TMEM lane/columns, read back with tcgen05.ld straight
//     into the registers that use them; sm_100a's 256 KiB/SM that a non-contraction leaves idle),
//     the next in shared memory (bulk-copied once at the start), the rest streamed from HBM with
//     coalesced loads every iteration.
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

#ifndef PERKS_CG_IPT
#define PERKS_CG_IPT 12
#endif
#ifndef PERKS_CG_NT
#define PERKS_CG_NT 512
#endif
#ifndef PERKS_CG_CPS
#define PERKS_CG_CPS 1
#endif
// One CTA of 512 threads per SM.  Two CTAs of 256 per SM (the paper's TB/SM knob)
// would overlap one CTA's per-tile barrier with the other's work, but a kernel containing
// tcgen05.alloc is limited to one CTA per SM by the occupancy calculator (measured:
// cudaOccupancyMaxActiveBlocksPerMultiprocessor = 1 at any register/shared-memory footprint),
// so the TMEM tier and CPS > 1 exclude each other in a cooperative launch.
#ifndef PERKS_CG_MAXREG  // two 256-thread CTAs per SM need <= 120 registers (measured occupancy)
#define PERKS_CG_MAXREG (PERKS_CG_CPS > 1 ? 120 : 128)
#endif
constexpr int NT = PERKS_CG_NT;     // threads per CTA
constexpr int CPS = PERKS_CG_CPS;   // co-resident CTAs per SM
constexpr int IPT = PERKS_CG_IPT;   // items per thread per tile
constexpr int TI = NT * IPT;        // items per tile
constexpr int kSmemMax = 227 * 1024 / PERKS_CG_CPS - (PERKS_CG_CPS > 1 ? 1024 : 0);
constexpr int kMaxG = 512;
constexpr int PAD = 0x7fffffff;     // an empty item slot (after the CTA's last item)
constexpr int COLMASK = 0x7fffffff; // column bits of an item word; 0x7fffffff = no column
constexpr int TMEM_COLS = 512 / CPS;  // the CTAs of an SM split its 512 TMEM columns
// warps w, w+4, ... share lane quarter w%4: each thread gets its share of the CTA's columns
constexpr int TMEM_COLS_PER_THREAD = TMEM_COLS / (NT / 128);
static_assert(NT % 128 == 0 && TMEM_COLS >= 32, "TMEM geometry");

// Bytes of one tile record (global and shared memory): values [TI] | item words [TI] | headers [NT].
template <typename T> constexpr int tile_bytes() { return TI * ((int)sizeof(T) + 4) + NT * 4; }
// TMEM words per thread per tile (values, item words, header), rounded to 8-column loads.
template <typename T> constexpr int tmem_wpt() { return (IPT * (int)sizeof(T) / 4 + IPT + 1 + 7) / 8 * 8; }
template <typename T> constexpr int tmem_tiles() { return TMEM_COLS_PER_THREAD / tmem_wpt<T>(); }

template <typename T> struct Params {
  int n, G;
  const unsigned char *tiles;  // tile records, CTA c's at [ctile[c], ctile[c+1])
  const int *ctile;            // G+1
  const int *crow;             // G+1 row boundaries
  const T *b;
  T *x;                        // output
  T *r, *p0, *p1, *q;          // workspace vectors (global)
  const T *xin;                // spmv: input vector (output in q)
  double *slots;               // 2*G partial sums
  double *scal;                // host loop: <r,r> by iteration parity [2]
  long long *state;            // host loop: [0] done, [1] iterations, [2] status
  unsigned *bar;               // grid barrier words
  unsigned long long *dbg;     // nullable: phase timer (PERKS_CG_TIMING)
  double *hist;                // nullable, kmax+1
  long long *info;             // nullable, 2
  long long kmax;
  double tol2;
  int rows_max;                // max own rows over CTAs (VEC arrays)
  int tm_tiles;                // tiles per CTA resident in TMEM (MAT)
  int sm_tiles;                // tiles per CTA resident in shared memory (MAT)
  int nbuf;                    // stream ring buffers (0: direct loads)
  int fused;                   // persistent: 2 barriers/iteration (p recomputed at the gather)
};

// Dynamic shared memory layout.
struct Smem {
  static constexpr int RED = 0;                        // 32 doubles
  static constexpr int MBAR = RED + 256;               // mbarriers: resident tiles, ring [<= 7]
  static constexpr int TMEMB = MBAR + 64;              // TMEM base address
  static constexpr int BCAST = TMEMB + 16;             // reduction broadcasts [4] (doubles)
  static constexpr int TCAR = BCAST + 32;              // tile carries [2]: row, have, value (16 B each)
  static constexpr int CROW = TCAR + 32;               // [2][NT] ints: carry row | HAVE
  static constexpr int CVAL = CROW + 2 * NT * 4;       // [2][NT] T (8-byte slots)
  static constexpr int VEC = CVAL + 2 * NT * 8;        // VEC arrays, then resident tiles
};
__host__ __device__ inline int a16(long long b) { return (int)((b + 15) & ~15ll); }
template <typename T> inline int smem_bytes(int vec_rows, int nbuf, int sm_tiles) {
  return Smem::VEC + 4 * a16((long long)vec_rows * (int)sizeof(T)) + (nbuf + sm_tiles) * tile_bytes<T>();
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
PERKS_DEVINL double slots_sum(const double *slots, int G, double *s_bc) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double t = 0.0;
    for (int j0 = 0; j0 < G; j0 += 4 * 32) {  // 4 loads in flight, summed in order
      double v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = j0 + 32 * j + lane;
        v[j] = c < G ? __ldcg(slots + c) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) t += v[j];
    }
    t = warp_sum(t);
    if (lane == 0) *s_bc = t;
  }
  __syncthreads();
  return *s_bc;
}

// ------------------------------------------------------------------------ tiles
// One thread's items of one tile, in registers.
template <typename T> struct Items {
  T v[IPT];
  int w[IPT];  // column | END (bit 31); PAD = empty slot
  int hdr;     // first row | OPEN (bit 31)
};

template <typename T>
PERKS_DEVINL void items_from(const unsigned char *rec, Items<T> &it, bool stream) {
  const T *val = reinterpret_cast<const T *>(rec);
  const int *wrd = reinterpret_cast<const int *>(rec + TI * sizeof(T));
  const int *hdr = reinterpret_cast<const int *>(rec + TI * (sizeof(T) + 4));
  const int t = threadIdx.x;
  if (stream) {  // HBM stream: read once per iteration, do not keep in L1
#pragma unroll
    for (int e = 0; e < IPT; ++e) { it.v[e] = __ldcs(val + e * NT + t); it.w[e] = __ldcs(wrd + e * NT + t); }
    it.hdr = __ldcs(hdr + t);
  } else {       // shared-memory resident tile
#pragma unroll
    for (int e = 0; e < IPT; ++e) { it.v[e] = val[e * NT + t]; it.w[e] = wrd[e * NT + t]; }
    it.hdr = hdr[t];
  }
}

// TMEM: thread (warp w, lane l) owns lane 32*(w%4)+l, columns (w/4)*128 + slot*WPT .. +WPT.
template <typename T> PERKS_DEVINL uint32_t tmem_addr(uint32_t base, int slot) {
  const int w = threadIdx.x >> 5;
  return base + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * TMEM_COLS_PER_THREAD + slot * tmem_wpt<T>());
}
template <typename T> PERKS_DEVINL void items_to_tmem(uint32_t taddr, const Items<T> &it) {
  constexpr int W = tmem_wpt<T>();
  uint32_t wd[W];
#pragma unroll
  for (int i = 0; i < W; ++i) wd[i] = 0;
#pragma unroll
  for (int e = 0; e < IPT; ++e) {
    if constexpr (sizeof(T) == 8) {
      const unsigned long long b = (unsigned long long)__double_as_longlong((double)it.v[e]);
      wd[2 * e] = (uint32_t)b;
      wd[2 * e + 1] = (uint32_t)(b >> 32);
    } else {
      wd[e] = __float_as_uint((float)it.v[e]);
    }
    wd[IPT * sizeof(T) / 4 + e] = (uint32_t)it.w[e];
  }
  wd[IPT * sizeof(T) / 4 + IPT] = (uint32_t)it.hdr;
#pragma unroll
  for (int g = 0; g < W / 8; ++g) {
    uint32_t c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = wd[8 * g + j];
    tmem_st8(taddr + 8 * g, c);
  }
}
template <typename T> PERKS_DEVINL void items_from_tmem(uint32_t taddr, Items<T> &it) {
  constexpr int W = tmem_wpt<T>();
  uint32_t wd[W];
#pragma unroll
  for (int g = 0; g < W / 8; ++g) {
    uint32_t c[8];
    tmem_ld8(taddr + 8 * g, c);
#pragma unroll
    for (int j = 0; j < 8; ++j) wd[8 * g + j] = c[j];
  }
  tmem_wait_ld();
#pragma unroll
  for (int e = 0; e < IPT; ++e) {
    if constexpr (sizeof(T) == 8)
      it.v[e] = (T)__longlong_as_double((long long)((unsigned long long)wd[2 * e] | ((unsigned long long)wd[2 * e + 1] << 32)));
    else
      it.v[e] = (T)__uint_as_float(wd[e]);
    it.w[e] = (int)wd[IPT * sizeof(T) / 4 + e];
  }
  it.hdr = (int)wd[IPT * sizeof(T) / 4 + IPT];
}

// Tile carry between consecutive tiles of one CTA: the partial sum of the row a tile ends in.
template <typename T> struct TileCarry {
  int row, have;
  T val;
};

// SpMV of one tile's items (see the header comment).  gather.load(col, a, b) issues the loads
// for column `col` (col < 0: none), gather.value(col, a, b) returns the vector value;
// qstore(row, v) stores a completed row.  `m` = tile index in the CTA (parity of the carry
// buffers); `last` = no carry into a next tile.  Contains one __syncthreads (between the walk
// and the carry fix-up); the fix-up's q stores become visible after the caller's next barrier.
template <typename T, class Gather, class QStore>
PERKS_DEVINL void tile_spmv(const Items<T> &it, unsigned char *smem, int m, bool last, const Gather &gather,
                            QStore qstore) {
  const int par = m & 1;
  int *s_crow = reinterpret_cast<int *>(smem + Smem::CROW) + par * NT;
  T *s_cval = reinterpret_cast<T *>(smem + Smem::CVAL + par * NT * 8);
  const TileCarry<T> *tc = reinterpret_cast<TileCarry<T> *>(smem + Smem::TCAR) + par;
  TileCarry<T> *tn = reinterpret_cast<TileCarry<T> *>(smem + Smem::TCAR) + (par ^ 1);
  const int tid = threadIdx.x;
  // gathers: every load issued before any is used
  int jc[IPT];
  T ga[IPT], gb[IPT];
#pragma unroll
  for (int e = 0; e < IPT; ++e) {
    const int c = it.w[e] & COLMASK;  // PAD and empty-row items carry no column
    jc[e] = c == COLMASK ? -1 : c;
    gather.load(jc[e], ga[e], gb[e]);
  }
  // the walk: an unrolled fma chain per row segment
  int row = it.hdr & 0x7fffffff;
  bool open = it.hdr < 0;
  T acc = T(0), sval = T(0);
  bool have = false;
  int srow = -1;
  // (PAD slots only follow the CTA's last row: their zero terms and `have` are never read)
#pragma unroll
  for (int e = 0; e < IPT; ++e) {
    acc = fma_rn(it.v[e], gather.value(jc[e], ga[e], gb[e]), acc);
    have = true;
    if (it.w[e] < 0) {  // END: row complete
      if (open) { srow = row; sval = acc; open = false; }
      else qstore(row, acc);
      acc = T(0);
      have = false;
      ++row;
    }
  }
  s_crow[tid] = row | (have ? (int)0x80000000 : 0);
  s_cval[tid] = acc;
  __syncthreads();
  if (srow >= 0) {  // the first row of this thread began earlier: partials in thread order
    const int key = srow | (int)0x80000000;
    int t0 = tid;
    while (t0 > 0 && s_crow[t0 - 1] == key) --t0;
    bool h = false;
    T v = T(0);
    if (t0 == 0 && tc->have && tc->row == srow) { v = tc->val; h = true; }
    for (int u = t0; u < tid; ++u) { v = h ? v + s_cval[u] : s_cval[u]; h = true; }
    qstore(srow, h ? v + sval : sval);
  }
  if (!last && tid == NT - 1) {  // carry into the next tile (full tiles only: no padding)
    const int key = s_crow[NT - 1];
    TileCarry<T> o;
    o.row = key & 0x7fffffff;
    o.have = 0;
    o.val = T(0);
    if (key < 0) {
      int t0 = NT;
      while (t0 > 0 && s_crow[t0 - 1] == key) --t0;
      bool h = false;
      T v = T(0);
      if (t0 == 0 && tc->have && tc->row == o.row) { v = tc->val; h = true; }
      for (int u = t0; u < NT; ++u) { v = h ? v + s_cval[u] : s_cval[u]; h = true; }
      o.have = 1;
      o.val = v;
    }
    *tn = o;
  }
}

// Tiles of CTA c: the first tm in TMEM, the next sm in shared memory, the rest streamed — through
// a ring of nb shared-memory buffers filled by bulk copies (TMA, mbarrier completion) issued nb
// tiles ahead of the consumer (nb = 0: coalesced loads straight into registers).  Persistent
// launches keep streaming across iteration boundaries (the next iteration's first tiles load
// during the all-reduces); `issued` counts streamed sequence numbers issued, `u` consumed.
struct TileSet {
  int tb, nt, tm, sm, nb;
  uint32_t tbase;             // TMEM base address (tm > 0)
  const unsigned char *sres;  // shared-memory resident tiles
  unsigned char *ring;        // nb stream buffers
  long long u, issued;
  bool wrap;
};

template <typename T> PERKS_DEVINL void ring_issue(const Params<T> &P, TileSet &ts, unsigned char *smem) {
  // thread 0 only
  const int first = ts.tm + ts.sm, ns = ts.nt - first;
  if (ts.nb == 0 || ns <= 0) return;
  uint64_t *mb = reinterpret_cast<uint64_t *>(smem + Smem::MBAR) + 1;
  while (ts.issued < ts.u + ts.nb && (ts.wrap || ts.issued < ns)) {
    const int m = first + (int)(ts.issued % ns);
    const int b = (int)(ts.issued % ts.nb);
    mbar_arrive_tx(mb + b, (unsigned)tile_bytes<T>());
    bulk_load(ts.ring + (size_t)b * tile_bytes<T>(), P.tiles + (size_t)(ts.tb + m) * tile_bytes<T>(),
              (unsigned)tile_bytes<T>(), mb + b);
    ++ts.issued;
  }
}

template <typename T, class Gather, class QStore>
PERKS_DEVINL void spmv_cta(const Params<T> &P, TileSet &ts, unsigned char *smem, const Gather &gather,
                           QStore qstore) {
  if (threadIdx.x == 0) reinterpret_cast<TileCarry<T> *>(smem + Smem::TCAR)->have = 0;
  // (the carry reset is read only after the first tile's __syncthreads)
  uint64_t *mb = reinterpret_cast<uint64_t *>(smem + Smem::MBAR) + 1;
  for (int m = 0; m < ts.nt; ++m) {
    Items<T> it;
    const bool streamed = m >= ts.tm + ts.sm;
    if (m < ts.tm) {
      items_from_tmem<T>(tmem_addr<T>(ts.tbase, m), it);
    } else if (!streamed) {
      items_from<T>(ts.sres + (size_t)(m - ts.tm) * tile_bytes<T>(), it, false);
    } else if (ts.nb > 0) {
      const int b = (int)(ts.u % ts.nb);
      mbar_wait(mb + b, (unsigned)((ts.u / ts.nb) & 1));
      items_from<T>(ts.ring + (size_t)b * tile_bytes<T>(), it, false);
    } else {
      items_from<T>(P.tiles + (size_t)(ts.tb + m) * tile_bytes<T>(), it, true);
    }
    tile_spmv<T>(it, smem, m, m == ts.nt - 1, gather, qstore);
    // (tile_spmv's __syncthreads follows every thread's item reads: the ring slot is free)
    if (streamed && ts.nb > 0) {
      ++ts.u;
      if (threadIdx.x == 0) ring_issue<T>(P, ts, smem);
    }
  }
  __syncthreads();  // the last fix-up's stores before anyone reads q
}

// Resident tiles (persistent MAT/MIX): TMEM tiles through registers, shared-memory tiles by one
// bulk copy each; the stream ring's first copies.  Returns the CTA's tile set.
template <typename T>
PERKS_DEVINL TileSet tiles_init(const Params<T> &P, unsigned char *smem, int vec_rows, bool resident, bool wrap) {
  TileSet ts;
  const int c = blockIdx.x;
  ts.tb = P.ctile[c];
  ts.nt = P.ctile[c + 1] - ts.tb;
  ts.tm = resident ? min(ts.nt, P.tm_tiles) : 0;
  ts.sm = resident ? min(ts.nt - ts.tm, P.sm_tiles) : 0;
  ts.nb = P.nbuf;
  ts.tbase = 0;
  ts.ring = smem + Smem::VEC + 4 * a16((long long)vec_rows * (int)sizeof(T));
  ts.sres = ts.ring + (size_t)ts.nb * tile_bytes<T>();
  ts.u = 0;
  ts.issued = 0;
  ts.wrap = wrap;
  uint64_t *mb = reinterpret_cast<uint64_t *>(smem + Smem::MBAR);
  if (threadIdx.x == 0) {
    for (int b = 0; b <= ts.nb; ++b) mbar_init(mb + b, 1);
    mbar_fence_init();
    if (ts.sm > 0) {
      mbar_arrive_tx(mb, (unsigned)(ts.sm * tile_bytes<T>()));
      for (int s = 0; s < ts.sm; ++s)
        bulk_load(const_cast<unsigned char *>(ts.sres) + (size_t)s * tile_bytes<T>(),
                  P.tiles + (size_t)(ts.tb + ts.tm + s) * tile_bytes<T>(), (unsigned)tile_bytes<T>(), mb);
    }
    ring_issue<T>(P, ts, smem);
  }
  if (ts.tm > 0) {
    uint32_t *s_tb = reinterpret_cast<uint32_t *>(smem + Smem::TMEMB);
    if (threadIdx.x < 32) {
      tmem_alloc(s_tb, TMEM_COLS);
      tmem_relinquish();
    }
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
    ts.tbase = *s_tb;
    for (int m = 0; m < ts.tm; ++m) {
      Items<T> it;
      items_from<T>(P.tiles + (size_t)(ts.tb + m) * tile_bytes<T>(), it, true);
      items_to_tmem<T>(tmem_addr<T>(ts.tbase, m), it);
    }
    tmem_wait_st();
  }
  if (ts.sm > 0) mbar_wait(mb, 0);
  __syncthreads();
  return ts;
}

template <typename T> PERKS_DEVINL void tiles_fini(TileSet &ts, unsigned char *smem) {
  // every issued bulk copy must land before the CTA exits
  uint64_t *mb = reinterpret_cast<uint64_t *>(smem + Smem::MBAR) + 1;
  if (threadIdx.x == 0)
    for (long long v = ts.u; v < ts.issued; ++v) mbar_wait(mb + (v % ts.nb), (unsigned)((v / ts.nb) & 1));
  if (ts.tm > 0) {
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
    if (threadIdx.x < 32) tmem_dealloc(ts.tbase, TMEM_COLS);
  }
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
  unsigned char *v = smem + Smem::VEC;
  o.s_r = reinterpret_cast<T *>(v);
  o.s_x = reinterpret_cast<T *>(v + vb);
  o.s_p = reinterpret_cast<T *>(v + 2 * vb);
  o.s_q = reinterpret_cast<T *>(v + 3 * vb);
  return o;
}

// x_0 = 0, r_0 = b, p_{-1} = 0 (published for the gathers); returns this thread's part of
// <r_0, r_0>.
template <typename T, bool VEC> PERKS_DEVINL double cg_prologue(const Params<T> &P, const Own<T, VEC> &o) {
  double acc = 0.0;
  for (int j = threadIdx.x; j < o.rows; j += NT) {
    const int i = o.R0 + j;
    const T bi = P.b[i];
    if (VEC) { o.s_x[j] = T(0); o.s_r[j] = bi; o.s_p[j] = T(0); }
    else P.x[i] = T(0);
    P.r[i] = bi;
    P.p1[i] = T(0);  // p_{-1} = 0: p_0 = fma(0, p_{-1}, r_0) = r_0 with the general update
    acc = fma_rn((double)bi, (double)bi, acc);
  }
  return acc;
}

// Vector loads (p, r, x, A p).  Plain, L1-cacheable loads: every value another CTA wrote is
// read only after a grid barrier whose acquire (thread 0) and __syncthreads order it before the
// load (and the acquire invalidates the SM's L1), and the own CTA's writes go through L1.  The
// gathers reuse p[j] across neighbouring rows, so L1 hits matter: with L2-only (.cg) loads every
// CTA but the first ran 1.5x slower on the stencil-like matrices (profiles/r02_cg_*).
template <typename T> PERKS_DEVINL T ldv(const T *p) { return *p; }

// Own-row passes visit rows j = tid, tid+NT, ... in that order (the order of every per-thread
// inner-product chain); U rows per batch so their loads are in flight together.
constexpr int U = 4;

// p_k (own rows) = fma(beta, p_{k-1}, r_k) (k = 0: beta = 0 and p_{-1} = 0, so p_0 = r_0),
// published into pcur.
template <typename T, bool VEC>
PERKS_DEVINL void cg_p_update(const Params<T> &P, const Own<T, VEC> &o, T beta, const T *pprev, T *pcur) {
  for (int j0 = threadIdx.x; j0 < o.rows; j0 += U * NT) {
    T r[U], pp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * NT, i = o.R0 + j;
      const bool ok = j < o.rows;
      r[u] = ok ? (VEC ? o.s_r[j] : ldv(P.r + i)) : T(0);
      pp[u] = ok ? (VEC ? o.s_p[j] : ldv(pprev + i)) : T(0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * NT;
      if (j < o.rows) {
        const T p = fma_rn(beta, pp[u], r[u]);
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
      p[u] = ok ? (VEC ? o.s_p[j] : ldv(pcur + i)) : T(0);
      q[u] = ok ? (VEC ? o.s_q[j] : ldv(P.q + i)) : T(0);
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
        p[u] = ok ? ldv(pcur + i) : T(0); q[u] = ok ? ldv(P.q + i) : T(0);
        x[u] = ok ? ldv(P.x + i) : T(0); r[u] = ok ? ldv(P.r + i) : T(0);
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

// Gather of p_k at column jc for the SpMV of iteration k.
//   FUSED (two barriers per iteration): own columns from the buffer this CTA just wrote, other
//   CTAs' columns recomputed as fma(beta, p_{k-1}, r_k) from their published p_{k-1} and r_k (the
//   owner computed p_k with the same fma: identical values).
//   !FUSED (three barriers): every CTA published p_k before a grid barrier; one load.
// load() issues the loads (branch-free: selects and a predicated second load), value()
// combines them.  jc = -1: no column (padding / empty row), value 0.
template <typename T, bool FUSED> struct CgGather {
  int R0, rows;
  T beta;
  const T *pcur, *pprev, *r;
  PERKS_DEVINL void load(int jc, T &a, T &b) const {
    const int j = jc < 0 ? 0 : jc;
    if (!FUSED) {
      a = ldv(pcur + j);
      b = T(0);
      return;
    }
    const bool own = (unsigned)(j - R0) < (unsigned)rows;
    a = ldv((own ? pcur : pprev) + j);
    b = own ? T(0) : ldv(r + j);
  }
  PERKS_DEVINL T value(int jc, T a, T b) const {
    if (jc < 0) return T(0);
    if (!FUSED) return a;
    const bool own = (unsigned)(jc - R0) < (unsigned)rows;
    return own ? a : fma_rn(beta, a, b);
  }
};

template <typename T> struct PlainGather {  // standalone SpMV: x[j]
  const T *x;
  PERKS_DEVINL void load(int j, T &a, T &b) const {
    a = __ldg(x + (j < 0 ? 0 : j));
    b = T(0);
  }
  PERKS_DEVINL T value(int j, T a, T) const { return j < 0 ? T(0) : a; }
};

template <typename T, bool VEC>
PERKS_DEVINL void cg_spmv(const Params<T> &P, const Own<T, VEC> &o, TileSet &ts, unsigned char *smem, bool fused,
                          T beta, const T *pprev, const T *pcur) {
  const int R0 = o.R0;
  T *q = P.q;
  T *sq = o.s_q;
  auto qstore = [=](int row, T v) {
    if (VEC) sq[row - R0] = v;
    else q[row] = v;
  };
  if (fused) spmv_cta<T>(P, ts, smem, CgGather<T, true>{o.R0, o.rows, beta, pcur, pprev, P.r}, qstore);
  else spmv_cta<T>(P, ts, smem, CgGather<T, false>{o.R0, o.rows, beta, pcur, pprev, P.r}, qstore);
}

// ------------------------------------------------------------------------ kernels
// Phase timer (development, PERKS_CG_TIMING=1): CTA 0 / thread 0 accumulates globaltimer deltas
// per phase into P.dbg[0..3] (0 p update, 1 SpMV, 2 <p,Ap> + all-reduce, 3 x/r update +
// all-reduce); P.dbg[8] += iterations.
// Every CTA's thread 0 also adds its own SpMV time to P.dbg[16 + c] (load balance).
struct PhaseClock {
  unsigned long long *dbg;
  unsigned long long t;
  PERKS_DEVINL explicit PhaseClock(unsigned long long *d) : dbg(threadIdx.x == 0 ? d : nullptr), t(0) {
    if (dbg) {
      t = globaltimer_ns();
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      dbg[16 + kMaxG + blockIdx.x] = smid;
    }
  }
  PERKS_DEVINL void tick(int ph) {
    if (dbg) {
      const unsigned long long n = globaltimer_ns();
      if (blockIdx.x == 0) dbg[ph] += n - t;
      if (ph == 1) dbg[16 + blockIdx.x] += n - t;
      t = n;
    }
  }
};

// (b)/(c): the whole solve in one cooperative launch.
template <typename T, bool VEC> __global__ void __maxnreg__(PERKS_CG_MAXREG) cg_persistent_kernel(Params<T> P) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *s_red = reinterpret_cast<double *>(smem + Smem::RED);
  double *s_bc = reinterpret_cast<double *>(smem + Smem::BCAST);
  const Own<T, VEC> o = own_view<T, VEC>(P, smem);
  TileSet ts = tiles_init<T>(P, smem, VEC ? P.rows_max : 0, true, true);
  const int c = blockIdx.x;
  // all-reduce of the per-CTA partials: slot write, grid barrier, slot read in a fixed order
  // (kind 0 = <p,Ap>, 1 = <r,r>).  A barrier-free variant with tagged (LL) slots polled by every
  // CTA was measured slower on B200 (G2 12.9 vs 9.6 us/iteration: 148 pollers on one set of L2
  // lines) and removed.
  unsigned nb = 0;
  auto allreduce = [&](int kind, double part, double *bc) -> double {
    if (threadIdx.x == 0) P.slots[kind * P.G + c] = part;
    grid_barrier(P.bar, ++nb);
    return slots_sum(P.slots + kind * P.G, P.G, bc);
  };
  double part = block_sum(cg_prologue<T, VEC>(P, o), s_red);
  double rr = allreduce(1, part, s_bc);  // (the barrier also publishes r_0 = b, p_{-1} = 0)
  if (c == 0 && threadIdx.x == 0 && P.hist) P.hist[0] = rr;
  PhaseClock clk(P.dbg);
  long long k = 0;
  int status = 0;
  double beta = 0.0;
  while (k < P.kmax) {
    if (!(rr > P.tol2)) break;  // reading RC2: <r_k,r_k> <= tol^2 stops before the iteration
    T *pcur = (k & 1) ? P.p1 : P.p0;
    const T *pprev = (k & 1) ? P.p0 : P.p1;
    const T bt = (T)beta;
    cg_p_update<T, VEC>(P, o, bt, pprev, pcur);
    if (P.fused) __syncthreads();
    else grid_barrier(P.bar, ++nb);  // every CTA's p_k published before the gathers
    clk.tick(0);
    cg_spmv<T, VEC>(P, o, ts, smem, P.fused, bt, pprev, pcur);
    clk.tick(1);
    part = block_sum(cg_pap<T, VEC>(P, o, pcur), s_red);
    const double pap = allreduce(0, part, s_bc + 1);
    clk.tick(2);
    if (!(pap > 0.0)) { status = 1; break; }  // reading RC4: not positive definite
    const double alpha = rr / pap;
    part = block_sum(cg_xr_update<T, VEC>(P, o, (T)alpha, pcur), s_red);
    const double rr_new = allreduce(1, part, s_bc + 2);  // (publishes r_{k+1} for fused gathers)
    clk.tick(3);
    beta = rr_new / rr;
    rr = rr_new;
    ++k;
    if (c == 0 && threadIdx.x == 0 && P.hist) P.hist[k] = rr;
  }
  if (clk.dbg && c == 0) clk.dbg[8] += k;
  if (VEC)
    for (int j = threadIdx.x; j < o.rows; j += NT) P.x[o.R0 + j] = o.s_x[j];
  if (c == 0 && threadIdx.x == 0 && P.info) { P.info[0] = k; P.info[1] = status; }
  tiles_fini<T>(ts, smem);
}

// (a) host loop: prologue, then per iteration kernel A (p update, SpMV, <p,Ap>) and kernel B
// (x/r update, <r,r>), then a finishing kernel.  Same partition, same arithmetic, same order.
template <typename T> __global__ void __launch_bounds__(NT, 1) cg_hl_prologue_kernel(Params<T> P) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *s_red = reinterpret_cast<double *>(smem + Smem::RED);
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
  TileSet ts = tiles_init<T>(P, smem, 0, false, false);
  T *pcur = (k & 1) ? P.p1 : P.p0;
  const T *pprev = (k & 1) ? P.p0 : P.p1;
  const T bt = (T)beta;
  cg_p_update<T, false>(P, o, bt, pprev, pcur);
  __syncthreads();
  cg_spmv<T, false>(P, o, ts, smem, true, bt, pprev, pcur);
  const double part = block_sum(cg_pap<T, false>(P, o, pcur), s_red);
  if (threadIdx.x == 0) P.slots[c] = part;
  tiles_fini<T>(ts, smem);
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
  TileSet ts = tiles_init<T>(P, smem, 0, false, false);
  const PlainGather<T> gather{P.xin};
  T *y = P.q;
  auto qstore = [=](int row, T v) { y[row] = v; };
  spmv_cta<T>(P, ts, smem, gather, qstore);
  tiles_fini<T>(ts, smem);
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
  int ntiles = 0;                   // tiles over all CTAs
  int tiles_max = 0;                // most tiles of one CTA
  std::vector<int> h_crow;          // G+1
  std::vector<int> h_ctile;         // G+1
  void *d_mem = nullptr;            // one allocation: tiles | ctile | crow
  unsigned char *d_tiles = nullptr;
  int *d_ctile = nullptr, *d_crow = nullptr;
  std::mutex mu;
  // solve_host scratch (device buffers + stream), kept across calls, grown on demand
  char *hbuf = nullptr;
  size_t hbuf_bytes = 0;
  cudaStream_t hstream = nullptr;
  size_t elem() const { return dtype == PERKS_F64 ? 8 : 4; }
};

namespace {

// Merge-path search on the global CSR: (rows completed, nonzeros consumed) at diagonal d.
void path_coord(const int64_t *ro, int64_t n, int64_t nnz, int64_t d, int64_t &i, int64_t &k) {
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
  size_t ws_bytes, off_r, off_p0, off_p1, off_q, off_slots, off_scal, off_state, off_bar, off_dbg;
};
Layout ws_layout(const perks_cg_s *h) {
  Layout L{};
  const size_t vb = align256((size_t)std::max<int64_t>(h->n, 1) * h->elem());
  size_t o = 0;
  L.off_bar = o; o += 256;
  L.off_dbg = o; o += 256 + 16 * kMaxG;  // bytes 256..: phase timer (tools/cg_timing.py reads it there)
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
  bool fused = true;    // persistent: 2 barriers/iteration (p_k recomputed at the gathers)
  int nbuf = 0;         // stream ring buffers
  int tm = 0, sm = 0;   // resident tiles per CTA: TMEM, shared memory
  int smem = 0;
  int64_t cached_items_tmem = 0, cached_items_smem = 0, cached_rows = 0;
  double dram = 0, unfused = 0;
};

CgPlan make_plan(const perks_cg_s *h, perks_variant v, perks_cg_policy pol) {
  CgPlan pl;
  if (v == PERKS_AUTO) v = PERKS_PERKS;
  if (pol == PERKS_CG_AUTO) pol = PERKS_CG_MIX;
  if (v == PERKS_HOSTLOOP || v == PERKS_PERSISTENT) pol = PERKS_CG_IMP;
  pl.variant = v;
  pl.policy = pol;
  const bool f64 = h->dtype == PERKS_F64;
  const int S = (int)h->elem();
  const int tb = f64 ? tile_bytes<double>() : tile_bytes<float>();
  const int vecb = 4 * a16((long long)h->rows_max * S);
  const bool mat = pol == PERKS_CG_MAT || pol == PERKS_CG_MIX;
  const int tmem_t = mat ? std::min(h->tiles_max, f64 ? tmem_tiles<double>() : tmem_tiles<float>()) : 0;
  const bool streams = h->tiles_max > tmem_t;
  // VEC only where it leaves room for a stream ring of two buffers (when the SpMV streams):
  // a one-deep ring costs more than the vector caching saves (G4: 67.5 vs 56.1 us/iteration)
  pl.vec = (pol == PERKS_CG_VEC || pol == PERKS_CG_MIX) &&
           Smem::VEC + vecb + (streams ? 2 * tb : 0) <= kSmemMax;
  const int base = Smem::VEC + (pl.vec ? vecb : 0);
  const int fit = std::max(0, (kSmemMax - base) / tb);  // tile records that fit next to VEC
  if (mat) {
    pl.tm = tmem_t;
    const int rest = h->tiles_max - pl.tm;
    if (rest <= fit) {
      pl.sm = rest;  // everything resident: no stream
    } else {         // keep a stream ring of up to 3 buffers, the rest resident
      pl.nbuf = std::min(fit, 3);
      pl.sm = fit - pl.nbuf;
    }
  } else if (h->tiles_max > 0) {
    pl.nbuf = std::min(fit, env_int("PERKS_CG_NBUF", 3));
  }
  pl.nbuf = std::min(pl.nbuf, 6);
  pl.smem = base + (pl.nbuf + pl.sm) * tb;
  // two barriers (p_k recomputed at the gathers) only for one-tile shares; from two tiles per CTA
  // up one gather load per nonzero costs more than the third barrier (measured: G2 9.0 vs 10.1,
  // G3 14.1 vs 13.5, G4 98.9 vs 84.7 us/iteration fused vs not; PERKS_CG_FUSED overrides)
  pl.fused = env_int("PERKS_CG_FUSED", h->tiles_max <= 1 ? 1 : 0) != 0;
  // each CTA allocates 512/CPS TMEM columns: at most CPS CTAs per SM (shared memory > 1/(CPS+1))
  if (pl.tm > 0) pl.smem = std::max(pl.smem, 228 * 1024 / (CPS + 1) + 1024);
  // what is cached, per CTA as tiles_init decides; bytes per iteration
  const int64_t items_total = (int64_t)h->ntiles * TI;
  for (int c = 0; c < h->G; ++c) {
    const int nt = h->h_ctile[c + 1] - h->h_ctile[c];
    const int tm = std::min(nt, pl.tm), sm = std::min(nt - tm, pl.sm);
    pl.cached_items_tmem += (int64_t)tm * TI;
    pl.cached_items_smem += (int64_t)sm * TI;
    if (pl.vec) pl.cached_rows += h->h_crow[c + 1] - h->h_crow[c];
  }
  // Unfused (the metric): A once in CSR (values, columns, row offsets), the gathered p once per
  // row, and the vector passes of Algorithm: p update (r, p read, p written), <p,Ap>
  // (p, q read), x update (x, p read, x written), r update (r, q read, r written), <r,r> (r
  // read) = 13 vector accesses per row, plus A p written once.
  const double n = (double)h->n, nnz = (double)h->nnz;
  pl.unfused = nnz * (S + 4) + (n + 1) * 4 + n * S * (1 + 13 + 1);
  // Modelled DRAM: streamed tile records + the vectors leaving the SM (r and p published and
  // gathered back: counted once each), plus own-row vector traffic without VEC.
  const double rec = (double)tb / TI;  // bytes per item slot incl. headers
  const double streamed = (double)(items_total - pl.cached_items_tmem - pl.cached_items_smem);
  pl.dram = streamed * rec + (pl.vec ? n * S * 2 : n * S * 11);
  return pl;
}

template <typename T> Params<T> make_params(perks_cg_s *h, void *ws, const CgPlan &pl) {
  const Layout L = ws_layout(h);
  unsigned char *w = static_cast<unsigned char *>(ws);
  Params<T> P{};
  P.n = (int)h->n;
  P.G = h->G;
  P.tiles = h->d_tiles;
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
  P.dbg = env_int("PERKS_CG_TIMING", 0) ? reinterpret_cast<unsigned long long *>(w + L.off_dbg) : nullptr;
  P.rows_max = h->rows_max;
  P.tm_tiles = pl.tm;
  P.sm_tiles = pl.sm;
  P.nbuf = pl.nbuf;
  P.fused = pl.fused ? 1 : 0;
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
    const int smem = smem_bytes<T>(0, pl.nbuf, 0);
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
  if ((e = cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared)) !=
      cudaSuccess)
    return e;
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
  int occ = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, NT, (size_t)pl.smem)) != cudaSuccess) return e;
  if (occ * h->num_sms < h->G) {
    return cudaErrorCooperativeLaunchTooLarge;
  }
  return cudaLaunchKernelExC(&cfg, kfn, args);
}

template <typename T> cudaError_t launch_spmv(perks_cg_s *h, const void *xin, void *y, void *ws, cudaStream_t s) {
  CgPlan pl = make_plan(h, PERKS_HOSTLOOP, PERKS_CG_IMP);
  Params<T> P = make_params<T>(h, ws, pl);
  P.xin = static_cast<const T *>(xin);
  P.q = static_cast<T *>(y);
  const int smem = smem_bytes<T>(0, pl.nbuf, 0);
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

// Build the item tiles of every CTA (see the header comment) into `buf` (tile records).
template <typename T>
void build_tiles(const perks_csr_desc *d, const std::vector<int> &crow, const std::vector<int> &ctile,
                 std::vector<unsigned char> &buf) {
  const int G = (int)crow.size() - 1;
  const size_t tbytes = tile_bytes<T>();
  buf.assign((size_t)ctile[G] * tbytes, 0);
  std::vector<int> irow, iword;
  std::vector<T> ival;
  std::vector<char> ifirst;
  for (int c = 0; c < G; ++c) {
    irow.clear(); iword.clear(); ival.clear(); ifirst.clear();
    for (int64_t i = crow[c]; i < crow[c + 1]; ++i) {
      const int64_t a = d->row_offsets[i], b = d->row_offsets[i + 1];
      if (a == b) {  // empty row: one zero item without a column
        irow.push_back((int)i); iword.push_back((int)0xffffffff); ival.push_back(T(0)); ifirst.push_back(1);
        continue;
      }
      for (int64_t k = a; k < b; ++k) {
        irow.push_back((int)i);
        iword.push_back(d->col_indices[k] | (k == b - 1 ? (int)0x80000000 : 0));
        ival.push_back((T)d->values[k]);  // rounded once (reading RC3)
        ifirst.push_back(k == a);
      }
    }
    const int64_t ni = (int64_t)irow.size();
    for (int m = 0; m < ctile[c + 1] - ctile[c]; ++m) {
      unsigned char *rec = buf.data() + (size_t)(ctile[c] + m) * tbytes;
      T *val = reinterpret_cast<T *>(rec);
      int *wrd = reinterpret_cast<int *>(rec + TI * sizeof(T));
      int *hdr = reinterpret_cast<int *>(rec + TI * (sizeof(T) + 4));
      for (int t = 0; t < NT; ++t) {
        const int64_t i0 = (int64_t)m * TI + (int64_t)t * IPT;
        hdr[t] = i0 < ni ? (irow[i0] | (ifirst[i0] ? 0 : (int)0x80000000)) : crow[c + 1];
        for (int e = 0; e < IPT; ++e) {
          const int64_t it = i0 + e;
          val[e * NT + t] = it < ni ? ival[it] : T(0);
          wrd[e * NT + t] = it < ni ? iword[it] : PAD;
        }
      }
    }
  }
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
  // CTA-level (TB-level) merge-path partition, row aligned
  const int64_t L = n + nnz;
  h->G = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(CPS * h->num_sms, kMaxG), (L + 1023) / 1024));
  h->h_crow.resize(h->G + 1);
  for (int c = 0; c <= h->G; ++c) {
    int64_t i, k;
    path_coord(d->row_offsets, n, nnz, L * c / h->G, i, k);
    h->h_crow[c] = (int)(c == h->G ? n : i);
  }
  // items per CTA (nonzeros + one per empty row) -> tiles
  h->h_ctile.assign(h->G + 1, 0);
  for (int c = 0; c < h->G; ++c) {
    h->rows_max = std::max(h->rows_max, h->h_crow[c + 1] - h->h_crow[c]);
    int64_t items = d->row_offsets[h->h_crow[c + 1]] - d->row_offsets[h->h_crow[c]];
    for (int64_t i = h->h_crow[c]; i < h->h_crow[c + 1]; ++i) items += d->row_offsets[i + 1] == d->row_offsets[i];
    const int nt = (int)((items + TI - 1) / TI);
    h->tiles_max = std::max(h->tiles_max, nt);
    h->h_ctile[c + 1] = h->h_ctile[c] + nt;
  }
  h->ntiles = h->h_ctile[h->G];
  std::vector<unsigned char> tiles;
  if (h->dtype == PERKS_F64) build_tiles<double>(d, h->h_crow, h->h_ctile, tiles);
  else build_tiles<float>(d, h->h_crow, h->h_ctile, tiles);
  const size_t b_t = align256(tiles.size() + 16), b_c = align256((h->G + 1) * 4);
  e = cudaMalloc(&h->d_mem, b_t + 2 * b_c);
  if (e != cudaSuccess) { delete h; return cg_cuda_fail(e); }
  char *m = static_cast<char *>(h->d_mem);
  h->d_tiles = reinterpret_cast<unsigned char *>(m);
  h->d_ctile = reinterpret_cast<int *>(m + b_t);
  h->d_crow = reinterpret_cast<int *>(m + b_t + b_c);
  if ((!tiles.empty() && (e = cudaMemcpy(h->d_tiles, tiles.data(), tiles.size(), cudaMemcpyHostToDevice)) != cudaSuccess) ||
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
  const size_t ob_b = 0, ob_x = align256(vb), ob_h = 2 * align256(vb), ob_i = ob_h + align256(hb),
               ob_w = ob_i + 256, total = ob_w + wsb;
  cudaError_t e = cudaSuccess;
  if (h->hbuf_bytes < total) {  // grow the cached device scratch
    if (h->hbuf) cudaFree(h->hbuf);
    h->hbuf = nullptr;
    h->hbuf_bytes = 0;
    if ((e = cudaMalloc(&h->hbuf, total)) != cudaSuccess) return cg_cuda_fail(e);
    h->hbuf_bytes = total;
  }
  if (!h->hstream && (e = cudaStreamCreateWithFlags(&h->hstream, cudaStreamNonBlocking)) != cudaSuccess)
    return cg_cuda_fail(e);
  char *buf = h->hbuf;
  cudaStream_t s = h->hstream;
  perks_status st = PERKS_OK;
  if (h->n > 0) e = cudaMemcpyAsync(buf + ob_b, h_b, h->n * h->elem(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    st = perks_cg_solve(h, v, pol, buf + ob_b, buf + ob_x, kmax, tol, reinterpret_cast<double *>(buf + ob_h),
                        reinterpret_cast<int64_t *>(buf + ob_i), buf + ob_w, wsb, s);
    if (st == PERKS_OK) {
      if (h->n > 0) e = cudaMemcpyAsync(h_x, buf + ob_x, h->n * h->elem(), cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess && h_hist) e = cudaMemcpyAsync(h_hist, buf + ob_h, hb, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess && h_info) e = cudaMemcpyAsync(h_info, buf + ob_i, 16, cudaMemcpyDeviceToHost, s);
    }
  }
  const cudaError_t es = cudaStreamSynchronize(s);
  if (st != PERKS_OK) return st;
  if (e == cudaSuccess) e = es;
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
  info->smem_per_cta = pl.smem;
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
  info->cached_nnz_smem = pl.cached_items_smem;
  info->cached_nnz_tmem = pl.cached_items_tmem;
  info->tmem_tiles_per_cta = pl.tm;
  info->smem_tiles_per_cta = pl.sm;
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
    if (h->hbuf) cudaFree(h->hbuf);
    if (h->hstream) cudaStreamDestroy(h->hstream);
  }
  delete h;
  return PERKS_OK;
}

}  // extern "C"
