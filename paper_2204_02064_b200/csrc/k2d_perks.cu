// k2d_perks.cu — variant (c) PERKS for 2D stencils whose domain fits on chip.
//
// The time loop runs inside one cooperative launch (Fig. 3 right).  Each CTA (1 per SM)
// owns a TX x TY tile and keeps it resident across ALL steps ("cache inter-step data in
// registers and shared memory"): RR rows per thread in registers (reg_cache) and RS rows in
// shared memory (sm_cache) (Fig. 6 Source/Destination switch).  Only the tile's
// boundary cells leave the SM: each step a CTA publishes its four edges to a global exchange slot
// (the vertical edges stored contiguously, "we transpose the vertical edges of the halo region in
// global memory") and reads its neighbours' edges through L2 (halo cells are never cached,
// P:348-355).  Instead of a device-wide grid.sync each CTA waits only on the flags of the
// (up to 8) neighbours it reads — the paper's dependency is only between adjacent TBs.
// Exchange slots and smem edge buffers are double-buffered by step parity, so one flag per step
// suffices (no write-after-read hazard: a CTA overwrites parity p only after its neighbours have
// published the next step, which they do after reading parity p).
//
// Inside the CTA, thread (wx*32+lane, wy) owns V consecutive x cells and R = RR+RS consecutive
// rows.  x-neighbours come from warp shuffles (lanes 0/31 from shared-memory column buffers at
// warp edges); the rows above/below a thread's segment come from shared-memory row buffers.
// The compute body is the same FMA chain as the host-loop kernel (reading R5) so results are
// bit-identical to variants (a) and (b).
#include <algorithm>
#include <type_traits>
#include <cstdio>

#include "common.cuh"
#include "internal.h"
#include "shapes.cuh"
#include "tmem.cuh"

// timing experiments only (wrong results): skip the halo tag waits / the per-step CTA barrier
#ifndef PERKS_P2D_XNOWAIT
#define PERKS_P2D_XNOWAIT 0
#endif
#ifndef PERKS_P2D_TPRE  // issue each TMEM row's load one row ahead of its use
#define PERKS_P2D_TPRE 1
#endif
#ifndef PERKS_P2D_SUNROLL  // unroll of the shared-memory row loop (0: full; 3 = the window period)
#define PERKS_P2D_SUNROLL 0
#endif
#ifndef PERKS_P2D_XNOHALO
#define PERKS_P2D_XNOHALO 0
#endif
#ifndef PERKS_P2D_XNOBAR
#define PERKS_P2D_XNOBAR 0
#endif
#ifndef PERKS_P2D_HPMIN  // fewest warps per CTA at which every warp takes part in the halo polls
#define PERKS_P2D_HPMIN 8
#endif

namespace perks {

// RR rows per thread in registers, RT rows in Tensor Memory (tmem.cuh: each thread's rows in its own
// TMEM lane, 4 columns per row — a register-file extension, sm_100a), RS rows in shared memory.
template <typename T, int V_, int WX_, int WY_, int RR_, int RS_, int RT_ = 0>
struct Geo2P {
  static constexpr int V = V_, WX = WX_, WY = WY_, RR = RR_, RS = RS_, RT = RT_, R = RR_ + RT_ + RS_;
  static constexpr int RS0 = RR + RT;  // first shared-memory row
  // TMEM columns per CTA: warps sharing a lane quarter take consecutive column groups
  static constexpr int WPR = V * (int)sizeof(T) / 4;  // TMEM columns per row segment
  static constexpr int TCOLS_RAW = RT * WPR * ((WX * WY + 3) / 4);
  static constexpr int TCOLS = TCOLS_RAW == 0 ? 0 : TCOLS_RAW <= 32 ? 32 : TCOLS_RAW <= 64 ? 64
                               : TCOLS_RAW <= 128 ? 128 : TCOLS_RAW <= 256 ? 256 : 512;
  static_assert(TCOLS_RAW <= 512, "TMEM rows exceed 512 columns");
  static constexpr int NT = 32 * WX * WY;
  static constexpr int TX = 32 * V * WX, TY = WY * R;
  static constexpr int ROWW = TX + 2;  // x = -1 .. TX
  // shared memory (elements): sm_cache | row buffers | column buffers
  static constexpr int CACHE = RS * NT * V;
  static constexpr int ROWBUF = 2 /*par*/ * 2 /*top,bot*/ * (WY + 1) * ROWW;
  static constexpr int COLBUF = 2 /*par*/ * 2 /*left,right*/ * (WX + 1) * TY;
  // + one scratch word per thread: the sink of the branch-free column-buffer stores (per thread, so
  // no two threads ever write the same word: compute-sanitizer racecheck clean)
  static constexpr size_t SMEM_BYTES = (size_t)(CACHE + ROWBUF + COLBUF + NT) * sizeof(T);
  static constexpr int SLOT = 2 * (TX + TY);  // one parity of one tile's exchange slot
};

// Copy n tagged values (all carrying `tag`) from src to smem dst, lane-strided; each lane first
// issues all its E loads, then re-polls only the words whose tag has not arrived yet.
template <typename T, int E>
PERKS_DEVINL void poll_copy(const LLWord *src, int n, unsigned tag, bool exists, T *dst, int lane) {
  constexpr int W = LL<T>::WORDS;
  if (!exists) {
    for (int i = lane; i < n; i += 32) dst[i] = T(0);
    return;
  }

  T val[E];
  unsigned pending = 0;
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int i = lane + 32 * e;
    if (i < n && !LL<T>::get(src + i * W, tag, val[e])) pending |= 1u << e;
  }
  if (PERKS_P2D_XNOWAIT) pending = 0;
  if (pending) {
    const unsigned long long t0 = globaltimer_ns();
    while (pending) {
#pragma unroll
      for (int e = 0; e < E; e++)
        if ((pending >> e) & 1u) {
          const int i = lane + 32 * e;
          if (LL<T>::get(src + i * W, tag, val[e])) pending &= ~(1u << e);
        }
      if (pending && globaltimer_ns() - t0 > PERKS_WATCHDOG_NS) watchdog_fire("perks2d halo", pending, tag);
    }
  }
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int i = lane + 32 * e;
    if (i < n) dst[i] = val[e];
  }
}

struct Tiles2 {
  int ntx, nty;
};

// Sliding-window rows of the compute body.  Scalar: x-1 .. x+V of one row.  Packed (fp32, V = 4k,
// PERKS_FFMA2): per group g of 4 cells (b = 4g), the four stride-2 pairs (w_b,w_b+2),
// (w_b+1,w_b+3), (w_b+2,w_b+4), (w_b+3,w_b+5) of w = x-1 .. x+V, so the group's output pairs
// (n_b,n_b+2) and (n_b+1,n_b+3) take every chain operand as one register pair (an FFMA2 per term
// for two cells; neighbours dx = -1, 0, +1 of (n_b,n_b+2) are the group's pairs 0, 1, 2, of
// (n_b+1,n_b+3) pairs 1, 2, 3).  A cached row is stored in the matching order {v_b, v_b+2, v_b+1,
// v_b+3} per group.
template <typename T, int V> struct SWin {
  T w[V + 2];
};
template <int V> struct PWin {
  f32x2 p[V / 4][4];
};
// storage order of a cached row <-> natural order (self-inverse)
template <bool PK, typename T, int V> PERKS_DEVINL void perm_row(const T (&a)[V], T (&b)[V]) {
  if constexpr (PK) {
#pragma unroll
    for (int g = 0; g < V / 4; g++) {
      b[4 * g] = a[4 * g]; b[4 * g + 1] = a[4 * g + 2]; b[4 * g + 2] = a[4 * g + 1]; b[4 * g + 3] = a[4 * g + 3];
    }
  } else {
#pragma unroll
    for (int i = 0; i < V; i++) b[i] = a[i];
  }
}

template <typename T, int S, class G>
__global__ void __launch_bounds__(G::NT, 1) perks2d_kernel(const T *__restrict__ in,
                                                           T *__restrict__ out, LLWord *gslot,
                                                           int nx, int ny,
                                                           Tiles2 tl, int64_t steps,
                                                           Coef<T, Shape<S>::N> c) {
  constexpr int V = G::V, R = G::R, RR = G::RR, RT = G::RT, RS0 = G::RS0, NT = G::NT, TX = G::TX, TY = G::TY;
  constexpr int WX = G::WX, WY = G::WY, ROWW = G::ROWW, NWARP = NT / 32;
  constexpr bool BOX = has_corners<S>();
  // fully unrolled shared-memory rows: compile-time row offsets (C2: 6.25 -> 5.89 us/step against
  // an unroll of 3, profiles/r02_c2_ffma2.txt)
  constexpr int SROW_UNROLL = PERKS_P2D_SUNROLL ? PERKS_P2D_SUNROLL : (G::RS > 1 ? G::RS : 1);
  // packed-pair body (FFMA2): fp32 with 4 cells per thread-row
  constexpr bool PK = PERKS_FFMA2 && sizeof(T) == 4 && V % 4 == 0 && RR <= 8;  // (16 register rows + pair windows spill)
  using Win = typename std::conditional<PK, PWin<V>, SWin<T, V>>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *const sm = reinterpret_cast<T *>(smem_raw);
  // shared-memory map (element offsets):
  //   sm_cache        [0, CACHE)                      row r>=RR of thread tid at (r-RR)*NT*V + tid*V
  //   row buffers     TOP(par,j) j=0..WY, BOT(par,jp1) jp1=0..WY, each ROWW wide (x=-1..TX)
  //   column buffers  LEFT(par,k) k=0..WX, RIGHT(par,kp1) kp1=0..WX, each TY tall
  //   scratch         NT elements (one sink word per thread for the branch-free column stores)
  constexpr int ROW0 = G::CACHE, COL0 = G::CACHE + G::ROWBUF;
  constexpr int SCR0 = G::CACHE + G::ROWBUF + G::COLBUF;
  constexpr int PAR_ROW = 2 * (WY + 1) * ROWW, PAR_COL = 2 * (WX + 1) * TY;
  auto TOP = [](int j) { return ROW0 + j * ROWW; };                    // + par*PAR_ROW
  auto BOT = [](int jp1) { return ROW0 + (WY + 1 + jp1) * ROWW; };     // + par*PAR_ROW
  auto LEFT = [](int k) { return COL0 + k * TY; };                     // + par*PAR_COL
  auto RIGHT = [](int kp1) { return COL0 + (WX + 1 + kp1) * TY; };     // + par*PAR_COL

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wx = warp % WX, wy = warp / WX;
  const int tile = blockIdx.x;
  const int tx = tile % tl.ntx, ty = tile / tl.ntx;
  const int x0 = tx * TX, y0 = ty * TY;
  const int xr = (wx * 32 + lane) * V;  // x relative to tile
  const int yr0 = wy * R;               // first row relative to tile
  const int x = x0 + xr;
  // global exchange slot of tile t, parity par: [top TX | bot TX | left TY | right TY]
  // tagged words (LL<T>::WORDS per value); tag of x^s is s+1 (slots are zeroed per run)
  constexpr int W = LL<T>::WORDS;
  auto GS = [&](int t, int par) -> LLWord * { return gslot + ((size_t)t * 2 + par) * G::SLOT * W; };

  for (int i = tid; i < G::ROWBUF + G::COLBUF + NT; i += NT) sm[ROW0 + i] = T(0);

  // per-thread shared-memory offsets (parity 0; add par*PAR_ROW / par*PAR_COL)
  const bool is_l = lane == 0, is_r = lane == 31;
  const int o_top = TOP(wy) + xr + 1, o_bot = BOT(wy + 1) + xr + 1;        // publish rows
  const int o_colL = is_l ? LEFT(wx) + yr0 : SCR0 + tid;                    // publish cols
  const int o_colR = is_r ? RIGHT(wx + 1) + yr0 : SCR0 + tid;
  // row strides of the column stores (1 for lanes 0 / 31, 0 for the scratch sink), opaque to the
  // compiler so each row's address is one IMAD (base + r * step) rather than a select chain
  int o_colL_step = is_l ? 1 : 0, o_colR_step = is_r ? 1 : 0;
  asm volatile("" : "+r"(o_colL_step), "+r"(o_colR_step));
  int colL_at = o_colL, colR_at = o_colR;  // + this step's parity offset (set per step)
  const int o_rdL = RIGHT(wx) + yr0, o_rdR = LEFT(wx + 1) + yr0;           // read cols
  const int o_above = BOT(wy) + xr, o_below = TOP(wy + 1) + xr;             // read rows
  const bool g_top = wy == 0, g_bot = wy == WY - 1;
  const bool g_l = is_l && wx == 0, g_r = is_r && wx == WX - 1;
  T *const my_smc = sm + (size_t)tid * V;

  // publish row r (values v) into parity pb: smem edges for neighbours inside the CTA, and the
  // global exchange slot for the neighbouring tiles (vertical edges stored contiguously)
  auto publish_row = [&](int pb, LLWord *g, unsigned tag, int r, const T (&v)[V],
                         bool maybe_edge_row = true) {
    const int pr = pb * PAR_ROW, pc = pb * PAR_COL;
    if (maybe_edge_row && r == 0) {
#pragma unroll
      for (int i = 0; i < V; i++) sm[pr + o_top + i] = v[i];
      if (g_top) {
#pragma unroll
        for (int i = 0; i < V; i++) LL<T>::put(g + (xr + i) * W, v[i], tag);
      }
    }
    if (maybe_edge_row && r == R - 1) {
#pragma unroll
      for (int i = 0; i < V; i++) sm[pr + o_bot + i] = v[i];
      if (g_bot) {
#pragma unroll
        for (int i = 0; i < V; i++) LL<T>::put(g + (TX + xr + i) * W, v[i], tag);
      }
    }
    // branch-free: lanes without a column-buffer cell store to a scratch word (predicated
    // stores measured 30 % slower: 11.9 vs 9.1 us/step on C2).  One warp per tile row (WX == 1):
    // no warp has a neighbour inside the tile, nothing to store.
    if constexpr (WX > 1) {
      sm[colL_at + o_colL_step * r] = v[0];
      sm[colR_at + o_colR_step * r] = v[V - 1];
    }
    // tile-edge columns: WX > 1 publishes them once per step from the column buffers (flush_cols);
    // one warp per row band has no column buffer and publishes row by row
    if constexpr (WX == 1) {
      if (g_l) LL<T>::put(g + (2 * TX + yr0 + r) * W, v[0], tag);
      if (g_r) LL<T>::put(g + (2 * TX + TY + yr0 + r) * W, v[V - 1], tag);
    }
  };
  // WX > 1: after a sweep, the tile-edge warps copy their R column values (lane 0 / 31 wrote them to
  // LEFT(0) / RIGHT(WX) of parity pb) to the exchange slot, one lane per row: one store instruction per
  // step instead of one divergent store per row (the exchange is off the critical path:
  // profiles/r01_c2_tile_scaling.txt)
  auto flush_cols = [&](int pb, LLWord *g, unsigned tag) {
    if constexpr (WX > 1) {
      const int pc = pb * PAR_COL;
      if (wx == 0 || wx == WX - 1) {
        __syncwarp();
        for (int i = lane; i < R; i += 32) {
          if (wx == 0) LL<T>::put(g + (2 * TX + yr0 + i) * W, sm[pc + LEFT(0) + yr0 + i], tag);
          if (wx == WX - 1) LL<T>::put(g + (2 * TX + TY + yr0 + i) * W, sm[pc + RIGHT(WX) + yr0 + i], tag);
        }
      }
    }
  };

  // ---- TMEM rows: one warp allocates, every CTA relinquishes its permit (tmem.cuh)
  __shared__ uint32_t tmem_base_slot;
  uint32_t tb = 0;  // this thread's TMEM row 0 (lane quarter of its warp + the warp's column group)
  if constexpr (RT > 0) {
    if (warp == 0) {
      tmem_alloc(&tmem_base_slot, (uint32_t)G::TCOLS);
      tmem_relinquish();
    }
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
    tb = tmem_base_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * RT * G::WPR);
    tb = __shfl_sync(0xffffffffu, tb, 0);  // warp-uniform by construction: lets ptxas keep it in a uniform register
  }
  auto trow = [&](int r) { return tb + (uint32_t)((r - RR) * G::WPR); };  // TMEM address of row r

  // ---- prologue: load the tile into the caches (P:519 the one-time 2·D_cache term, load half)
  T reg[RR > 0 ? RR : 1][V];
  auto load_row = [&](int r, T (&v)[V]) {
    const int y = y0 + yr0 + r;
#pragma unroll
    for (int i = 0; i < V; i++) v[i] = (y < ny && x + i < nx) ? in[(size_t)y * nx + x + i] : T(0);
  };
  __syncthreads();  // zeroed buffers before anyone publishes
  {
    LLWord *g0 = GS(tile, 0);
#pragma unroll
    for (int r = 0; r < RR; r++) {
      T v[V];
      load_row(r, v);
      perm_row<PK, T, V>(v, reg[r]);
      publish_row(0, g0, 1u, r, v);
    }
#pragma unroll
    for (int r = RR; r < RS0; r++) {
      T v[V], sv[V];
      load_row(r, v);
      perm_row<PK, T, V>(v, sv);
      tmem_st_row<T, V>(trow(r), sv);
      publish_row(0, g0, 1u, r, v);
    }
    if constexpr (RT > 0) tmem_wait_st();
#pragma unroll 1
    for (int r = RS0; r < R; r++) {
      T v[V], sv[V];
      load_row(r, v);
      perm_row<PK, T, V>(v, sv);
      vstore<T, V>(my_smc + (size_t)(r - RS0) * NT * V, sv);
      publish_row(0, g0, 1u, r, v);
    }
    flush_cols(0, g0, 1u);
  }

  // frame predicates (reading R1): most threads own no frame cell and skip the select
  const int ylo = max(0, 1 - (y0 + yr0)), yhi = min(R, ny - 1 - (y0 + yr0));
  const bool all_interior = ylo == 0 && yhi == R && x >= 1 && x + V - 1 <= nx - 2;
  // warp-uniform: does any lane of this warp own a frame cell?  (a uniform branch per row instead of a
  // divergent one; the selects inside stay per lane)
  const bool warp_frame = __any_sync(0xffffffffu, !all_interior);
  unsigned xmask = 0;
#pragma unroll
  for (int i = 0; i < V; i++) xmask |= ((x + i) >= 1 && (x + i) <= nx - 2) ? (1u << i) : 0u;

  for (int64_t t = 0; t < steps; t++) {
    const int par = (int)(t & 1), np = par ^ 1;
    const int pr = par * PAR_ROW, pc = par * PAR_COL;
    // ---- halo: warp s (s = 0 up, 1 down, 2 left, 3 right; round-robin if fewer warps) reads that
    //      neighbour's x^t edge (tag t+1) from its exchange slot (parity par) through L2 into the
    //      smem halo.  Each lane issues all its loads, then re-polls only words whose tag is not
    //      yet t+1.  Halo cells are never cached.
    const unsigned tag_in = (unsigned)(t + 1);
#pragma unroll 1
    // HP warps per side (all warps take part once there are >= 8): warp w reads segment w / 4 of
    // side w % 4, so the halo phase (and the CTA barrier after it) shortens with the warp count
    constexpr int HP = NWARP >= PERKS_P2D_HPMIN ? NWARP / 4 : 1;
    for (int sw = warp; sw < (PERKS_P2D_XNOHALO ? 0 : 4 * HP); sw += NWARP) {
      const int side = sw % 4, part = sw / 4;
      const int ddx = side < 2 ? 0 : (side == 2 ? -1 : 1);
      const int ddy = side < 2 ? (side == 0 ? -1 : 1) : 0;
      const int ntx = tx + ddx, nty = ty + ddy;
      const bool ex = ntx >= 0 && ntx < tl.ntx && nty >= 0 && nty < tl.nty;
      const int nt = nty * tl.ntx + ntx;
      if (side < 2) {
        const int dst = pr + (side == 0 ? BOT(0) : TOP(WY));
        const int lo = part * TX / HP, hi = (part + 1) * TX / HP;
        const LLWord *src = GS(ex ? nt : 0, par) + (side == 0 ? TX : 0) * W;
        poll_copy<T, (TX / HP + 31) / 32>(src + lo * W, hi - lo, tag_in, ex, sm + dst + 1 + lo, lane);
        if (BOX && part == 0 && lane < 2) {  // diagonal corners x = -1 (lane 0) and x = TX (lane 1)
          const int cx = ntx + (lane == 0 ? -1 : 1);
          const bool cex = cx >= 0 && cx < tl.ntx && nty >= 0 && nty < tl.nty;
          const LLWord *cs = GS(cex ? nty * tl.ntx + cx : 0, par) + ((side == 0 ? TX : 0) + (lane == 0 ? TX - 1 : 0)) * W;
          T val = T(0);
          if (cex && !LL<T>::get(cs, tag_in, val)) {
            const unsigned long long t0 = globaltimer_ns();
            while (!LL<T>::get(cs, tag_in, val))
              if (globaltimer_ns() - t0 > PERKS_WATCHDOG_NS) watchdog_fire("perks2d halo corner", 0u, tag_in);
          }
          sm[dst + (lane == 0 ? 0 : TX + 1)] = val;
        }
      } else {
        const bool left = side == 2;
        const int dst = pc + (left ? RIGHT(0) : LEFT(WX));
        const int lo = part * TY / HP, hi = (part + 1) * TY / HP;
        const LLWord *src = GS(ex ? nt : 0, par) + (2 * TX + (left ? TY : 0)) * W;
        poll_copy<T, (TY / HP + 31) / 32>(src + lo * W, hi - lo, tag_in, ex, sm + dst + lo, lane);
        if (BOX) {
          __syncwarp();
          // internal corners of the row buffers at x = -1 / TX for thread-row boundaries: each
          // value is copied by the warp that polled it
          const int xc = left ? 0 : TX + 1;
          for (int j = 1 + lane; j < WY; j += 32) {
            if (j * R - 1 >= lo && j * R - 1 < hi) sm[pr + BOT(j) + xc] = sm[dst + j * R - 1];
            if (j * R >= lo && j * R < hi) sm[pr + TOP(j) + xc] = sm[dst + j * R];
          }
        }
      }
    }
    if (!PERKS_P2D_XNOBAR) __syncthreads();
    // ---- compute x^{t+1} for the thread's V x R cells (sliding window over rows)
    LLWord *gnp = GS(tile, np);
    const unsigned tag_out = (unsigned)(t + 2);
    colL_at = o_colL + (is_l ? np * PAR_COL : 0);
    colR_at = o_colR + (is_r ? np * PAR_COL : 0);
    // the sweep, instantiated with and without the frame selects: a warp owns frame cells or
    // not for the whole run, so the test is one uniform branch per step instead of one per row
    // (which also cost register-merge moves after every row)
    auto sweep = [&](auto frame_c) {
      constexpr bool FR = decltype(frame_c)::value;
      Win prev, cur, nxt;
      // own row (old values, storage order) + x-neighbours: shuffles inside the warp; lanes 0/31
      // take the neighbouring warp's / tile's edge column (broadcast reads, branch free)
      // the warp-edge column values are loaded one row ahead (rows are widened in order 0, 1, ...,
      // R-1), so their shared-memory latency is off the row's dependency chain; the load past the
      // last row reads the neighbouring buffer and is never used
      T pcl = sm[pc + o_rdL], pcr = sm[pc + o_rdR];
      auto widen = [&](Win &w, const T (&v)[V], int r) {
        T n[V];
        perm_row<PK, T, V>(v, n);  // natural order
        const T l = __shfl_up_sync(0xffffffffu, n[V - 1], 1);
        const T rr = __shfl_down_sync(0xffffffffu, n[0], 1);
        const T cl = pcl, cr = pcr;
        pcl = sm[pc + o_rdL + r + 1];
        pcr = sm[pc + o_rdR + r + 1];
        const T left = is_l ? cl : l, right = is_r ? cr : rr;
        if constexpr (PK) {
#pragma unroll
          for (int g = 0; g < V / 4; g++) {
            const int b = 4 * g;
            w.p[g][0] = pack2(b == 0 ? left : n[b - 1], n[b + 1]);
            w.p[g][1] = pack2(v[b], v[b + 1]);      // (n_b, n_b+2): the stored pair as is
            w.p[g][2] = pack2(v[b + 2], v[b + 3]);  // (n_b+1, n_b+3)
            w.p[g][3] = pack2(n[b + 2], b + 4 < V ? n[b + 4] : right);
          }
        } else {
          w.w[0] = left;
          w.w[V + 1] = right;
#pragma unroll
          for (int i = 0; i < V; i++) w.w[i + 1] = n[i];
        }
      };
      // a halo row (x-1 .. x+V) from a shared-memory row buffer
      auto halo_row = [&](Win &w, int off) {
        T h[V + 2];
#pragma unroll
        for (int i = 0; i < V + 2; i++) h[i] = sm[off + i];
        if constexpr (PK) {
#pragma unroll
          for (int g = 0; g < V / 4; g++)
#pragma unroll
            for (int j = 0; j < 4; j++) w.p[g][j] = pack2(h[4 * g + j], h[4 * g + j + 2]);
        } else {
#pragma unroll
          for (int i = 0; i < V + 2; i++) w.w[i] = h[i];
        }
      };
      auto halo_below = [&](Win &w) { halo_row(w, pr + o_below); };
      // FMA chain (reading R5) + frame select + publish; rotates the window.  ns: the new row in
      // storage order
      auto finish_row = [&](int r, T (&ns)[V], bool maybe_edge_row = true) {
        T nv[V], cv[V];  // natural order: new values, old values (frame cells keep them)
        if constexpr (PK) {
          f32x2 A[V / 4], B[V / 4];  // per group: cells (b, b+2), (b+1, b+3)
#pragma unroll
          for (int p = 0; p < Shape<S>::N; p++) {
            const int dy = Shape<S>::dy(p), dx = Shape<S>::dx(p);
            const Win &src = dy < 0 ? prev : (dy > 0 ? nxt : cur);
#pragma unroll
            for (int g = 0; g < V / 4; g++) {
              A[g] = (p == 0) ? mul2_rn(c.w[0], src.p[g][1 + dx]) : fma2_rn(c.w[p], src.p[g][1 + dx], A[g]);
              B[g] = (p == 0) ? mul2_rn(c.w[0], src.p[g][2 + dx]) : fma2_rn(c.w[p], src.p[g][2 + dx], B[g]);
            }
          }
#pragma unroll
          for (int g = 0; g < V / 4; g++) {
            const int b = 4 * g;
            unpack2(A[g], nv[b], nv[b + 2]);
            unpack2(B[g], nv[b + 1], nv[b + 3]);
            unpack2(cur.p[g][1], cv[b], cv[b + 2]);
            unpack2(cur.p[g][2], cv[b + 1], cv[b + 3]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < V; i++) {
            T acc;
#pragma unroll
            for (int p = 0; p < Shape<S>::N; p++) {
              const int dy = Shape<S>::dy(p), dx = Shape<S>::dx(p);
              const T val = dy < 0 ? prev.w[i + 1 + dx] : (dy > 0 ? nxt.w[i + 1 + dx] : cur.w[i + 1 + dx]);
              acc = (p == 0) ? mul_rn(c.w[0], val) : fma_rn(c.w[p], val, acc);
            }
            nv[i] = acc;
            cv[i] = cur.w[i + 1];
          }
        }
        if constexpr (FR) {
          const bool rin = r >= ylo && r < yhi;
#pragma unroll
          for (int i = 0; i < V; i++) nv[i] = (rin && ((xmask >> i) & 1u)) ? nv[i] : cv[i];
        }
        publish_row(np, gnp, tag_out, r, nv, maybe_edge_row);
        perm_row<PK, T, V>(nv, ns);
        prev = cur;
        cur = nxt;
      };
      // the TMEM row in flight: row rn + 1 is issued as soon as row rn is taken (PERKS_P2D_TPRE)
      TmemRowInFlight<T, V> tpre;
      if constexpr (RT > 0 && PERKS_P2D_TPRE) tpre.issue(trow(RR));
      auto tmem_row = [&](int rn, T (&v)[V]) {
        if constexpr (PERKS_P2D_TPRE) {
          tpre.take(v);
          if (rn + 1 < RS0) tpre.issue(trow(rn + 1));
        } else {
          tmem_ld_row<T, V>(trow(rn), v);
        }
      };
      {
        halo_row(prev, pr + o_above);  // x = xr-1 .. xr+V
        T v[V];
        if (RR > 0) {
#pragma unroll
          for (int i = 0; i < V; i++) v[i] = opaque_copy(reg[0][i]);
        } else if (RT > 0) {
          tmem_row(0, v);
        } else {
          vload<T, V>(v, my_smc);
        }
        widen(cur, v, 0);
      }
      // the first row of the next tier (TMEM, then shared memory) or the halo below
      auto next_tier_row = [&](int rn) {
        if (RT > 0 && rn < RS0) {
          T v[V];
          tmem_row(rn, v);
          widen(nxt, v, rn);
        } else if (RS0 < R) {
          T v[V];
          vload<T, V>(v, my_smc + (size_t)(rn - RS0) * NT * V);
          widen(nxt, v, rn);
        } else {
          halo_below(nxt);
        }
      };
      // rows held in registers: fully unrolled so reg[][] is statically indexed
#pragma unroll
      for (int r = 0; r < RR; r++) {
        if (r + 1 < RR) {
          T v[V];
#pragma unroll
          for (int i = 0; i < V; i++) v[i] = opaque_copy(reg[r + 1 < RR ? r + 1 : 0][i]);
          widen(nxt, v, r + 1);
        } else {
          next_tier_row(r + 1);
        }
        T nv[V];
        finish_row(r, nv);
#pragma unroll
        for (int i = 0; i < V; i++) reg[r][i] = nv[i];
      }
      // rows held in TMEM: fully unrolled (compile-time column offsets); row r's old values are no
      // longer needed once row r+1 is in the window, so its new values go straight back
#pragma unroll
      for (int r = RR; r < RS0; r++) {
        next_tier_row(r + 1);
        T nv[V];
        finish_row(r, nv);
        tmem_st_row<T, V>(trow(r), nv);
      }
      if constexpr (RT > 0) tmem_wait_st();
      // rows held in shared memory (sm_cache); unrolled (SROW_UNROLL); the last row
      // (which reads the row below the segment) is peeled so the loop body has no row tests
      if (RS0 < R) {
#pragma unroll(SROW_UNROLL)
        for (int r = RS0; r < R - 1; r++) {
          T v[V];
          vload<T, V>(v, my_smc + (size_t)(r + 1 - RS0) * NT * V);
          widen(nxt, v, r + 1);
          T nv[V];
          finish_row(r, nv, RS0 == 0 && r == 0);
          vstore<T, V>(my_smc + (size_t)(r - RS0) * NT * V, nv);
        }
        halo_below(nxt);
        T nv[V];
        finish_row(R - 1, nv);
        vstore<T, V>(my_smc + (size_t)(R - 1 - RS0) * NT * V, nv);
      }
    };
    if (warp_frame) sweep(std::true_type{});
    else sweep(std::false_type{});
    flush_cols(np, gnp, tag_out);
    // every warp signals "my part of x^{t+1}'s boundary is published": flag = (t+2)*NWARP when the
    // whole tile edge is out.  No CTA barrier here: the next step's halo phase only touches the
    // other parity's buffers, and its __syncthreads orders this step's smem edge writes.
  }

  // ---- epilogue: flush the cache to `out` (the store half of the 2·D_cache term).
  // Addresses go through an empty asm barrier so ptxas cannot hoist 4*RR predicated store
  // addresses above the time loop (that alone cost ~80 registers; P:860 register pressure).
  int ybase = y0 + yr0, xe = x;
  T *oute = out;
  asm volatile("" : "+r"(ybase), "+r"(xe), "+l"(oute));
  auto store_row = [&](int r, const T (&v)[V]) {
    const int y = ybase + r;
    if (y < ny) {
#pragma unroll
      for (int i = 0; i < V; i++)
        if (xe + i < nx) oute[(size_t)y * nx + xe + i] = v[i];
    }
  };
#pragma unroll
  for (int r = 0; r < RR; r++) {
    T n[V];
    perm_row<PK, T, V>(reg[r], n);
    store_row(r, n);
  }
#pragma unroll
  for (int r = RR; r < RS0; r++) {
    T v[V], n[V];
    tmem_ld_row<T, V>(trow(r), v);
    perm_row<PK, T, V>(v, n);
    store_row(r, n);
  }
#pragma unroll 1
  for (int r = RS0; r < R; r++) {
    T v[V], n[V];
    vload<T, V>(v, my_smc + (size_t)(r - RS0) * NT * V);
    perm_row<PK, T, V>(v, n);
    store_row(r, n);
  }
  if constexpr (RT > 0) {
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
    if (warp == 0) tmem_dealloc(tmem_base_slot, (uint32_t)G::TCOLS);
  }
}

// (The barrier-free dataflow variant of round 1 was measured slower on C2, 8.33 vs 7.39 us/step,
// profiles/r01_c2_flow.txt, and removed; this kernel keeps the one CTA barrier per step.)


// ------------------------------------------------------------------ host side

namespace {
// Configurations (index = Plan::cfg).  f32 V=4, f64 V=2 (16-byte vectors per thread-row).
#ifndef PERKS_P2F_WY
#define PERKS_P2F_WY 4
#endif
#ifndef PERKS_P2F_RR
#define PERKS_P2F_RR 16
#endif
#ifndef PERKS_P2F_RS
#define PERKS_P2F_RS 48
#endif
#ifndef PERKS_P2F_V
#define PERKS_P2F_V 4
#endif
using P2F_A = Geo2P<float, PERKS_P2F_V, 8 / PERKS_P2F_V, PERKS_P2F_WY, PERKS_P2F_RR, PERKS_P2F_RS>;   // default 256 x 256 tile, 256 thr, 64 KiB regs + 192 KiB smem
// Tile configurations, largest first; the planner takes the SMALLEST tile whose count still fits one
// CTA per SM, so mid-size domains use (nearly) every SM instead of a few large tiles
// (profiles/r01_sweep2d.txt: 2048^2 on 64 tiles of 256^2 ran slower than the persistent kernel).
using P2F_A2 = Geo2P<float, 4, 2, 4, 16, 32>;  // 256 x 192 tile, 256 thr
using P2F_A3 = Geo2P<float, 4, 2, 4, 16, 16>;  // 256 x 128 tile, 256 thr
using P2F_B = Geo2P<float, 4, 1, 8, 8, 8>;     // 128 x 128 tile, 256 thr
using P2F_B2 = Geo2P<float, 4, 1, 8, 8, 0>;    // 128 x  64 tile, 256 thr
using P2F_C = Geo2P<float, 4, 1, 4, 8, 0>;     // 128 x  32 tile, 128 thr
// 256 x 256 tile with twice the threads: 8 register + 8 TMEM + 16 shared-memory rows per thread
// (TMEM as a register-file extension frees the shared memory the 16-warp row buffers need)
using P2D_A = Geo2P<double, 2, 2, 4, 16, 16>;  // 128 x 128 tile, 256 thr, 64 KiB regs + 64 KiB smem
using P2D_A2 = Geo2P<double, 2, 2, 4, 16, 8>;  // 128 x  96 tile, 256 thr
using P2D_A3 = Geo2P<double, 2, 2, 4, 16, 0>;  // 128 x  64 tile, 256 thr
using P2D_B = Geo2P<double, 2, 2, 4, 8, 0>;    // 128 x  32 tile, 256 thr
using P2D_C = Geo2P<double, 2, 1, 2, 8, 0>;    //  64 x  16 tile,  64 thr
// 16-warp tiles with a Tensor-Memory row tier (tmem.cuh): twice the threads of the 8-warp tiles,
// each with half the rows; TMEM (a per-thread register-file extension) holds the rows the 16-warp
// row buffers leave no shared memory for.  C2: 9.08 -> 8.25 us/step (profiles/r01_c2_tmem_rows.txt).
// register / shared-memory / TMEM rows per thread of the 256 x 256 16-warp tile (sweeps only:
// profiles/r01_c2_cache_location.txt)
#ifndef PERKS_P2T_RR
#define PERKS_P2T_RR 4
#endif
#ifndef PERKS_P2T_RS
#define PERKS_P2T_RS 12
#endif
#ifndef PERKS_P2T_RT
#define PERKS_P2T_RT 16
#endif
using P2F_T0 = Geo2P<float, 4, 2, 8, PERKS_P2T_RR, PERKS_P2T_RS, PERKS_P2T_RT>;  // 256 x 256 tile, 512 thr
using P2F_T1 = Geo2P<float, 4, 2, 8, 4, 8, 12>;    // 256 x 192
using P2F_T2 = Geo2P<float, 4, 2, 8, 4, 4, 8>;     // 256 x 128
#ifndef PERKS_P2V8_RT
#define PERKS_P2V8_RT 8
#endif
// 256 x 256, one warp per row band (V = 8: no intra-tile column exchange), forced-only: measured
// 7.85 us/step on C2 vs 7.32 for P2F_T0 (profiles/r01_c2_tmem_rows.txt)
using P2F_V8 = Geo2P<float, 8, 1, 16, 0, 16 - PERKS_P2V8_RT, PERKS_P2V8_RT>;
using P2D_T0 = Geo2P<double, 2, 2, 8, 4, 4, 8>;    // 128 x 128 tile, 512 thr
using P2D_T1 = Geo2P<double, 2, 2, 8, 4, 0, 8>;    // 128 x  96
using P2D_T2 = Geo2P<double, 2, 2, 8, 4, 0, 4>;    // 128 x  64
constexpr int NCFG_F = 6, NCFG_D = 5;   // configurations the planner chooses among
constexpr int NCFG_F_ALL = 10, NCFG_D_ALL = 8;  // + forced-only (PERKS_P2D_CFG) 8-warp alternatives
int ncfg(const Problem &p) { return p.dtype == PERKS_F32 ? NCFG_F : NCFG_D; }

struct CfgInfo {
  void *k;
  int TX, TY, NT;
  size_t smem;
  int64_t reg_cells, smem_cells, tmem_cells;
  int tcols;
};

template <typename T, int S, class G> CfgInfo info(bool flow) {
  void *k = (void *)perks2d_kernel<T, S, G>;
  size_t smem = G::SMEM_BYTES;
  (void)flow;
  return CfgInfo{k, G::TX, G::TY, G::NT, smem,
                 (int64_t)G::RR * G::V * G::NT, (int64_t)G::RS * G::V * G::NT,
                 (int64_t)G::RT * G::V * G::NT, G::TCOLS};
}
template <typename T, int S> CfgInfo info_t(int cfg, bool flow);
template <int S> CfgInfo info_f(int c, bool flow) {
  switch (c) {
    case 0: return info<float, S, P2F_T0>(flow);
    case 1: return info<float, S, P2F_T1>(flow);
    case 2: return info<float, S, P2F_T2>(flow);
    case 3: return info<float, S, P2F_B>(flow);
    case 4: return info<float, S, P2F_B2>(flow);
    case 5: return info<float, S, P2F_C>(flow);
    case 6: return info<float, S, P2F_A>(flow);
    case 7: return info<float, S, P2F_A2>(flow);
    case 8: return info<float, S, P2F_A3>(flow);
    default: return info<float, S, P2F_V8>(flow);
  }
}
template <int S> CfgInfo info_d(int c, bool flow) {
  switch (c) {
    case 0: return info<double, S, P2D_T0>(flow);
    case 1: return info<double, S, P2D_T1>(flow);
    case 2: return info<double, S, P2D_T2>(flow);
    case 3: return info<double, S, P2D_B>(flow);
    case 4: return info<double, S, P2D_C>(flow);
    case 5: return info<double, S, P2D_A>(flow);
    case 6: return info<double, S, P2D_A2>(flow);
    default: return info<double, S, P2D_A3>(flow);
  }
}
template <> CfgInfo info_t<float, SHAPE_2D5>(int c, bool fl) { return info_f<SHAPE_2D5>(c, fl); }
template <> CfgInfo info_t<float, SHAPE_2D9>(int c, bool fl) { return info_f<SHAPE_2D9>(c, fl); }
template <> CfgInfo info_t<double, SHAPE_2D5>(int c, bool fl) { return info_d<SHAPE_2D5>(c, fl); }
template <> CfgInfo info_t<double, SHAPE_2D9>(int c, bool fl) { return info_d<SHAPE_2D9>(c, fl); }
// Plan::cfg = configuration index | kFlowBit when the dataflow kernel runs it
constexpr int kFlowBit = 0x100;
CfgInfo cfg_info(const Problem &p, int cfgf) {
  const int cfg = cfgf & 0xff;
  const bool fl = (cfgf & kFlowBit) != 0;
  if (p.dtype == PERKS_F32) return p.shape == SHAPE_2D5 ? info_t<float, SHAPE_2D5>(cfg, fl) : info_t<float, SHAPE_2D9>(cfg, fl);
  return p.shape == SHAPE_2D5 ? info_t<double, SHAPE_2D5>(cfg, fl) : info_t<double, SHAPE_2D9>(cfg, fl);
}
}  // namespace

Plan plan_perks2d(const Problem &p) {
  Plan pl;
  pl.variant = PERKS_PERKS;
  if (p.ndim != 2 || (p.shape != SHAPE_2D5 && p.shape != SHAPE_2D9) || p.bc != PERKS_BC_FRAME) {
    pl.why = "perks2d: needs 2D 5pt/9pt FRAME";
    return pl;
  }
  if (p.nx > (1 << 30) || p.ny > (1 << 30)) { pl.why = "perks2d: extent too large"; return pl; }
  // Planner: if the whole domain fits one CTA's tile, use one CTA (no inter-CTA sync at all —
  // small domains are latency bound).  Otherwise the smallest tile whose count
  // fits one CTA per SM (all CTAs co-resident; minimal occupancy).
  int forced = env_int("PERKS_P2D_CFG", -1);
  int best = -1;
  const int NCFG = ncfg(p);
  for (int cfg = NCFG - 1; cfg >= 0 && forced < 0; cfg--) {
    CfgInfo ci = cfg_info(p, cfg);
    if (p.nx <= ci.TX && p.ny <= ci.TY && ci.smem <= (size_t)p.max_smem_optin) { best = cfg; break; }
  }
  for (int cfg = forced >= 0 ? (p.dtype == PERKS_F32 ? NCFG_F_ALL : NCFG_D_ALL) - 1 : NCFG - 1; cfg >= 0 && best < 0; cfg--) {
    if (forced >= 0 && cfg != forced) continue;
    CfgInfo ci = cfg_info(p, cfg);
    const int64_t tiles = ((p.nx + ci.TX - 1) / ci.TX) * ((p.ny + ci.TY - 1) / ci.TY);
    if (tiles <= p.num_sms && ci.smem <= (size_t)p.max_smem_optin) { best = cfg; break; }
  }
  if (best < 0) { pl.why = "perks2d: domain does not fit on chip (tiles > SMs)"; return pl; }
  CfgInfo ci = cfg_info(p, best);
  if (cudaFuncSetAttribute(ci.k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ci.smem) != cudaSuccess) {
    pl.why = "cudaFuncSetAttribute"; return pl;
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, ci.k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ci.k, ci.NT, ci.smem);
  const int ntx = (int)((p.nx + ci.TX - 1) / ci.TX), nty = (int)((p.ny + ci.TY - 1) / ci.TY);
  pl.cfg = best;
  pl.grid = ntx * nty;
  if (occ < 1 || pl.grid > occ * p.num_sms) { pl.why = "perks2d: not co-resident"; return pl; }
  pl.block = ci.NT;
  pl.ctas_per_sm = 1;
  pl.tile[0] = ci.TX; pl.tile[1] = ci.TY; pl.tile[2] = 1;
  pl.regs = fa.numRegs;
  pl.smem = (int)ci.smem;
  pl.units = pl.grid;
  pl.cached_reg = ci.reg_cells * pl.grid;
  pl.cached_smem = ci.smem_cells * pl.grid;
  pl.cached_tmem = ci.tmem_cells * pl.grid;
  pl.tcols = ci.tcols;
  const double S = (double)p.elem();
  pl.dram_bytes_step = 0.0;  // domain fully resident: only the one-time 2·D_cache term
  pl.halo_bytes_step = S * 2.0 * pl.grid * 2.0 * (ci.TX + ci.TY);  // publish + read, L2
  // tagged exchange words: 8 bytes per fp32 value, 16 per fp64 value
  const size_t slot_bytes = (size_t)pl.grid * 2 * 2 * (ci.TX + ci.TY) * (p.elem() == 8 ? 16 : 8);
  pl.ws_bytes = align256(slot_bytes);
  snprintf(pl.name, sizeof(pl.name), "perks2d_%s_%s_cfg%d_t%dx%d%s", p.shape == SHAPE_2D5 ? "5pt" : "9pt",
           p.dtype == PERKS_F32 ? "f32" : "f64", best & 0xff, ci.TX, ci.TY, (best & kFlowBit) ? "_flow" : "");
  pl.ok = true;
  return pl;
}

template <typename T, int S>
static cudaError_t launch_p2d(const Problem &p, const Plan &pl, const T *in, T *out, void *ws,
                              int64_t steps, cudaStream_t s) {
  CfgInfo ci = cfg_info(p, pl.cfg);
  Coef<T, Shape<S>::N> c;
  for (int i = 0; i < Shape<S>::N; i++) c.w[i] = sizeof(T) == 4 ? (T)p.wf[i] : (T)p.wd[i];
  LLWord *gslot = (LLWord *)ws;
  const size_t slot_bytes = (size_t)pl.grid * 2 * 2 * (ci.TX + ci.TY) * LL<T>::WORDS * sizeof(LLWord);
  cudaError_t e = cudaMemsetAsync(gslot, 0, slot_bytes, s);  // tags restart at 1 every run
  if (e != cudaSuccess) return e;
  Tiles2 tl{(int)((p.nx + ci.TX - 1) / ci.TX), (int)((p.ny + ci.TY - 1) / ci.TY)};
  int nx = (int)p.nx, ny = (int)p.ny;
  void *args[] = {(void *)&in, (void *)&out, (void *)&gslot, (void *)&nx, (void *)&ny,
                  (void *)&tl, (void *)&steps, (void *)&c};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(ci.NT);
  cfg.dynamicSmemBytes = ci.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, ci.k, args);
}

cudaError_t run_perks2d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws,
                        int64_t steps, cudaStream_t s) {
  if (p.dtype == PERKS_F32) {
    if (p.shape == SHAPE_2D5) return launch_p2d<float, SHAPE_2D5>(p, pl, (const float *)in, (float *)out, ws, steps, s);
    return launch_p2d<float, SHAPE_2D9>(p, pl, (const float *)in, (float *)out, ws, steps, s);
  }
  if (p.shape == SHAPE_2D5) return launch_p2d<double, SHAPE_2D5>(p, pl, (const double *)in, (double *)out, ws, steps, s);
  return launch_p2d<double, SHAPE_2D9>(p, pl, (const double *)in, (double *)out, ws, steps, s);
}

}  // namespace perks
