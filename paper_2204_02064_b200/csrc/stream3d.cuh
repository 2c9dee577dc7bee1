// stream3d.cuh — the 3D plane-streaming compute body shared by the host-loop (a), persistent (b)
// and PERKS (c) variants.  "2D planes are loaded one after the other in shared memory, and each
// thread computes the cells in a vertical direction".
//
// A CTA owns an xy tile of TX x TY cells (TX = 32*V: one warp spans x; TY = NWARP*R) and a z range.
// Planes arrive in increasing z into a ring of NS shared-memory slots with NS-1 planes in flight.
// Each slot holds the tile plus a one-cell halo ring; rows are padded by PAD = 16 B so the interior
// starts 16-byte aligned.  Thread (lane, warp) owns V x R cells of every plane.  When plane q is
// resident, the chain terms of outputs q+1 / q / q-1 that read plane q are applied in list order
// (stages A/B/C of shapes.cuh), so each plane is read from shared memory once per thread.
//
// Two loaders fill the ring:
//   * TMA (Blackwell/Hopper tensor-memory accelerator): ONE thread issues one 3D tensor box
//     {P, TY+2, 1} per plane (cp.async.bulk.tensor, out-of-bounds cells zero-filled by hardware)
//     completing on the slot's mbarrier — no per-thread address arithmetic in the plane loop.
//     Requires 16-byte aligned rows (nx*S % 16 == 0).
//   * cp.async (fallback for ragged nx): every thread copies its own cells.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "dist.cuh"
#include "shapes.cuh"
#include "tmem.cuh"

namespace perks {

// Unroll factor of the per-plane loops (3 turns the stage-accumulator rotation into register
// renaming; sweeps only, the default keeps register pressure low).
#ifndef PERKS_NB_LDS
#define PERKS_NB_LDS 1
#endif
#ifndef PERKS_WS_UNROLL
#define PERKS_WS_UNROLL 1
#endif
constexpr int kWsUnroll = PERKS_WS_UNROLL;

template <typename T, int V_, int R_, int NWARP_, int NS_>
struct Geo3D {
  static constexpr int V = V_, R = R_, NWARP = NWARP_, NS = NS_;
  static constexpr int NT = 32 * NWARP;
  static constexpr int TX = 32 * V, TY = NWARP * R;
  static constexpr int PAD = 16 / (int)sizeof(T);  // interior starts 16-B aligned
  static constexpr int P = TX + 2 * PAD;             // row pitch (elements) = TMA box width
  static constexpr int ROWS = TY + 2;
  static constexpr int SLOT_RAW = ROWS * P;
  static constexpr int SLOT = (SLOT_RAW * (int)sizeof(T) + 127) / 128 * 128 / (int)sizeof(T);
  static constexpr size_t SLOT_BYTES = (size_t)SLOT * sizeof(T);  // 128-B multiple (TMA dst)
  static constexpr unsigned BOX_BYTES = (unsigned)(SLOT_RAW * sizeof(T));
  static constexpr unsigned ROW_BYTES = (unsigned)(P * sizeof(T));
  // after the NS ring slots: full / empty / tfull mbarriers (3 x NS x 8 B) and the TMEM base
  // address, padded to 128 B (the PERKS plane cache follows)
  static constexpr size_t BAR_BYTES = (3 * NS * 8 + 16 + 127) / 128 * 128;
  static constexpr size_t RING_BYTES = (size_t)NS * SLOT_BYTES + BAR_BYTES;

  static_assert(V * (int)sizeof(T) == 16 || V * (int)sizeof(T) == 8, "one 16- or 8-byte vector per thread per row");
  static_assert(NT >= 2 * ROWS, "halo-column loaders");
  static_assert(P <= 256 && ROWS <= 256, "TMA box dims <= 256");
};

struct Dom3 {
  int nx, ny, nz;
  int zlo, zhi;  // planes zlo..zhi are z-interior (single GPU: 1..nz-2; slab faces with a neighbour
                 // are interior, reading R12)
};

// TMA descriptors of the (up to) three buffers a run reads: 0 = in, 1 = out, 2 = tmp.
struct Maps3 {
  CUtensorMap box[3];  // box {P, ROWS, 1}: a whole tile plane with its halo ring
  CUtensorMap row[3];  // box {P, 1, 1}: one halo row (cached planes)
  CUtensorMap ghost;   // multi-GPU ghost planes G[4][ny][nx] (dist.cuh), box {P, ROWS, 1}
};

// ---------------------------------------------------------------- mbarrier / TMA primitives
PERKS_DEVINL void mbar_init(uint64_t *b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
PERKS_DEVINL void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
PERKS_DEVINL void mbar_arrive_tx(uint64_t *b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
PERKS_DEVINL void mbar_arrive_cnt(uint64_t *b, unsigned count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
PERKS_DEVINL void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
// arrive when all of this thread's prior cp.async copies have landed
PERKS_DEVINL void mbar_arrive_cpasync(uint64_t *b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
PERKS_DEVINL void mbar_arrive_release(uint64_t *b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
// try_wait suspends the thread for a hardware time slice; once the first try fails the spin
// reads %globaltimer and traps after PERKS_WATCHDOG_NS (all in one asm block: no registers stay
// live outside it and nothing is added to the fast path but one predicated branch).
PERKS_DEVINL void mbar_wait(uint64_t *b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      ".reg .u64 t0, t1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\n"
      "mov.u64 t0, %%globaltimer;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\n"
      "mov.u64 t1, %%globaltimer;\n"
      "sub.u64 t1, t1, t0;\n"
      "setp.gt.u64 p, t1, %2;\n"
      "@p trap;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity), "l"((unsigned long long)PERKS_WATCHDOG_NS)
      : "memory");
}
// 1D bulk async copy global -> shared (16-B aligned, size multiple of 16), completes on `bar`.
PERKS_DEVINL void bulk_load(void *sdst, const void *gsrc, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
PERKS_DEVINL void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
PERKS_DEVINL void tma_load_3d(void *sdst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(sdst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- cp.async loader (fallback)
// Issue cp.async copies of plane q of `src` (tile origin x0,y0) into `slot`.  Cells outside the
// domain are zero-filled (they only feed frame cells, whose results are discarded).
// If `halo_only`, only the one-cell ring around the tile is fetched (PERKS cached planes).
template <typename T, class G>
PERKS_DEVINL void issue_plane(T *slot, const T *__restrict__ src, const Dom3 &d, int q, int x0,
                              int y0, bool halo_only) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool zin = q >= 0 && q < d.nz;
  const size_t pl = (size_t)d.nx * d.ny;
  const T *base = src + (zin ? (size_t)q * pl : 0);
  const int x = x0 + lane * G::V;
  const bool xin = x < d.nx;
  // one row segment of V cells: a 16-byte copy when rows are vector aligned (nx % V == 0),
  // else V element copies with per-element bounds (ragged nx)
  const bool vec = (d.nx % G::V) == 0;
  auto seg = [&](int j, bool rowok) {
    const int y = y0 - 1 + j;
    T *s = slot + j * G::P + G::PAD + lane * G::V;
    if (vec) {
      const bool ok = rowok && xin;
      cp_async<16>(s, ok ? base + (size_t)y * d.nx + x : src, ok);
    } else {
#pragma unroll
      for (int i = 0; i < G::V; i++) {
        const bool ok = rowok && x + i < d.nx;
        cp_async<(int)sizeof(T)>(s + i, ok ? base + (size_t)y * d.nx + x + i : src, ok);
      }
    }
  };
  if (!halo_only) {
#pragma unroll
    for (int r = 0; r < G::R; r++) {
      const int j = warp * G::R + r + 1;  // slot row
      seg(j, zin && (y0 - 1 + j) < d.ny);
    }
  }
  // halo rows y0-1 (warp 0) and y0+TY (last warp)
  if (warp == 0 || warp == G::NWARP - 1) {
    const int j = warp == 0 ? 0 : G::ROWS - 1;
    const int y = y0 - 1 + j;
    seg(j, zin && y >= 0 && y < d.ny);
  }
  // halo columns x0-1 and x0+TX for all ROWS rows (corners included)
  if (tid < 2 * G::ROWS) {
    const int j = tid >> 1;
    const bool right = tid & 1;
    const int y = y0 - 1 + j;
    const int xx = right ? x0 + G::TX : x0 - 1;
    const bool ok = zin && y >= 0 && y < d.ny && xx >= 0 && xx < d.nx;
    const T *g = ok ? base + (size_t)y * d.nx + xx : src;
    cp_async<(int)sizeof(T)>(slot + j * G::P + (right ? G::PAD + G::TX : G::PAD - 1), g, ok);
  }
}

// ---------------------------------------------------------------- compute
// Neighbourhood of the thread's V x R cells in one resident plane:
// nb[j][i] = cell (x - 1 + i, y - 1 + j) for j in [0, R+2), i in [0, V+2).
template <typename T, class G>
PERKS_DEVINL void read_nb(const T *slot, T (&nb)[G::R + 2][G::V + 2]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int j = 0; j < G::R + 2; j++) {
    const T *row = slot + (warp * G::R + j) * G::P;
    T v[G::V];
    vload<T, G::V>(v, row + G::PAD + lane * G::V);
#if PERKS_NB_LDS
    // x-neighbours straight from shared memory (the slot holds the halo columns): two scalar
    // loads, no shuffle / select on the dependency chain
    nb[j][0] = row[G::PAD + lane * G::V - 1];
    nb[j][G::V + 1] = row[G::PAD + lane * G::V + G::V];
#else
    const T l = shfl_up1(v[G::V - 1]);
    const T r = shfl_down1(v[0]);
    const T el = row[G::PAD - 1 + (lane == 31 ? G::TX + 1 : 0)];  // one broadcast-free LDS
    nb[j][0] = lane == 0 ? el : l;
    nb[j][G::V + 1] = lane == 31 ? el : r;
#endif
#pragma unroll
    for (int i = 0; i < G::V; i++) nb[j][i + 1] = v[i];
  }
}

// Apply chain terms [PB, PE) of shape S for all V x R cells.  Terms with dz == DZ_NB read the
// resident plane (nb); other terms read the retained centre values `cen` (checked at compile time
// by stage_end in shapes.cuh).
template <typename T, int S, class G, int PB, int PE, int DZ_NB>
PERKS_DEVINL void apply_terms(T (&acc)[G::R][G::V], const T (&nb)[G::R + 2][G::V + 2],
                              const T (&cen)[G::R][G::V], const Coef<T, Shape<S>::N> &c) {
#pragma unroll
  for (int p = PB; p < PE; p++) {
#pragma unroll
    for (int r = 0; r < G::R; r++) {
#pragma unroll
      for (int i = 0; i < G::V; i++) {
        const T val = (Shape<S>::dz(p) == DZ_NB)
                          ? nb[r + 1 + Shape<S>::dy(p)][i + 1 + Shape<S>::dx(p)]
                          : cen[r][i];
        acc[r][i] = (p == 0) ? mul_rn(c.w[0], val) : fma_rn(c.w[p], val, acc[r][i]);
      }
    }
  }
}

// Per-thread streaming state across arrivals.
template <typename T, class G>
struct StreamState {
  T accA[G::R][G::V];  // output q+1 (chain prefix with dz=-1)
  T accB[G::R][G::V];  // output q
  T accC[G::R][G::V];  // output q-1
  T cm1[G::R][G::V];   // centre of the previous plane (q-1)
  PERKS_DEVINL void zero() {
#pragma unroll
    for (int r = 0; r < G::R; r++)
#pragma unroll
      for (int i = 0; i < G::V; i++) accA[r][i] = accB[r][i] = accC[r][i] = cm1[r][i] = T(0);
  }
};

// Process the arrival of plane q (resident in `slot`): finish output q-1 (returned in `out`),
// advance outputs q and q+1, rotate the state.  `center_q` receives plane q's own cells.
template <typename T, int S, class G>
PERKS_DEVINL void arrival(StreamState<T, G> &st, const T *slot, const Coef<T, Shape<S>::N> &c,
                          T (&out)[G::R][G::V], T (&center_q)[G::R][G::V]) {
  constexpr int e0 = stage_end<S>(0), e1 = stage_end<S>(1), e2 = stage_end<S>(2);
  T nb[G::R + 2][G::V + 2];
  read_nb<T, G>(slot, nb);
#pragma unroll
  for (int r = 0; r < G::R; r++)
#pragma unroll
    for (int i = 0; i < G::V; i++) center_q[r][i] = nb[r + 1][i + 1];
  // stage C: output q-1 reads plane q (dz=+1) or its own retained centre (dz=0)
  apply_terms<T, S, G, e1, e2, 1>(st.accC, nb, st.cm1, c);
#pragma unroll
  for (int r = 0; r < G::R; r++)
#pragma unroll
    for (int i = 0; i < G::V; i++) out[r][i] = st.accC[r][i];
  // stage B: output q reads plane q (dz=0) or retained centre of q-1 (dz=-1)
  apply_terms<T, S, G, e0, e1, 0>(st.accB, nb, st.cm1, c);
  // stage A: output q+1 reads plane q (dz=-1)
  apply_terms<T, S, G, 0, e0, -1>(st.accA, nb, st.cm1, c);
#pragma unroll
  for (int r = 0; r < G::R; r++)
#pragma unroll
    for (int i = 0; i < G::V; i++) {
      st.accC[r][i] = st.accB[r][i];
      st.accB[r][i] = st.accA[r][i];
    }
}

// Per-thread, per-unit constants for stores and frame selection (computed once per unit).
template <class G>
struct ThreadTile {
  int x, y;          // first owned cell
  unsigned fmask;    // bit r*V+i: cell (x+i, y+r) is an x/y frame cell or outside the domain
  unsigned pmask;    // bit r*V+i: cell (x+i, y+r) is on the tile perimeter and inside the domain
  bool full;         // x < nx, rows 16-byte aligned and all R rows inside: branch-free vector I/O
  PERKS_DEVINL void init(const Dom3 &d, int x0, int y0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    x = x0 + lane * G::V;
    y = y0 + warp * G::R;
    full = x < d.nx && (d.nx % G::V) == 0 && y + G::R <= d.ny;
    const int xl = min(x0 + G::TX, d.nx) - 1, yl = min(y0 + G::TY, d.ny) - 1;  // last tile cells
    unsigned xin = 0, xint = 0, xper = 0;  // per column i: inside / interior / tile edge
#pragma unroll
    for (int i = 0; i < G::V; i++) {
      xin |= (unsigned)(x + i < d.nx) << i;
      xint |= (unsigned)(x + i >= 1 && x + i <= d.nx - 2) << i;
      xper |= (unsigned)(x + i == x0 || x + i == xl) << i;
    }
    fmask = 0;
    pmask = 0;
#pragma unroll
    for (int r = 0; r < G::R; r++) {
      const int yy = y + r;
      const unsigned row = (yy >= 1 && yy <= d.ny - 2) ? xint : 0u;
      fmask |= (~row & ((1u << G::V) - 1)) << (r * G::V);
      const unsigned per = (yy < d.ny) ? ((yy == y0 || yy == yl) ? xin : (xper & xin)) : 0u;
      pmask |= per << (r * G::V);
    }
  }
  PERKS_DEVINL size_t off(const Dom3 &d) const { return (size_t)y * d.nx + x; }
};

// Frame select (reading R1) of output plane o; `old` = its step-k values (centre).  Interior
// threads of interior planes pay one uniform compare and one mask test.
template <typename T, class G>
PERKS_DEVINL void frame_select(const Dom3 &d, const ThreadTile<G> &tt, int o, T (&val)[G::R][G::V],
                               const T (&old)[G::R][G::V]) {
  const bool zint = o >= d.zlo && o <= d.zhi;
  if (zint && tt.fmask == 0) return;
  const unsigned m = zint ? tt.fmask : ~0u;
#pragma unroll
  for (int r = 0; r < G::R; r++)
#pragma unroll
    for (int i = 0; i < G::V; i++)
      if ((m >> (r * G::V + i)) & 1u) val[r][i] = old[r][i];
}

// Store the thread's cells of plane o (already frame-selected).
template <typename T, class G>
PERKS_DEVINL void store_cells(T *__restrict__ dst, const Dom3 &d, const ThreadTile<G> &tt, int o,
                              const T (&v)[G::R][G::V]) {
  if (tt.full) {  // the common case: R aligned vector stores, no per-row tests
    T *p = dst + (size_t)o * d.nx * d.ny + tt.off(d);
#pragma unroll
    for (int r = 0; r < G::R; r++) vstore<T, G::V>(p + (size_t)r * d.nx, v[r]);
    return;
  }
  if (tt.x >= d.nx) return;
  T *base = dst + (size_t)o * d.nx * d.ny;
#pragma unroll
  for (int r = 0; r < G::R; r++) {
    const int y = tt.y + r;
    if (y >= d.ny) break;
    if ((d.nx % G::V) == 0) {
      vstore<T, G::V>(base + (size_t)y * d.nx + tt.x, v[r]);
    } else {
#pragma unroll
      for (int i = 0; i < G::V; i++)
        if (tt.x + i < d.nx) base[(size_t)y * d.nx + tt.x + i] = v[r][i];
    }
  }
}

// Load the thread's cells of plane o from src (cells outside the domain read as zero: they only
// feed frame cells, whose results are discarded).  PERKS TMEM-tier prologue.
template <typename T, class G>
PERKS_DEVINL void load_own_cells(const T *__restrict__ src, const Dom3 &d, const ThreadTile<G> &tt, int o,
                                 T (&v)[G::R][G::V]) {
  const T *base = src + (size_t)o * d.nx * d.ny;
#pragma unroll
  for (int r = 0; r < G::R; r++) {
    const int y = tt.y + r;
    if (tt.full) {
      vload<T, G::V>(v[r], base + tt.off(d) + (size_t)r * d.nx);
      continue;
    }
#pragma unroll
    for (int i = 0; i < G::V; i++)
      v[r][i] = (y < d.ny && tt.x + i < d.nx) ? base[(size_t)y * d.nx + tt.x + i] : T(0);
  }
}

// ---------------------------------------------------------------- ring (TMA or cp.async)
// Arrival counter `gk` runs across units and steps: slot = gk % NS, mbarrier parity = (gk/NS)&1.
template <typename T, class G, bool TMA>
struct Ring {
  T *slots;        // NS slots
  uint64_t *bars;  // NS mbarriers (TMA)
  unsigned gk;     // arrivals consumed so far (this CTA)

  PERKS_DEVINL T *slot(unsigned k) const { return slots + (size_t)(k % G::NS) * G::SLOT; }
  PERKS_DEVINL uint64_t *bar(unsigned k) const { return bars + (k % G::NS); }

  // one-time init (all threads call; thread 0 initialises the barriers)
  PERKS_DEVINL void init(T *s, uint64_t *b, unsigned col_arrivals) {
    slots = s;
    bars = b;
    gk = 0;
    if (TMA && threadIdx.x == 0) {
      for (int i = 0; i < G::NS; i++) mbar_init(bars + i, 1 + col_arrivals);
      mbar_fence_init();
    }
    __syncthreads();
  }

  // Full plane q of buffer `src` (TMA map `map`) into the slot of arrival k.
  PERKS_DEVINL void issue_full(unsigned k, const T *src, const CUtensorMap *map, const Dom3 &d,
                               int q, int x0, int y0, bool col_arrive) {
    if constexpr (TMA) {
      if (threadIdx.x == 0) {
        fence_proxy_async();  // order earlier generic smem writes to this slot before the TMA
        mbar_arrive_tx(bar(k), G::BOX_BYTES);
        tma_load_3d(slot(k), map, x0 - G::PAD, y0 - 1, q, bar(k));
      }
      if (col_arrive && threadIdx.x >= 32 && threadIdx.x < 32 + 2 * G::TY) mbar_arrive(bar(k));
    } else {
      issue_plane<T, G>(slot(k), src, d, q, x0, y0, false);
      cp_async_commit();
    }
  }
  // Ghost plane (multi-GPU, TMA only): plane -1 / nz of this slab lives in the neighbour-written
  // ghost buffer at z coordinate gz; wait until exchange e fully arrived (system-scope acquire),
  // order that acquire before the async-proxy (TMA) read, then load the tile box as usual.
  PERKS_DEVINL void issue_ghost(unsigned k, const CUtensorMap *gmap, int gz, int x0, int y0,
                                const unsigned long long *ctr, unsigned long long target,
                                bool col_arrive) {
    if constexpr (TMA) {
      if (threadIdx.x == 0) {
        wait_counter_sys(ctr, target);
        fence_proxy_async_global();
        fence_proxy_async();
        mbar_arrive_tx(bar(k), G::BOX_BYTES);
        tma_load_3d(slot(k), gmap, x0 - G::PAD, y0 - 1, gz, bar(k));
      }
      if (col_arrive && threadIdx.x >= 32 && threadIdx.x < 32 + 2 * G::TY) mbar_arrive(bar(k));
    }
  }
  // Past the unit's last plane: cp.async commits an empty group so wait_group counting stays
  // uniform; the TMA ring simply does not use the arrival index (indices stay contiguous).
  PERKS_DEVINL void issue_none() {
    if constexpr (!TMA) cp_async_commit();
  }
  // Wait until arrival k's data is resident and visible to all threads.
  PERKS_DEVINL void wait(unsigned k) {
    if constexpr (TMA) {
      mbar_wait(bar(k), (k / G::NS) & 1u);
      __syncthreads();  // also: everyone is done with the slot the next issue overwrites
    } else {
      cp_async_wait<G::NS - 2>();
      __syncthreads();
    }
  }
  PERKS_DEVINL void drain() {
    if constexpr (!TMA) cp_async_wait<0>();
  }
};

// Stream one unit (tile x0,y0; planes [zs, ze)) of one time step from src to dst (no caching).
// Arrivals q = zs-1 .. ze; NS-1 planes in flight.
// Multi-GPU face hooks shared by every 3D kernel (dist.cuh).  `e` = index of the exchange this step
// reads; the step's output planes 0 / nz-1 are exchange e+1.
struct DistStep {
  const DistK *k;  // points at a __grid_constant__ kernel parameter (read from the param bank)
  const CUtensorMap *gmap;
  unsigned long long e;
  unsigned long long plane_cells;  // nx * ny
};
// Which ghost side plane q comes from (-1: an ordinary plane of the local buffers).
PERKS_DEVINL int ghost_side(const DistStep &ds, const Dom3 &d, int q) {
  return (q < 0 && ds.k->has_lo) ? 0 : ((q >= d.nz && ds.k->has_hi) ? 1 : -1);
}
// Issue plane q into ring arrival k from the local buffer or, for a slab face, the ghost planes.
template <typename T, class G, bool TMA, bool DIST>
PERKS_DEVINL void issue_plane_any(Ring<T, G, TMA> &ring, unsigned k, const T *src,
                                  const CUtensorMap *map, const Dom3 &d, int q, int x0, int y0,
                                  bool col_arrive, const DistStep &ds) {
  if constexpr (!DIST) {
    ring.issue_full(k, src, map, d, q, x0, y0, col_arrive);
    return;
  }
  const int gs = ghost_side(ds, d, q);
  if (gs < 0) {
    ring.issue_full(k, src, map, d, q, x0, y0, col_arrive);
  } else {
    ring.issue_ghost(k, ds.gmap, (int)(ds.e & 1) * 2 + gs, x0, y0, ds.k->ctr + gs,
                     (ds.e + 1) * ds.plane_cells, col_arrive);
  }
}
// After output plane o was stored locally: a face plane also goes to the neighbour's ghost plane.
template <typename T, class G>
PERKS_DEVINL void send_face(const DistStep &ds, const Dom3 &d, const ThreadTile<G> &tt, int o,
                            int x0, int y0, const T (&v)[G::R][G::V]) {
  const bool lo = o == 0 && ds.k->has_lo, hi = o == d.nz - 1 && ds.k->has_hi;
  if (!lo && !hi) return;
  const int gz = (int)((ds.e + 1) & 1) * 2 + (lo ? 1 : 0);  // lower neighbour's side 1 / upper's 0
  store_cells<T, G>(reinterpret_cast<T *>(lo ? ds.k->send_lo : ds.k->send_hi), d, tt, gz, v);
  const unsigned long long cells =
      (unsigned long long)min(G::TX, d.nx - x0) * (unsigned long long)min(G::TY, d.ny - y0);
  signal_counter_sys(lo ? ds.k->peer_ctr_lo : ds.k->peer_ctr_hi, cells);  // (local nz >= 2: never both)
}

// PERKS plane cache of one unit (k3d_stream.cu): the cache-code map is indexed by the unit's
// arrival index k (plane czs - 1 + k, k in [0, cze - czs + 2), plus one -1 sentinel), so a lookup is
// one shared-memory load at a fixed offset from the map.
// Cache codes (one signed byte per arrival): -1 = streamed; 0 <= c < kTmemCode: shared-memory
// slot c; c >= kTmemCode: TMEM plane c - kTmemCode (tmem.cuh), staged into the ring slot of its
// arrival one arrival ahead.
constexpr int kTmemCode = 64;
PERKS_DEVINL bool is_smem_code(int c) { return c >= 0 && c < kTmemCode; }
PERKS_DEVINL bool is_tmem_code(int c) { return c >= kTmemCode; }
// Dynamic shared memory of the persistent 3D kernels: ring slots, 128 B of mbarriers and the TMEM
// address, then (PERKS) nc cache slots and the CTA's cache-code map.  Every address is the
// dynamic-smem base plus an offset (no pointer registers).
PERKS_DEVINL unsigned char *dyn_smem() {
  extern __shared__ __align__(128) unsigned char perks_ws_dyn_smem[];
  return perks_ws_dyn_smem;
}
// PERKS plane cache of one CTA (k3d_stream.cu): the cached planes are spread evenly over ALL the
// CTA's units of a step (so the HBM stream of every CTA continues through the whole step); the
// code map is indexed by the CTA's arrival index within the step (units back to back, each unit
// contributing its planes zs-1 .. ze, plus a -1 sentinel).
template <typename T, class G> struct CacheView {
  int nc;          // shared-memory slots of the layout (kernel parameter)
  int kbase;       // arrival index of the current unit's first arrival within the step
  uint32_t tbase;  // TMEM address of cached plane 0 for this thread's warp (lane quarter + column)
  PERKS_DEVINL static T *cache() {
    return reinterpret_cast<T *>(dyn_smem() + G::RING_BYTES);
  }
  PERKS_DEVINL T *slot(int c) const { return cache() + (size_t)c * G::SLOT; }
  PERKS_DEVINL signed char *cmap() const { return reinterpret_cast<signed char *>(cache() + (size_t)nc * G::SLOT); }
};
template <typename T, class G> constexpr int tmem_cpp() {  // TMEM columns per cached plane (tmem.cuh)
  return TmemCells<T, G::R, G::V>::WPT * ((G::NWARP + 3) / 4);
}

template <typename T, class G>
PERKS_DEVINL void write_own(T *slot, const T (&v)[G::R][G::V]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < G::R; r++)
    vstore<T, G::V>(slot + (warp * G::R + r + 1) * G::P + G::PAD + lane * G::V, v[r]);
}
template <typename T, class G>
PERKS_DEVINL void read_own(const T *slot, T (&v)[G::R][G::V]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < G::R; r++)
    vload<T, G::V>(v[r], slot + (warp * G::R + r + 1) * G::P + G::PAD + lane * G::V);
}

// Publish the tile-perimeter cells of cached plane o to dst (neighbours read them as halo): the
// TB-boundary cells "continue to store and load from global memory".  Threads without
// perimeter cells (pmask == 0, most of the tile) skip it in one branch.
template <typename T, class G>
PERKS_DEVINL void publish_perimeter(T *__restrict__ dst, const Dom3 &d, const ThreadTile<G> &tt, int o,
                                    const T (&v)[G::R][G::V]) {
  if (tt.pmask == 0) return;
  T *base = dst + (size_t)o * d.nx * d.ny + (size_t)tt.y * d.nx + tt.x;
#pragma unroll
  for (int r = 0; r < G::R; r++)
#pragma unroll
    for (int i = 0; i < G::V; i++)
      if ((tt.pmask >> (r * G::V + i)) & 1u) base[(size_t)r * d.nx + i] = v[r][i];
}

template <typename T, int S, class G, bool TMA, bool DIST>
PERKS_DEVINL void stream_unit(Ring<T, G, TMA> &ring, const T *__restrict__ src,
                              const CUtensorMap *map, T *__restrict__ dst, const Dom3 &d, int x0,
                              int y0, int zs, int ze, const Coef<T, Shape<S>::N> &c,
                              const DistStep &ds, bool col_arrive = false) {
  constexpr int D = G::NS - 1;
  const int q0 = zs - 1;
  const int narr = ze - zs + 2;
  const unsigned k0 = ring.gk;
  ThreadTile<G> tt;
  tt.init(d, x0, y0);
  auto issue = [&](unsigned k, int q) {
    issue_plane_any<T, G, TMA, DIST>(ring, k, src, map, d, q, x0, y0, col_arrive, ds);
  };
#pragma unroll
  for (int k = 0; k < D; k++) {
    if (k < narr) issue(k0 + k, q0 + k);
    else ring.issue_none();
  }
  StreamState<T, G> st;
  st.zero();
#pragma unroll kWsUnroll
  for (int k = 0; k < narr; k++) {
    const int q = q0 + k;
    ring.wait(k0 + k);
    if (k + D < narr) issue(k0 + k + D, q + D);
    else ring.issue_none();
    T out[G::R][G::V], cq[G::R][G::V];
    arrival<T, S, G>(st, ring.slot(k0 + k), c, out, cq);
    if (q - 1 >= zs) {
      frame_select<T, G>(d, tt, q - 1, out, st.cm1);
      store_cells<T, G>(dst, d, tt, q - 1, out);
      if constexpr (DIST) send_face<T, G>(ds, d, tt, q - 1, x0, y0, out);
    }
#pragma unroll
    for (int r = 0; r < G::R; r++)
#pragma unroll
      for (int i = 0; i < G::V; i++) st.cm1[r][i] = cq[r][i];
  }
  ring.gk = k0 + narr;
  ring.drain();
}


// ================================================================ warp-specialised pipeline (TMA)

// Warps 0..NWARP-1 compute ("consumers"); warp NWARP is the producer.  Slot i of the NS-slot ring
// has two mbarriers: full[i] (1 expect_tx arrival + 32 producer-lane arrivals, TMA/bulk
// transaction bytes) and empty[i] (one arrival per consumer warp).  Consumer warps never
// synchronise with each other per plane — each waits only for the plane it needs and releases it
// when done — so warps drift within the ring depth and latency is hidden with few CTAs per SM
// (the occupancy-vs-concurrency trade-off of P:719-738 without a CTA barrier per plane).
// Arrival index k runs across units and steps; slot = k % NS, phase = (k / NS) & 1.
template <typename T, class G>
struct WsPipe {
  static constexpr unsigned FULL_COUNT = 33;
  // The ring sits at the start of dynamic shared memory (slots, then full / empty / tfull
  // mbarriers): addresses are compile-time offsets from the dynamic-smem base, not registers.
  unsigned gk;
  unsigned tph;     // TMEM tier: phase bit per slot of the tfull mbarriers (after full/empty: one
                    // arrival per consumer warp once its cells are staged; identical sequence)

  PERKS_DEVINL static unsigned char *base() { return dyn_smem(); }
  PERKS_DEVINL static uint64_t *bars() { return reinterpret_cast<uint64_t *>(base() + (size_t)G::NS * G::SLOT_BYTES); }
  PERKS_DEVINL T *slot(unsigned k) const { return reinterpret_cast<T *>(base()) + (size_t)(k % G::NS) * G::SLOT; }
  PERKS_DEVINL uint64_t *fb(unsigned k) const { return bars() + (k % G::NS); }
  PERKS_DEVINL uint64_t *eb(unsigned k) const { return bars() + G::NS + (k % G::NS); }
  PERKS_DEVINL uint64_t *tb(unsigned k) const { return bars() + 2 * G::NS + (k % G::NS); }

  // all threads: thread 0 initialises the barriers
  PERKS_DEVINL void init() {
    gk = 0;
    tph = 0;
    if (threadIdx.x == 0) {
      for (int i = 0; i < G::NS; i++) {
        mbar_init(fb(i), FULL_COUNT);
        mbar_init(eb(i), G::NWARP);
        mbar_init(tb(i), G::NWARP);  // tfull (TMEM tier)
      }
      mbar_fence_init();
    }
    __syncthreads();
  }
  // ---- producer (warp NWARP, all lanes) ----
  // slot of arrival k free again (all consumer warps released arrival k - NS)
  PERKS_DEVINL void acquire(unsigned k) {
    if (k >= G::NS) mbar_wait(eb(k), ((k / G::NS) + 1) & 1u);
    if ((threadIdx.x & 31) == 0) fence_proxy_async();  // consumers' generic reads -> TMA writes
    __syncwarp();
  }
  PERKS_DEVINL void load_box(unsigned k, T *dst, const CUtensorMap *map, int x0, int y0, int z) {
    if ((threadIdx.x & 31) == 0) {
      mbar_arrive_tx(fb(k), G::BOX_BYTES);
      tma_load_3d(dst, map, x0 - G::PAD, y0 - 1, z, fb(k));
    }
    mbar_arrive(fb(k));
  }
  PERKS_DEVINL void load_full(unsigned k, const CUtensorMap *map, int x0, int y0, int q) {
    load_box(k, slot(k), map, x0, y0, q);
  }
  PERKS_DEVINL void load_ghost(unsigned k, const CUtensorMap *gmap, int gz, int x0, int y0,
                               const unsigned long long *ctr, unsigned long long target) {
    if ((threadIdx.x & 31) == 0) {
      wait_counter_sys(ctr, target);
      fence_proxy_async_global();
    }
    __syncwarp();
    load_box(k, slot(k), gmap, x0, y0, gz);
  }
  // halo ring only (PERKS cached plane q) into `dst` (a cache slot, or the ring slot of a TMEM
  // plane whose interior the consumers stage): rows by bulk copies (lane 0), the two columns by
  // per-lane cp.async completing on the same barrier.  Halo cells are never cached.
  PERKS_DEVINL void load_halo(unsigned k, T *dst, const T *src, const Dom3 &d, int q, int x0, int y0) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
      const int xa = max(x0 - G::PAD, 0), xb = min(x0 + G::TX + G::PAD, d.nx);
      const unsigned rb = (unsigned)((xb - xa) * (int)sizeof(T));
      const bool top = y0 >= 1, bot = y0 + G::TY < d.ny;
      mbar_arrive_tx(fb(k), (top ? rb : 0u) + (bot ? rb : 0u));
      const size_t pl = (size_t)d.nx * d.ny;
      if (top) bulk_load(dst + (xa - (x0 - G::PAD)), src + (size_t)q * pl + (size_t)(y0 - 1) * d.nx + xa, rb, fb(k));
      if (bot)
        bulk_load(dst + (G::ROWS - 1) * G::P + (xa - (x0 - G::PAD)),
                  src + (size_t)q * pl + (size_t)(y0 + G::TY) * d.nx + xa, rb, fb(k));
    }
    for (int t = lane; t < 2 * G::TY; t += 32) {
      const int j = 1 + (t >> 1);
      const bool right = t & 1;
      const int y = y0 - 1 + j;
      const int xx = right ? x0 + G::TX : x0 - 1;
      const bool ok = y < d.ny && xx >= 0 && xx < d.nx;
      const T *g = ok ? src + ((size_t)q * d.ny + y) * d.nx + xx : src;
      cp_async<(int)sizeof(T)>(dst + j * G::P + (right ? G::PAD + G::TX : G::PAD - 1), g, ok);
    }
    mbar_arrive_cpasync(fb(k));
  }
  // ---- consumers (warps 0..NWARP-1) ----
  PERKS_DEVINL void wait_full(unsigned k) { mbar_wait(fb(k), (k / G::NS) & 1u); }
  PERKS_DEVINL void release(unsigned k) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive_release(eb(k));
  }
  // every consumer warp has released arrival k (its slot's reads are complete)
  PERKS_DEVINL void wait_released(unsigned k) { mbar_wait(eb(k), (k / G::NS) & 1u); }
  // TMEM tier: this warp's cells of arrival k are in its slot / every warp's are
  PERKS_DEVINL void staged(unsigned k) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive_release(tb(k));
  }
  PERKS_DEVINL void wait_staged(unsigned k) {
    const unsigned i = k % G::NS;
    mbar_wait(tb(k), (tph >> i) & 1u);
    tph ^= 1u << i;
  }
};

// Named barrier over the consumer warps only (the producer keeps streaming).
template <class G> PERKS_DEVINL void consumers_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(32 * G::NWARP) : "memory");
}

// Face plane o to the neighbour's ghost plane (multi-GPU), consumer warps only.
template <typename T, class G>
PERKS_DEVINL void send_face_ws(const DistStep &ds, const Dom3 &d, const ThreadTile<G> &tt, int o,
                               int x0, int y0, const T (&v)[G::R][G::V]) {
  const bool lo = o == 0 && ds.k->has_lo, hi = o == d.nz - 1 && ds.k->has_hi;
  if (!lo && !hi) return;
  const int gz = (int)((ds.e + 1) & 1) * 2 + (lo ? 1 : 0);
  store_cells<T, G>(reinterpret_cast<T *>(lo ? ds.k->send_lo : ds.k->send_hi), d, tt, gz, v);
  __threadfence_system();
  consumers_sync<G>();
  if (threadIdx.x == 0) {
    const unsigned long long cells =
        (unsigned long long)min(G::TX, d.nx - x0) * (unsigned long long)min(G::TY, d.ny - y0);
    red_release_sys_add_u64(lo ? ds.k->peer_ctr_lo : ds.k->peer_ctr_hi, cells);
  }
}

// TMEM tier, consumer warp: the thread's own cells of TMEM plane t into the ring slot of arrival k
// (the producer loads the slot's halo ring), then this warp's arrival on the slot's tfull barrier.
template <typename T, class G>
PERKS_DEVINL void stage_tmem_plane(WsPipe<T, G> &pp, const CacheView<T, G> &cv, unsigned k, int t) {
  T v[G::R][G::V];
  TmemCells<T, G::R, G::V>::load(cv.tbase + (uint32_t)(t * tmem_cpp<T, G>()), v);
  write_own<T, G>(pp.slot(k), v);
  pp.staged(k);
}

// One unit (tile x0,y0; planes [zs, ze)) of one step through the warp-specialised pipeline.
// Called by ALL warps of the CTA; the producer issues arrivals zs-1 .. ze, the consumers run the
// staged plane body (arrival(), stages A/B/C) and store / cache the outputs.
template <typename T, int S, class G, bool DIST, bool CACHE = false>
PERKS_DEVINL void stream_unit_ws(WsPipe<T, G> &pp, const T *__restrict__ src, const CUtensorMap *map,
                                 T *__restrict__ dst, const Dom3 &d, int x0, int y0, int zs, int ze,
                                 const Coef<T, Shape<S>::N> &c, const DistStep &ds,
                                 const CacheView<T, G> &cv = CacheView<T, G>{}) {
  const int q0 = zs - 1;
  const int narr = ze - zs + 2;
  const unsigned k0 = pp.gk;
  const signed char *cmk = CACHE ? cv.cmap() + cv.kbase : nullptr;  // this unit's arrival codes
  auto cs = [&](int k) -> int {
    if constexpr (!CACHE) return -1;
    return (int)cmk[k];
  };
  pp.gk = k0 + narr;
  if ((int)(threadIdx.x >> 5) == G::NWARP) {  // ---- producer
    for (int k = 0; k < narr; k++) {
      const unsigned kk = k0 + k;
      const int q = q0 + k;
      pp.acquire(kk);
      const int sl = cs(k);
      if (CACHE && is_smem_code(sl)) {
        pp.load_halo(kk, cv.slot(sl), src, d, q, x0, y0);
      } else if (CACHE && is_tmem_code(sl)) {
        pp.load_halo(kk, pp.slot(kk), src, d, q, x0, y0);  // interior staged by the consumers
      } else {
        const int gs = DIST ? ghost_side(ds, d, q) : -1;
        if (gs < 0) pp.load_full(kk, map, x0, y0, q);
        else pp.load_ghost(kk, ds.gmap, (int)(ds.e & 1) * 2 + gs, x0, y0, ds.k->ctr + gs,
                           (ds.e + 1) * ds.plane_cells);
      }
    }
    return;
  }
  // ---- consumers
  ThreadTile<G> tt;
  tt.init(d, x0, y0);
  StreamState<T, G> st;
  st.zero();
  // output plane o = zs, zs+1, ... in arrival order: the fast-path store pointer just advances
  const size_t plane = (size_t)d.nx * d.ny;
  T *sp = dst + (size_t)zs * plane + tt.off(d);
  int slq = cs(0), slo = -1;  // cache codes of this arrival / of the output plane (rotated)
#pragma unroll kWsUnroll  // (3: the accumulator rotation of arrival() becomes renaming)
  for (int k = 0; k < narr; k++) {
    const unsigned kk = k0 + k;
    const int q = q0 + k;
    const int sln = cs(k + 1);  // next arrival's code (sentinel -1 after the unit's last)
    pp.wait_full(kk);
    if (CACHE && is_tmem_code(slq)) pp.wait_staged(kk);
    T out[G::R][G::V], cq[G::R][G::V];
    {  // the plane's slot: a cache slot or the ring slot, as one offset from the dynamic-smem base
      const size_t off = (CACHE && is_smem_code(slq)) ? G::RING_BYTES + (size_t)slq * G::SLOT_BYTES
                                                       : (size_t)(kk % G::NS) * G::SLOT_BYTES;
      arrival<T, S, G>(st, reinterpret_cast<const T *>(dyn_smem() + off), c, out, cq);
    }
    pp.release(kk);
    if (q - 1 >= zs) {
      frame_select<T, G>(d, tt, q - 1, out, st.cm1);
      if (CACHE && is_smem_code(slo)) {
        // cached output: stays on chip once every warp has finished reading the old plane
        publish_perimeter<T, G>(dst, d, tt, q - 1, out);
        pp.wait_released(kk - 1);
        write_own<T, G>(cv.slot(slo), out);
      } else if (CACHE && is_tmem_code(slo)) {
        // TMEM-cached output: the thread's own columns (plane q-1 was staged from them at
        // arrival q-2, before this write in program order)
        publish_perimeter<T, G>(dst, d, tt, q - 1, out);
        TmemCells<T, G::R, G::V>::store(cv.tbase + (uint32_t)((slo - kTmemCode) * tmem_cpp<T, G>()), out);
      } else {
        if (tt.full) {
#pragma unroll
          for (int r = 0; r < G::R; r++) vstore<T, G::V>(sp + (size_t)r * d.nx, out[r]);
        } else {
          store_cells<T, G>(dst, d, tt, q - 1, out);
        }
        if constexpr (DIST) send_face_ws<T, G>(ds, d, tt, q - 1, x0, y0, out);
      }
      sp += plane;
    }
#pragma unroll
    for (int r = 0; r < G::R; r++)
#pragma unroll
      for (int i = 0; i < G::V; i++) st.cm1[r][i] = cq[r][i];
    slo = slq;
    slq = sln;
    if constexpr (CACHE) {
      // TMEM tier: stage the NEXT arrival's cells (TMEM -> registers -> its ring slot) one
      // arrival ahead, at the point of the body with the fewest live registers
      if (is_tmem_code(sln)) {
        if (kk + 1 >= (unsigned)G::NS) pp.wait_released(kk + 1 - G::NS);  // slot free
        stage_tmem_plane<T, G>(pp, cv, kk + 1, sln - kTmemCode);
      }
    }
  }
}

}  // namespace perks
