// k3d_tb.cu — PERKS (c) for 3D domains beyond the on-chip capacity: the persistent plane-streaming
// kernel advancing TWO time steps per pass over the domain, with the intermediate time level kept
// on chip (Tiled PERKS, [draft] P:416-441, in its streaming form; DESIGN.md §7 reading R13).
//
// The paper's PERKS caches part of the domain between time steps so that it is not re-read from
// global memory.  For a 3D domain several times the on-chip capacity (C3: 134 MB
// vs ~70 MB of shared memory + TMEM over 148 SMs; C4: 537 MB) what can stay on chip across a time
// step is the wavefront of planes in flight: here each CTA streams its unit (an xy tile, a z
// range) once per PAIR of steps and keeps time level t+1 of the planes in flight in shared memory,
// so DRAM moves 2·S bytes per cell per two steps instead of per step (A_gm halved).  The
// draft's Tiled PERKS "has a redundant halo region to enable the execution of consecutive time
// steps" and notes that "optimization methods related to temporal blocking are all applicable"
// (P:433-439): the redundancy here is a one-cell ring of level t+1 around each tile.
//
// Per CTA (one per SM, cooperative launch, grid barrier between passes):
//   * producer warp: TMA boxes {P, TY+4, 1} of the input planes (a two-cell halo in x and y,
//     zero-filled outside the domain) into an NS-slot ring (full/empty mbarriers);
//   * main warps (8): thread (lane, warp) owns V x R cells of the TX x TY output window.  Stage 1
//     applies plane p's chain terms to level t+1 of planes p-1..p+1 (stream3d.cuh arrival(),
//     reading R5 order), writes the finished plane p-1 of level t+1 into one of two intermediate
//     (IS) slots; stage 2 applies the previous tick's IS plane to level t+2 and stores the finished
//     output plane to HBM;
//   * halo warps: level t+1 on the one-cell ring around the window (2(TX+2) + 2TY cells per plane,
//     one cell per lane and pass of the loop), written into the same IS slot;
//   * one named barrier over main + halo warps per tick (IS slot written -> read next tick).
// Frame cells (reading R1) keep their value at both levels (frame_select with the stage's own
// centre), so the two-level result is bit-identical to two single steps.  Odd T: the first pass
// runs one step (stage 1 stored directly).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <type_traits>

#include "internal.h"
#include "stream3d.cuh"

namespace perks {

bool use_tma3(const Problem &p);
bool encode_map3(CUtensorMap *m, const Problem &p, const void *base, int bx, int by, int promo);
DistK make_distk(const DistRun *dr);

// Stage 2 takes its own cells from registers (1) or re-reads them from the IS slot (0: fewer live
// registers).
#ifndef PERKS_TB_OWN
#define PERKS_TB_OWN 1
#endif
constexpr bool kTbOwn = PERKS_TB_OWN != 0;
#ifndef PERKS_TB_NI
#define PERKS_TB_NI 4
#endif
// Tick order: 1 = stage 1 (input plane -> IS) then stage 2 (previous IS plane -> output); 0 = the reverse.
#ifndef PERKS_TB_S1FIRST
#define PERKS_TB_S1FIRST 0
#endif
constexpr bool kTbS1First = PERKS_TB_S1FIRST != 0;
// fp64: stage 1 first with stage 2's own cells re-read from the IS slot (PERKS_TB_F64_S1FIRST=1,
// measured 4 % faster on C3, profiles/r02_tb3d_variants4.txt "s1o0"; fp32 spills in that form)
#ifndef PERKS_TB_F64_S1FIRST
#define PERKS_TB_F64_S1FIRST 1
#endif
template <typename T> constexpr bool tb_s1first() { return sizeof(T) == 8 ? PERKS_TB_F64_S1FIRST != 0 : kTbS1First; }
template <typename T> constexpr bool tb_own() { return sizeof(T) == 8 && PERKS_TB_F64_S1FIRST != 0 ? false : kTbOwn; }
// Stage 2 of the z-major shapes (19/27-point: list = dz -1 terms, then 0, then +1) evaluated
// directly from three resident IS planes (no accumulator state across ticks: frees the registers
// of a second set of three accumulators); the 7-point star keeps the arrival form.
#ifndef PERKS_TB_D2
#define PERKS_TB_D2 1
#endif
#ifndef PERKS_TB_R27
#define PERKS_TB_R27 4
#endif
#ifndef PERKS_TB_NS
#define PERKS_TB_NS 4
#endif

// Rows per thread: 4 for the 7-point star (two accumulator arrays per level: (R+2)/R = 1.5 row
// reads per cell), 2 for the box / 19-point shapes (four arrays per level).
#ifndef PERKS_TB_R7
#define PERKS_TB_R7 4
#endif
#ifndef PERKS_TB_NW7
#define PERKS_TB_NW7 8
#endif
template <int S> constexpr bool z_major() {
  for (int p = 1; p < Shape<S>::N; p++)
    if (Shape<S>::dz(p) < Shape<S>::dz(p - 1)) return false;
  return true;
}
template <int S> constexpr int first_dz_at_least(int z) {
  int p = 0;
  while (p < Shape<S>::N && Shape<S>::dz(p) < z) p++;
  return p;
}
template <int S> constexpr bool tb_direct2() { return PERKS_TB_D2 != 0 && S != SHAPE_3D7 && z_major<S>(); }

template <typename T, int S> struct TbG {
  static constexpr int V = 16 / (int)sizeof(T), R = S == SHAPE_3D7 ? PERKS_TB_R7 : PERKS_TB_R27;
  static constexpr int NWARP = S == SHAPE_3D7 ? PERKS_TB_NW7 : 8, NS = PERKS_TB_NS;
  using G = Geo3D<T, V, R, NWARP, NS>;  // compute geometry (IS slot = G::SLOT: TY+2 rows of pitch P)
  static constexpr int TX = G::TX, TY = G::TY, P = G::P, PAD = G::PAD;
  static_assert(PAD >= 2, "two-cell x halo inside the row padding");
  static constexpr int RI = TY + 4;  // input box rows (two-cell y halo)
  static constexpr int IN_SLOT = (RI * P * (int)sizeof(T) + 127) / 128 * 128 / (int)sizeof(T);
  static constexpr unsigned IN_BOX_BYTES = (unsigned)(RI * P * sizeof(T));
  static constexpr int RING = 2 * (TX + 2) + 2 * TY;  // level t+1 cells around the window
  // halo warps: 3, so that main + halo + producer = 12 warps = 3 per SM sub-partition (a 13th warp
  // would cap the register budget at 128 per thread: 4 warps x 128 x 32 = one 16K-entry SMSP file)
  static constexpr int NHW = 3;
  static constexpr int HC = (RING + 32 * NHW - 1) / (32 * NHW);
  static constexpr int NCW = NWARP + NHW;  // consumer warps (main + halo)
  static constexpr int NTHR = 32 * (NCW + 1);
  // IS slots (direct stage 2: three resident + one being written)
  static constexpr int NI = PERKS_TB_NI;
  // The input arrival and IS plane counters are 32-bit and wrap on very long runs: slot = k % N and
  // phase = (k / N) & 1 stay continuous across the wrap only when N divides 2^31.
  static_assert((NS & (NS - 1)) == 0 && (NI & (NI - 1)) == 0, "ring depths must be powers of two");
  static_assert(!tb_direct2<S>() || NI >= 4, "direct stage 2: three resident IS planes + one being written");
  static constexpr size_t IS_OFF = (size_t)NS * IN_SLOT * sizeof(T);
  static constexpr size_t BAR_OFF = IS_OFF + (size_t)NI * G::SLOT_BYTES;
  // full[NS], empty[NS] (input ring), written[NI] (NCW arrivals), read[NI] (NWARP arrivals)
  static constexpr size_t SMEM = BAR_OFF + (2 * NS + 2 * NI) * 8;
};

struct TbMaps {
  CUtensorMap m[3];  // in, out, tmp: box {P, TY+4, 1}
  CUtensorMap ghost; // multi-GPU slabs: the ghost planes G[12][ny][nx], same box
};
// Multi-GPU slabs: ghost planes 4..11 of the library-owned G hold this kernel's
// exchanges, two planes per face and parity: plane 4 + parity*4 + side*2 + j, side 0 = planes -2, -1
// (j = 0, 1) from the lower neighbour, side 1 = planes nz, nz+1 from the upper neighbour (planes
// 0..3 belong to the one-step slab kernels).  Exchange k (0 = the run's input, k = pass + 1 = that
// pass's output) carries two planes per face; the arrival counters count cells, so exchange k is
// complete when a side's counter reaches (xbase + 2k + 2) * nx*ny (xbase in plane units).
PERKS_DEVINL int tb_ghost_plane(unsigned long long ex, int side, int j) {
  return 4 + (int)(ex & 1ull) * 4 + side * 2 + j;
}
struct TbUnits {
  int tx, ty, nzc, zc, rev;
  int range;  // 1: CTA b owns the contiguous run [b W / G, (b+1) W / G) of the W = tiles * nz
              // (tile, plane) sequence, split at tile boundaries (balanced work, one pipeline fill
              // per tile touched); 0: units of zc planes strided over the grid
};

// Single-cell geometry for the halo warps' chain (apply_terms needs only R and V).
struct G11 {
  static constexpr int R = 1, V = 1;
};

// arrival() of stream3d.cuh for one cell whose 3x3 neighbourhood in plane q is already loaded.
template <typename T, int S>
PERKS_DEVINL void arrival_cell(StreamState<T, G11> &st, const T (&nb)[3][3], const Coef<T, Shape<S>::N> &c,
                               T &out, T &center_q) {
  constexpr int e0 = stage_end<S>(0), e1 = stage_end<S>(1), e2 = stage_end<S>(2);
  center_q = nb[1][1];
  apply_terms<T, S, G11, e1, e2, 1>(st.accC, nb, st.cm1, c);
  out = st.accC[0][0];
  apply_terms<T, S, G11, e0, e1, 0>(st.accB, nb, st.cm1, c);
  apply_terms<T, S, G11, 0, e0, -1>(st.accA, nb, st.cm1, c);
  st.accC[0][0] = st.accB[0][0];
  st.accB[0][0] = st.accA[0][0];
}

// Producer's wait for a free slot: try_wait with a suspend-time hint (the thread sleeps until the
// phase completes or ~hint ns pass instead of re-polling and taking issue slots from the SMSP's
// consumer warps); watchdog as mbar_wait.
PERKS_DEVINL void mbar_wait_sleep(uint64_t *b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      ".reg .u64 t0, t1;\n"
      "mov.u64 t0, %%globaltimer;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %3;\n"
      "@p bra DONE_%=;\n"
      "mov.u64 t1, %%globaltimer;\n"
      "sub.u64 t1, t1, t0;\n"
      "setp.gt.u64 p, t1, %2;\n"
      "@p trap;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity), "l"((unsigned long long)PERKS_WATCHDOG_NS), "r"(20000u)
      : "memory");
}

// Stage 2's input neighbourhood: the thread's own R x V cells of the IS plane are the level t+1
// values it computed (and wrote) one tick earlier, kept in registers; only the x-neighbours of
// those rows and the rows above / below come from shared memory.
template <typename T, class G>
PERKS_DEVINL void read_nb_own(const T *slot, const T (&own)[G::R][G::V], T (&nb)[G::R + 2][G::V + 2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < G::R + 2; j++) {
    const T *row = slot + (warp * G::R + j) * G::P + G::PAD + lane * G::V;
    nb[j][0] = row[-1];
    nb[j][G::V + 1] = row[G::V];
    if (j == 0 || j == G::R + 1) {
      T v[G::V];
      vload<T, G::V>(v, row);
#pragma unroll
      for (int i = 0; i < G::V; i++) nb[j][i + 1] = v[i];
    } else {
#pragma unroll
      for (int i = 0; i < G::V; i++) nb[j][i + 1] = own[j - 1][i];
    }
  }
}

// One output plane of a z-major shape from its three input planes (slots of planes o-1, o, o+1),
// the chain in list order (reading R5), each plane's neighbourhood read once; `cen` = plane o's own
// cells (the frame rule's old values).
template <typename T, int S, class G>
PERKS_DEVINL void direct_plane(const T *sm1, const T *s0, const T *sp1, const Coef<T, Shape<S>::N> &c,
                               T (&out)[G::R][G::V], T (&cen)[G::R][G::V]) {
  constexpr int z0 = first_dz_at_least<S>(0), z1 = first_dz_at_least<S>(1);
  static_assert(z_major<S>() && z0 > 0, "direct_plane: z-major list starting with dz = -1 terms");
  {
    T nb[G::R + 2][G::V + 2];
    read_nb<T, G>(sm1, nb);
    apply_terms<T, S, G, 0, z0, -1>(out, nb, cen, c);
  }
  {
    T nb[G::R + 2][G::V + 2];
    read_nb<T, G>(s0, nb);
#pragma unroll
    for (int r = 0; r < G::R; r++)
#pragma unroll
      for (int i = 0; i < G::V; i++) cen[r][i] = nb[r + 1][i + 1];
    apply_terms<T, S, G, z0, z1, 0>(out, nb, cen, c);
  }
  {
    T nb[G::R + 2][G::V + 2];
    read_nb<T, G>(sp1, nb);
    apply_terms<T, S, G, z1, Shape<S>::N, 1>(out, nb, cen, c);
  }
}

// arrival() of stream3d.cuh with the plane-q neighbourhood already in registers.
template <typename T, int S, class G>
PERKS_DEVINL void arrival_nb(StreamState<T, G> &st, const T (&nb)[G::R + 2][G::V + 2], const Coef<T, Shape<S>::N> &c,
                             T (&out)[G::R][G::V], T (&center_q)[G::R][G::V]) {
  constexpr int e0 = stage_end<S>(0), e1 = stage_end<S>(1), e2 = stage_end<S>(2);
#pragma unroll
  for (int r = 0; r < G::R; r++)
#pragma unroll
    for (int i = 0; i < G::V; i++) center_q[r][i] = nb[r + 1][i + 1];
  apply_terms<T, S, G, e1, e2, 1>(st.accC, nb, st.cm1, c);
#pragma unroll
  for (int r = 0; r < G::R; r++)
#pragma unroll
    for (int i = 0; i < G::V; i++) out[r][i] = st.accC[r][i];
  apply_terms<T, S, G, e0, e1, 0>(st.accB, nb, st.cm1, c);
  apply_terms<T, S, G, 0, e0, -1>(st.accA, nb, st.cm1, c);
#pragma unroll
  for (int r = 0; r < G::R; r++)
#pragma unroll
    for (int i = 0; i < G::V; i++) {
      st.accC[r][i] = st.accB[r][i];
      st.accB[r][i] = st.accA[r][i];
    }
}

template <typename T, int S, bool DIST>
__global__ void __launch_bounds__(TbG<T, S>::NTHR, 1)
    tb3d_kernel(const T *__restrict__ in, T *out, T *tmp, const __grid_constant__ TbMaps maps, Dom3 d, TbUnits u,
                int64_t steps, unsigned *bar, Coef<T, Shape<S>::N> c, const __grid_constant__ DistK dk,
                unsigned long long xbase, unsigned long long tbx) {
  using B = TbG<T, S>;
  using G = typename B::G;
  unsigned char *sm = dyn_smem();
  T *const in_slots = reinterpret_cast<T *>(sm);
  T *const is_slots = reinterpret_cast<T *>(sm + B::IS_OFF);
  uint64_t *const bars = reinterpret_cast<uint64_t *>(sm + B::BAR_OFF);
  auto in_slot = [&](unsigned k) { return in_slots + (size_t)(k % B::NS) * B::IN_SLOT; };
  auto fullb = [&](unsigned k) { return bars + (k % B::NS); };
  auto emptyb = [&](unsigned k) { return bars + B::NS + (k % B::NS); };
  auto isw = [&](unsigned q) { return bars + 2 * B::NS + (q % B::NI); };          // IS q written
  auto isr = [&](unsigned q) { return bars + 2 * B::NS + B::NI + (q % B::NI); };  // IS q read

  const int warp = (int)(threadIdx.x >> 5), lane = (int)(threadIdx.x & 31);
  if (threadIdx.x == 0) {
    for (int i = 0; i < B::NS; i++) {
      mbar_init(bars + i, 1);
      mbar_init(bars + B::NS + i, B::NCW);
    }
    for (int i = 0; i < B::NI; i++) {
      mbar_init(bars + 2 * B::NS + i, B::NCW);
      mbar_init(bars + 2 * B::NS + B::NI + i, B::NWARP);
    }
    mbar_fence_init();
  }
  // zero the IS slots once: cells outside window + ring are never written (nor read for kept cells)
  for (int i = threadIdx.x; i < B::NI * G::SLOT; i += blockDim.x) is_slots[i] = T(0);
  __syncthreads();

  const int tiles = u.tx * u.ty;
  const int nunits = tiles * u.nzc;
  const long long W = (long long)tiles * d.nz;
  const long long rlo = W * (long long)blockIdx.x / (long long)gridDim.x;
  const long long rhi = W * ((long long)blockIdx.x + 1) / (long long)gridDim.x;
  const int nmine = u.range ? (rhi > rlo ? (int)((rhi - 1) / d.nz - rlo / d.nz) + 1 : 0)
                            : ((int)blockIdx.x < nunits ? (nunits - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0);
  const size_t plane = (size_t)d.nx * d.ny;
  const int64_t npass = (steps + 1) / 2;
  unsigned gk = 0;  // input arrivals so far (slot = gk % NS, phase = (gk / NS) & 1)
  unsigned gi = 0;  // IS planes written so far (slot = q % NI, phase = (q / NI) & 1)

  for (int64_t ps = 0; ps < npass; ps++) {
    const int nst = (ps == 0 && (steps & 1)) ? 1 : 2;
    const bool src_out = ps > 0 && ((npass - ps) & 1) == 0;
    const T *src = ps == 0 ? in : (src_out ? out : tmp);
    const int src_idx = ps == 0 ? 0 : (src_out ? 1 : 2);
    T *dst = ((npass - 1 - ps) & 1) == 0 ? out : tmp;
    (void)src;
    const bool rev = u.rev && (ps & 1);  // L2-aware traversal (zig-zag, [draft] P:395-404)
    for (int jj = 0; jj < nmine; jj++) {
      const int j = rev ? nmine - 1 - jj : jj;
      int t, zs, ze;
      if (u.range) {
        t = (int)(rlo / d.nz) + j;
        zs = j == 0 ? (int)(rlo % d.nz) : 0;
        ze = j == nmine - 1 ? (int)((rhi - 1) % d.nz) + 1 : d.nz;
      } else {
        const int id = (int)blockIdx.x + j * (int)gridDim.x;
        t = id % tiles;
        zs = (id / tiles) * u.zc;
        ze = min(zs + u.zc, d.nz);
      }
      const int x0 = (t % u.tx) * B::TX, y0 = (t / u.tx) * B::TY;
      const int zc = ze - zs;
      const int nin = nst == 2 ? zc + 4 : zc + 2;  // input planes zs-2..ze+1 (zs-1..ze)
      const int q0 = nst == 2 ? zs - 2 : zs - 1;
      const unsigned k0 = gk;
      gk += (unsigned)nin;
      const unsigned i0 = gi;  // IS plane of tick k: written i0 + k - 2, read by stage 2 at tick k + 1
      if (nst == 2) gi += (unsigned)(zc + 2);
      // IS plane q: slot / wait before writing (its previous use read) / publish / consume
      auto is_of = [&](unsigned q) { return is_slots + (size_t)(q % B::NI) * G::SLOT; };
      auto is_acquire_w = [&](unsigned q) {
        if (q >= (unsigned)B::NI) mbar_wait(isr(q), ((q / B::NI) + 1) & 1u);
      };
      auto is_publish = [&](unsigned q) {
        __syncwarp();
        if (lane == 0) mbar_arrive_release(isw(q));
      };
      auto is_acquire_r = [&](unsigned q) {
        mbar_wait(isw(q), (q / B::NI) & 1u);
      };
      auto is_done_r = [&](unsigned q) {
        __syncwarp();
        if (lane == 0) mbar_arrive_release(isr(q));
      };
      if (warp == B::NCW) {  // ---------------------------------------------------------- producer
        if (lane == 0) {
          if (jj == 0) fence_proxy_async_global();  // previous pass's generic stores -> TMA reads
          for (int k = 0; k < nin; k++) {
            const unsigned kk = k0 + (unsigned)k;
            if (kk >= (unsigned)B::NS) mbar_wait_sleep(emptyb(kk), ((kk / B::NS) + 1) & 1u);
            const int q = q0 + k;
            const int gs = DIST ? ((q < 0 && dk.has_lo) ? 0 : ((q >= d.nz && dk.has_hi) ? 1 : -1)) : -1;
            if (gs >= 0) {  // a neighbour's plane: wait until exchange ps fully arrived
              wait_counter_sys(dk.ctr + gs, (xbase + 2ull * (unsigned long long)ps + 2ull) * plane);
              fence_proxy_async_global();
            }
            fence_proxy_async();
            mbar_arrive_tx(fullb(kk), B::IN_BOX_BYTES);
            if (gs >= 0)
              tma_load_3d(in_slot(kk), &maps.ghost, x0 - B::PAD, y0 - 2,
                          tb_ghost_plane(tbx + (unsigned long long)ps, gs, gs == 0 ? q + 2 : q - d.nz), fullb(kk));
            else
              tma_load_3d(in_slot(kk), &maps.m[src_idx], x0 - B::PAD, y0 - 2, q, fullb(kk));
          }
        }
        __syncwarp();
        continue;
      }
      auto release = [&](unsigned kk) {
        __syncwarp();
        if (lane == 0) mbar_arrive_release(emptyb(kk));
      };
      if (warp < B::NWARP) {  // -------------------------------------------------------- main warps
        ThreadTile<G> tt;
        tt.init(d, x0, y0);
        StreamState<T, G> s1, s2;
        s1.zero();
        s2.zero();
        T own[G::R][G::V];  // this thread's cells of the IS plane written last tick
        T own_next[tb_s1first<T>() ? G::R : 1][G::V];  // (stage-1-first order: this tick's, until stage 2 ran)
        T *sp = dst + (size_t)zs * plane + tt.off(d);
        auto store = [&](int o, const T (&v)[G::R][G::V]) {
          if (tt.full) {
#pragma unroll
            for (int r = 0; r < G::R; r++) vstore<T, G::V>(sp + (size_t)r * d.nx, v[r]);
          } else {
            store_cells<T, G>(dst, d, tt, o, v);
          }
          sp += plane;
          if constexpr (DIST) {  // face planes of this pass's output to the neighbours' ghosts
            const bool lo = dk.has_lo && o <= 1, hi = dk.has_hi && o >= d.nz - 2;
            if (lo || hi) {
              const unsigned long long ex = tbx + (unsigned long long)ps + 1ull;
              if (lo) store_cells<T, G>(reinterpret_cast<T *>(dk.send_lo), d, tt, tb_ghost_plane(ex, 1, o), v);
              if (hi) store_cells<T, G>(reinterpret_cast<T *>(dk.send_hi), d, tt, tb_ghost_plane(ex, 0, o - (d.nz - 2)), v);
              __threadfence_system();
              asm volatile("bar.sync 2, %0;\n" ::"n"(32 * B::NWARP) : "memory");
              if (threadIdx.x == 0) {
                const unsigned long long cells =
                    (unsigned long long)min(B::TX, d.nx - x0) * (unsigned long long)min(B::TY, d.ny - y0);
                if (lo) red_release_sys_add_u64(dk.peer_ctr_lo, cells);
                if (hi) red_release_sys_add_u64(dk.peer_ctr_hi, cells);
              }
            }
          }
        };
        if (nst == 1) {
          for (int k = 0; k < nin; k++) {
            const unsigned kk = k0 + (unsigned)k;
            mbar_wait(fullb(kk), (kk / B::NS) & 1u);
            T o1[G::R][G::V], c1[G::R][G::V];
            arrival<T, S, G>(s1, in_slot(kk) + G::P, c, o1, c1);
            release(kk);
            if (k >= 2) {
              frame_select<T, G>(d, tt, zs - 2 + k, o1, s1.cm1);
              store(zs - 2 + k, o1);
            }
#pragma unroll
            for (int r = 0; r < G::R; r++)
#pragma unroll
              for (int i = 0; i < G::V; i++) s1.cm1[r][i] = c1[r][i];
          }
          continue;
        }
        // One tick: stage 2 on the IS plane written last tick (A2; ST: store its output), stage 1 on
        // input plane zs-2+k (A1; W1: write its output to the IS slot); order per tb_s1first.
        auto tick = [&](int k, auto a1, auto a2, auto st, auto w1) {
          constexpr bool A1 = decltype(a1)::value, A2 = decltype(a2)::value;
          constexpr bool ST = decltype(st)::value, W1 = decltype(w1)::value;
          const unsigned kk = k0 + (unsigned)k;
          T o2[G::R][G::V], c2[G::R][G::V], o1[G::R][G::V], c1[G::R][G::V];
          auto stage2 = [&]() {
            if constexpr (tb_direct2<S>()) {  // output plane zs-5+k from IS planes zs-6+k .. zs-4+k
              if constexpr (ST) {
                const unsigned qa = i0 + (unsigned)(k - 5);
                is_acquire_r(qa);
                is_acquire_r(qa + 1);
                is_acquire_r(qa + 2);
                direct_plane<T, S, G>(is_of(qa), is_of(qa + 1), is_of(qa + 2), c, o2, c2);
                is_done_r(qa);  // plane zs-6+k: its last read
              }
            } else {
              T nb[G::R + 2][G::V + 2];
              const unsigned q = i0 + (unsigned)(k - 3);
              is_acquire_r(q);
              if constexpr (tb_own<T>()) read_nb_own<T, G>(is_of(q), own, nb);
              else read_nb<T, G>(is_of(q), nb);
              is_done_r(q);
              arrival_nb<T, S, G>(s2, nb, c, o2, c2);
            }
          };
          auto stage2_out = [&]() {
            if constexpr (tb_direct2<S>()) {
              if constexpr (ST) {
                frame_select<T, G>(d, tt, zs - 5 + k, o2, c2);
                store(zs - 5 + k, o2);
              }
            } else {
              if constexpr (ST) {
                frame_select<T, G>(d, tt, zs - 5 + k, o2, s2.cm1);
                store(zs - 5 + k, o2);
              }
#pragma unroll
              for (int r = 0; r < G::R; r++)
#pragma unroll
                for (int i = 0; i < G::V; i++) s2.cm1[r][i] = c2[r][i];
            }
          };
          auto stage1 = [&]() {
            T nb[G::R + 2][G::V + 2];
            read_nb<T, G>(in_slot(kk) + G::P, nb);
            arrival_nb<T, S, G>(s1, nb, c, o1, c1);
          };
          auto stage1_out = [&]() {
            if constexpr (W1) {
              frame_select<T, G>(d, tt, zs - 3 + k, o1, s1.cm1);
              const unsigned q = i0 + (unsigned)(k - 2);
              is_acquire_w(q);
              write_own<T, G>(is_of(q), o1);
              is_publish(q);
              if constexpr (tb_own<T>()) {
#pragma unroll
                for (int r = 0; r < G::R; r++)
#pragma unroll
                  for (int i = 0; i < G::V; i++) (tb_s1first<T>() ? own_next : own)[r][i] = o1[r][i];
              }
            }
#pragma unroll
            for (int r = 0; r < G::R; r++)
#pragma unroll
              for (int i = 0; i < G::V; i++) s1.cm1[r][i] = c1[r][i];
          };
          if constexpr (tb_s1first<T>()) {
            // stage 1 first: it needs only the input plane (in flight for several ticks), and the
            // IS plane stage 2 then reads was published one tick earlier by every warp, so no
            // warp waits on another's just-finished work within a tick
            if constexpr (A1) {
              mbar_wait(fullb(kk), (kk / B::NS) & 1u);
              stage1();
              release(kk);
              stage1_out();
            }
            if constexpr (A2) {
              stage2();
              stage2_out();
            }
            if constexpr (A1 && W1 && tb_own<T>()) {
#pragma unroll
              for (int r = 0; r < G::R; r++)
#pragma unroll
                for (int i = 0; i < G::V; i++) own[r][i] = own_next[r][i];
            }
          } else {  // stage 2 and its store, then the input wait and stage 1
            if constexpr (A2) {
              stage2();
              stage2_out();
            }
            if constexpr (A1) {
              mbar_wait(fullb(kk), (kk / B::NS) & 1u);
              stage1();
              release(kk);
              stage1_out();
            }
          }
        };
        using Y = std::true_type;
        using N = std::false_type;
        // ticks 0..4 (pipeline fill), 5..zc+3 (steady state), zc+4 (drain): K = zc + 5 ticks
        tick(0, Y{}, N{}, N{}, N{});
        tick(1, Y{}, N{}, N{}, N{});
        tick(2, Y{}, N{}, N{}, Y{});
        tick(3, Y{}, Y{}, N{}, Y{});
        tick(4, Y{}, Y{}, N{}, Y{});
        for (int k = 5; k < zc + 4; k++) tick(k, Y{}, Y{}, Y{}, Y{});
        tick(zc + 4, N{}, Y{}, Y{}, N{});
        if constexpr (tb_direct2<S>()) {  // IS planes ze-1, ze: read (as o, o+1) but never as o-1
          is_done_r(i0 + (unsigned)zc);
          is_done_r(i0 + (unsigned)zc + 1);
        }
        continue;
      }
      // ------------------------------------------------------------------------------ halo warps
      if (nst == 1) {
        for (int k = 0; k < nin; k++) {
          const unsigned kk = k0 + (unsigned)k;
          mbar_wait(fullb(kk), (kk / B::NS) & 1u);
          release(kk);
        }
        continue;
      }
      int ioff[B::HC], soff[B::HC];
      unsigned hmask = 0, fmask = 0;  // bit j: cell j exists / is an x-y frame cell (or outside)
      const int hl = (warp - B::NWARP) * 32 + lane;
#pragma unroll
      for (int j = 0; j < B::HC; j++) {
        const int cc = hl + j * 32 * B::NHW;
        int hx, hy;
        if (cc < B::TX + 2) { hx = cc - 1; hy = -1; }
        else if (cc < 2 * (B::TX + 2)) { hx = cc - (B::TX + 2) - 1; hy = B::TY; }
        else if (cc < 2 * (B::TX + 2) + B::TY) { hx = -1; hy = cc - 2 * (B::TX + 2); }
        else { hx = B::TX; hy = cc - 2 * (B::TX + 2) - B::TY; }
        ioff[j] = (hy + 2) * B::P + B::PAD + hx;
        soff[j] = (hy + 1) * B::P + B::PAD + hx;
        hmask |= (unsigned)(cc < B::RING) << j;
        const int gx = x0 + hx, gy = y0 + hy;
        fmask |= (unsigned)!(gx >= 1 && gx <= d.nx - 2 && gy >= 1 && gy <= d.ny - 2) << j;
      }
      StreamState<T, G11> hs[B::HC];
#pragma unroll
      for (int j = 0; j < B::HC; j++) hs[j].zero();
      const int K = zc + 5;
      for (int k = 0; k < K; k++) {
        if (k < zc + 4) {
          const unsigned kk = k0 + (unsigned)k;
          mbar_wait(fullb(kk), (kk / B::NS) & 1u);
          const T *sl = in_slot(kk);
          T ho[B::HC], hc[B::HC];
#pragma unroll
          for (int j = 0; j < B::HC; j++) {
            if ((hmask >> j) & 1u) {
              T nb[3][3];
#pragma unroll
              for (int dy = 0; dy < 3; dy++)
#pragma unroll
                for (int dx = 0; dx < 3; dx++) nb[dy][dx] = sl[ioff[j] + (dy - 1) * B::P + dx - 1];
              arrival_cell<T, S>(hs[j], nb, c, ho[j], hc[j]);
            } else {
              ho[j] = hc[j] = T(0);
            }
          }
          release(kk);
          if (k >= 2) {
            const int o = zs - 3 + k;
            const bool zint = o >= d.zlo && o <= d.zhi;
            const unsigned q = i0 + (unsigned)(k - 2);
            is_acquire_w(q);
            T *is = is_of(q);
#pragma unroll
            for (int j = 0; j < B::HC; j++)
              if ((hmask >> j) & 1u) is[soff[j]] = (zint && !((fmask >> j) & 1u)) ? ho[j] : hs[j].cm1[0][0];
            is_publish(q);
          }
#pragma unroll
          for (int j = 0; j < B::HC; j++) hs[j].cm1[0][0] = hc[j];
        }
      }
    }
    if (ps + 1 < npass) grid_barrier(bar, (unsigned)(ps + 1));
  }
}

namespace {
template <typename T> void *tb_kernel(int shape) {
  return shape == SHAPE_3D7    ? (void *)tb3d_kernel<T, SHAPE_3D7, false>
         : shape == SHAPE_3D19 ? (void *)tb3d_kernel<T, SHAPE_3D19, false>
                               : (void *)tb3d_kernel<T, SHAPE_3D27, false>;
}
struct TbInfo {
  int TX, TY, NT, P, RI;
  size_t smem;
};
template <typename T, int S> TbInfo tb_info_s() {
  using B = TbG<T, S>;
  return TbInfo{B::TX, B::TY, B::NTHR, B::P, B::RI, B::SMEM};
}
template <typename T> TbInfo tb_info(int shape) {
  return shape == SHAPE_3D7 ? tb_info_s<T, SHAPE_3D7>() : shape == SHAPE_3D19 ? tb_info_s<T, SHAPE_3D19>()
                                                                              : tb_info_s<T, SHAPE_3D27>();
}
}  // namespace

Plan plan_tb3d(const Problem &p) {
  Plan pl;
  pl.variant = PERKS_PERKS;
  if (p.ndim != 3 || (p.shape != SHAPE_3D7 && p.shape != SHAPE_3D27 && p.shape != SHAPE_3D19) ||
      p.bc != PERKS_BC_FRAME || (p.nranks > 1 && (p.shape != SHAPE_3D7 || p.nz < 2))) {
    pl.why = "tb3d: needs 3D 7pt/19pt/27pt FRAME (multi-GPU slabs: 7pt, >= 2 planes)";
    return pl;
  }
  if (!use_tma3(p)) { pl.why = "tb3d: needs TMA (nx*S % 16 == 0)"; return pl; }
  const bool f32 = p.dtype == PERKS_F32;
  const TbInfo ti = f32 ? tb_info<float>(p.shape) : tb_info<double>(p.shape);
  const int TX = ti.TX, TY = ti.TY, NT = ti.NT;
  const size_t smem = ti.smem;
  void *k = f32 ? tb_kernel<float>(p.shape) : tb_kernel<double>(p.shape);
  if (p.nranks > 1)  // the slab kernel (7-point star, checked above)
    k = f32 ? (void *)tb3d_kernel<float, SHAPE_3D7, true> : (void *)tb3d_kernel<double, SHAPE_3D7, true>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    pl.why = "tb3d: cudaFuncSetAttribute";
    return pl;
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { cudaGetLastError(); pl.why = "cudaFuncGetAttributes"; return pl; }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem);
  if (occ < 1) { pl.why = "tb3d: not resident"; return pl; }
  occ = 1;  // one CTA per SM (launch bounds)
  const int tx = (int)((p.nx + TX - 1) / TX), ty = (int)((p.ny + TY - 1) / TY);
  const int64_t tiles = (int64_t)tx * ty;
  const int64_t resident = (int64_t)occ * p.num_sms;
  // z chunks: minimise the busiest CTA's ticks per pass, ceil(units / grid) * (chunk + 5)
  int nzc = 1;
  int64_t best = -1;
  for (int n = 1; n <= std::max<int64_t>(1, p.nz / 4); n++) {
    const int64_t zcn = (p.nz + n - 1) / n, nn = (p.nz + zcn - 1) / zcn;
    if (nn != n) continue;
    const int64_t un = tiles * n, g = std::min<int64_t>(un, resident);
    const int64_t cost = ((un + g - 1) / g) * (zcn + 5);
    if (best < 0 || cost < best) { best = cost; nzc = n; }
  }
  if (env_int("PERKS_TB_NZC", 0) > 0) nzc = std::min<int>(env_int("PERKS_TB_NZC", 0), (int)p.nz);
  const int zc = (int)((p.nz + nzc - 1) / nzc);
  nzc = (int)((p.nz + zc - 1) / zc);
  pl.units = tiles * nzc;
  pl.zchunk = zc;
  pl.grid = (int)std::min<int64_t>(pl.units, resident);
  // balanced contiguous runs instead (TbUnits.range, opt-in PERKS_TB_RANGE=1 or -1 = by tick count):
  // a run of ceil(W/G) planes touches at most ceil(len/nz)+1 tiles, each costing a 5-tick pipeline
  // fill.  Measured slower than the strided units despite fewer ticks (C3 30.96 vs 30.45, C5 1739 vs
  // 1626 us/step, profiles/r02_tb3d_range.txt): concurrently running CTAs then sit at unrelated z, so
  // the tiles' overlapping halo rows no longer meet in L2.
  {
    const int64_t W = tiles * p.nz, G = std::min<int64_t>(resident, std::max<int64_t>(1, W / 8));
    const int64_t len = (W + G - 1) / G, fills = std::min<int64_t>(tiles, (len + p.nz - 1) / p.nz + 1);
    const int64_t ticks_range = len + 5 * fills, ticks_units = best;
    const int force = env_int("PERKS_TB_RANGE", 0);
    if (force == 1 || (force < 0 && ticks_range < ticks_units)) {
      pl.cfg = 2;  // (range mode)
      pl.grid = (int)G;
      pl.units = G;
      pl.zchunk = (int)std::min<int64_t>(len, p.nz);
    }
  }
  pl.block = NT;
  pl.ctas_per_sm = occ;
  pl.tile[0] = TX; pl.tile[1] = TY; pl.tile[2] = zc;
  pl.regs = fa.numRegs;
  pl.smem = (int)smem;
  if (pl.cfg != 2) pl.cfg = 1;
  pl.family = 7;  // (3D PERKS, two time steps per pass)
  const double S = (double)p.elem();
  pl.cached_smem = 0;  // level t+1 is on chip only while its planes are in flight (no resident cells)
  pl.dram_bytes_step = S * (double)p.cells();  // 2·S·cells per pass of two steps
  // halo through L2 per step: the input box beyond the tile, once per two steps
  const int RI = ti.RI, PB = ti.P;
  pl.halo_bytes_step = 0.5 * S * (double)(RI * PB - TX * TY) * (double)tiles * (double)(p.nz + 4 * nzc);
  pl.ws_bytes = align256((size_t)p.cells() * p.elem()) + 256;
  snprintf(pl.name, sizeof(pl.name), "perks3d_tb2_%s_%s_t%dx%d_z%d",
           p.shape == SHAPE_3D7 ? "7pt" : p.shape == SHAPE_3D19 ? "19pt" : "27pt", f32 ? "f32" : "f64", TX, TY, zc);
  pl.ok = true;
  return pl;
}

namespace {
// Multi-GPU prologue of a run: the input's two bottom / top planes into the neighbours' ghosts as
// exchange 0 (parity tbx); blockIdx.y = side (0: planes 0, 1 to the lower neighbour's side 1;
// 1: planes nz-2, nz-1 to the upper neighbour's side 0), blockIdx.z = plane j, 8 rows per CTA.  Before
// writing, wait until every exchange of the previous run from that neighbour arrived (it produced
// its last one after reading ours: no write-after-read across runs).
template <typename T>
__global__ void __launch_bounds__(256) tb_dist_prologue_kernel(const T *__restrict__ in, DistK dk, int nx, int ny,
                                                               int nz, unsigned long long xbase,
                                                               unsigned long long tbx) {
  const int side = blockIdx.y, j = blockIdx.z;
  if (side == 0 ? !dk.has_lo : !dk.has_hi) return;
  const unsigned long long plane = (unsigned long long)nx * ny;
  if (threadIdx.x == 0) wait_counter_sys(dk.ctr + side, xbase * plane);
  __syncthreads();
  const int y0 = blockIdx.x * 8, y1 = min(y0 + 8, ny);
  const int zsrc = side == 0 ? j : nz - 2 + j;
  const T *srcp = in + (size_t)zsrc * plane + (size_t)y0 * nx;
  T *dstp = reinterpret_cast<T *>(side == 0 ? dk.send_lo : dk.send_hi) +
            (size_t)tb_ghost_plane(tbx, side == 0 ? 1 : 0, j) * plane + (size_t)y0 * nx;
  const int n16 = (int)((size_t)(y1 - y0) * nx * sizeof(T) / 16);  // nx*S % 16 == 0 (TMA)
  const uint4 *s4 = reinterpret_cast<const uint4 *>(srcp);
  uint4 *d4 = reinterpret_cast<uint4 *>(dstp);
  for (int i = threadIdx.x; i < n16; i += blockDim.x) d4[i] = s4[i];
  signal_counter_sys(side == 0 ? dk.peer_ctr_lo : dk.peer_ctr_hi, (unsigned long long)(y1 - y0) * nx);
}

template <typename T, int S, class B>
cudaError_t launch_tb_g(const Problem &p, const Plan &pl, const T *in, T *out, void *ws, int64_t steps,
                        cudaStream_t s, const DistRun *dr) {
  Coef<T, Shape<S>::N> c;
  for (int i = 0; i < Shape<S>::N; i++) c.w[i] = sizeof(T) == 4 ? (T)p.wf[i] : (T)p.wd[i];
  const bool dist = dr != nullptr && p.nranks > 1;
  // slab faces with a neighbour are interior (reading R12); so are the neighbours' planes -1 / nz,
  // whose level t+1 this kernel computes redundantly from the two-deep ghosts
  Dom3 d{(int)p.nx, (int)p.ny, (int)p.nz, (dist && p.rank > 0) ? -1 : 1,
         (dist && p.rank < p.nranks - 1) ? (int)p.nz : (int)p.nz - 2};
  TbUnits u{(int)((p.nx + B::TX - 1) / B::TX), (int)((p.ny + B::TY - 1) / B::TY), 0, pl.zchunk,
            env_int("PERKS_ZIGZAG", 1), pl.cfg == 2 ? 1 : 0};
  u.nzc = (int)((p.nz + u.zc - 1) / u.zc);
  char *w = (char *)ws;
  T *tmp = (T *)w;
  unsigned *bar = (unsigned *)(w + align256((size_t)p.cells() * p.elem()));
  TbMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  const void *b[3] = {in, out, tmp};
  // 64-byte L2 promotion: a box's two-cell x halo then costs one 64-B granule per row edge instead
  // of a 256-B block (C5: DRAM reads 1.40 -> 1.12 x S·cells per step, profiles/r02_tb3d_l2promo.txt)
  const int promo = env_int("PERKS_TMA_L2PROMO", 64);
  for (int i = 0; i < 3; i++)
    if (!encode_map3(&maps.m[i], p, b[i], B::P, B::RI, promo)) return cudaErrorInvalidValue;
  DistK dk = make_distk(dist ? dr : nullptr);
  unsigned long long xbase = dist ? dr->xbase : 0, tbx = dist ? dr->tbx : 0;
  if (dist) {
    Problem g = p;
    g.nz = 12;  // G[12][ny][nx]
    if (!encode_map3(&maps.ghost, g, dr->ghost, B::P, B::RI, promo)) return cudaErrorInvalidValue;
  }
  cudaError_t e = reset_grid_barrier(bar, s);
  if (e != cudaSuccess) return e;
  if (dist) {
    tb_dist_prologue_kernel<T><<<dim3((unsigned)((p.ny + 7) / 8), 2, 2), 256, 0, s>>>(
        in, dk, (int)p.nx, (int)p.ny, (int)p.nz, xbase, tbx);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  void *k = (void *)tb3d_kernel<T, S, false>;
  if constexpr (S == SHAPE_3D7) {  // (slabs: the 7-point star only)
    if (dist) k = (void *)tb3d_kernel<T, S, true>;
  }
  void *args[] = {(void *)&in,  (void *)&out,   (void *)&tmp,  (void *)&maps, (void *)&d,
                  (void *)&u,   (void *)&steps, (void *)&bar,  (void *)&c,    (void *)&dk,
                  (void *)&xbase, (void *)&tbx};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(pl.block);
  cfg.dynamicSmemBytes = (size_t)pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = (dist && dr->noncoop) ? 0 : 1;  // (several slabs resident on one device: run_group)
  return cudaLaunchKernelExC(&cfg, k, args);
}

template <typename T, int S>
cudaError_t launch_tb(const Problem &p, const Plan &pl, const T *in, T *out, void *ws, int64_t steps,
                      cudaStream_t s, const DistRun *dr) {
  if constexpr (S != SHAPE_3D7) {
    if (dr != nullptr && p.nranks > 1) return cudaErrorNotSupported;
  }
  return launch_tb_g<T, S, TbG<T, S>>(p, pl, in, out, ws, steps, s, dr);
}
}  // namespace

cudaError_t run_tb3d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws, int64_t steps,
                     cudaStream_t s, const DistRun *dr) {
  if (p.dtype == PERKS_F32)
    return p.shape == SHAPE_3D7    ? launch_tb<float, SHAPE_3D7>(p, pl, (const float *)in, (float *)out, ws, steps, s, dr)
           : p.shape == SHAPE_3D19 ? launch_tb<float, SHAPE_3D19>(p, pl, (const float *)in, (float *)out, ws, steps, s, dr)
                                   : launch_tb<float, SHAPE_3D27>(p, pl, (const float *)in, (float *)out, ws, steps, s, dr);
  return p.shape == SHAPE_3D7    ? launch_tb<double, SHAPE_3D7>(p, pl, (const double *)in, (double *)out, ws, steps, s, dr)
         : p.shape == SHAPE_3D19 ? launch_tb<double, SHAPE_3D19>(p, pl, (const double *)in, (double *)out, ws, steps, s, dr)
                                 : launch_tb<double, SHAPE_3D27>(p, pl, (const double *)in, (double *)out, ws, steps, s, dr);
}

}  // namespace perks
