// tmem.cuh — Tensor Memory (TMEM) as a third on-chip cache tier for PERKS (sm_100a).
//
// PERKS caches as much of the domain on chip as the SM's storage allows (registers + shared
// memory) and predicts that larger on-chip capacity raises the cached fraction
// and with it the speedup ([draft] P:395-404).  An sm_100a SM has a third
// store the paper's GPUs lack: 256 KiB of Tensor Memory (128 lanes x 512 columns x 32 bit), unused
// by a stencil (no step of the path is a contraction).  Here it holds whole tile planes of the 3D
// PERKS kernel across time steps:
//
//   * warp w of a CTA may only touch TMEM lanes 32*(w%4) .. 32*(w%4)+31 (tcgen05 lane quarters);
//     thread (lane, w) keeps ITS OWN cells of a cached plane (V x R values = WPT 32-bit words) in
//     lane 32*(w%4)+lane, columns  plane*CPP + (w/4)*WPT .. +WPT  (CPP = WPT * ceil(NWARP/4)).
//   * write-back of a cached output plane: tcgen05.st of the thread's cells (no inter-warp hazard:
//     every thread owns its columns);
//   * use in the next step: the thread's cells are tcgen05.ld'ed and written into a ring slot of
//     shared memory one arrival ahead (the stencil needs neighbouring warps' rows), while the
//     producer warp fills the slot's one-cell halo ring from global memory as for the shared-memory
//     cache tier.
// Allocation: one warp, power-of-two columns >= 32, at most 512 per SM over all co-resident CTAs
// (the planner makes every co-resident CTA take 512 / CTAs-per-SM, so alloc never blocks); every
// CTA relinquishes its allocation permit right away (tmem_relinquish).
#pragma once
#include "common.cuh"

namespace perks {

PERKS_DEVINL void tmem_alloc(uint32_t *smem_dst, uint32_t ncols) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
}
// Give up this CTA's right to allocate.  The block scheduler places a further CTA of a kernel that
// contains tcgen05.alloc on an SM only after the resident one relinquished its permit (measured:
// a persistent PERKS grid of 2 CTAs/SM whose CTAs never relinquish gets 1 CTA/SM resident and
// deadlocks in its first grid barrier), so EVERY CTA calls this first, allocating or not.
PERKS_DEVINL void tmem_relinquish() {  // whole warp
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
PERKS_DEVINL void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // whole warp (the allocating one)
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}
PERKS_DEVINL void tmem_fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
PERKS_DEVINL void tmem_fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
PERKS_DEVINL void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
PERKS_DEVINL void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n"); }

// 8 consecutive columns of this thread's lane (32x32b shape: thread i <-> lane base + i).  TMEM is
// invisible to the compiler's memory model: no "memory" clobber (asm volatile keeps the order of
// the tcgen05 statements among themselves; the loaded registers are tied to the wait).
PERKS_DEVINL void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
PERKS_DEVINL void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

// 4 consecutive columns of this thread's lane (32x32b.x4)
PERKS_DEVINL void tmem_st4(uint32_t taddr, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr), "r"(r0), "r"(r1),
               "r"(r2), "r"(r3));
}
PERKS_DEVINL void tmem_ld4_wait(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]));
}
// One row segment of this thread (V values, 16 or 32 bytes) in V*sizeof(T)/4 consecutive TMEM
// columns of its lane.
template <typename T, int V> PERKS_DEVINL void tmem_st_row(uint32_t taddr, const T (&v)[V]) {
  constexpr int WPR = V * (int)sizeof(T) / 4;
  static_assert(WPR == 4 || WPR == 8, "16- or 32-byte segments");
  uint32_t w[WPR];
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < V; i++) w[i] = __float_as_uint((float)v[i]);
  } else {
#pragma unroll
    for (int i = 0; i < V; i++) {
      const unsigned long long b = (unsigned long long)__double_as_longlong((double)v[i]);
      w[2 * i] = (uint32_t)b;
      w[2 * i + 1] = (uint32_t)(b >> 32);
    }
  }
#pragma unroll
  for (int g = 0; g < WPR / 4; g++) tmem_st4(taddr + 4 * g, w[4 * g], w[4 * g + 1], w[4 * g + 2], w[4 * g + 3]);
}
template <typename T, int V> PERKS_DEVINL void tmem_ld_row(uint32_t taddr, T (&v)[V]) {
  constexpr int WPR = V * (int)sizeof(T) / 4;
  static_assert(WPR == 4 || WPR == 8, "16- or 32-byte segments");
  uint32_t w[WPR];
#pragma unroll
  for (int g = 0; g < WPR / 4; g++) {
    uint32_t c[4];
    tmem_ld4_wait(taddr + 4 * g, c);
#pragma unroll
    for (int j = 0; j < 4; j++) w[4 * g + j] = c[j];
  }
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < V; i++) v[i] = (T)__uint_as_float(w[i]);
  } else {
#pragma unroll
    for (int i = 0; i < V; i++)
      v[i] = (T)__longlong_as_double((long long)((unsigned long long)w[2 * i] | ((unsigned long long)w[2 * i + 1] << 32)));
  }
}

// A row segment load split in two: issue (tcgen05.ld, no wait) and take (tcgen05.wait::ld with the
// in-flight words as in/out operands, so nothing reads them earlier), so one row's load latency
// overlaps the previous row's arithmetic.  At most one issued row may be outstanding (the wait
// covers every earlier load of the thread).
template <typename T, int V> struct TmemRowInFlight {
  static constexpr int WPR = V * (int)sizeof(T) / 4;
  static_assert(WPR == 4 || WPR == 8, "16- or 32-byte segments");
  uint32_t w[WPR];
  PERKS_DEVINL void issue(uint32_t taddr) {
#pragma unroll
    for (int g = 0; g < WPR / 4; g++)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                   : "=r"(w[4 * g]), "=r"(w[4 * g + 1]), "=r"(w[4 * g + 2]), "=r"(w[4 * g + 3])
                   : "r"(taddr + 4 * g));
  }
  PERKS_DEVINL void take(T (&v)[V]) {
    if constexpr (WPR == 4) {
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]));
    } else {
      asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                   : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]), "+r"(w[7]));
    }
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int i = 0; i < V; i++) v[i] = (T)__uint_as_float(w[i]);
    } else {
#pragma unroll
      for (int i = 0; i < V; i++)
        v[i] = (T)__longlong_as_double((long long)((unsigned long long)w[2 * i] | ((unsigned long long)w[2 * i + 1] << 32)));
    }
  }
};

// tcgen05.wait::ld with the loaded registers as in/out operands (the load's destination registers
// are undefined until the wait completes).
PERKS_DEVINL void tmem_wait_ld_dep(uint32_t (&r)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]));
}

// Words of a V x R cell block (V * sizeof(T) == 16 bytes per row).
template <typename T, int R, int V> struct TmemCells {
  static constexpr int WPT = R * V * (int)sizeof(T) / 4;
  static_assert(WPT % 8 == 0, "TMEM tier moves 8-column groups");
  PERKS_DEVINL static void pack(const T (&v)[R][V], uint32_t (&w)[WPT]) {
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
      for (int i = 0; i < V; i++) {
        if constexpr (sizeof(T) == 4) {
          w[r * V + i] = __float_as_uint((float)v[r][i]);
        } else {
          const unsigned long long b = (unsigned long long)__double_as_longlong((double)v[r][i]);
          w[2 * (r * V + i)] = (uint32_t)b;
          w[2 * (r * V + i) + 1] = (uint32_t)(b >> 32);
        }
      }
  }
  PERKS_DEVINL static void unpack(const uint32_t (&w)[WPT], T (&v)[R][V]) {
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
      for (int i = 0; i < V; i++) {
        if constexpr (sizeof(T) == 4) {
          v[r][i] = (T)__uint_as_float(w[r * V + i]);
        } else {
          const unsigned long long b =
              (unsigned long long)w[2 * (r * V + i)] | ((unsigned long long)w[2 * (r * V + i) + 1] << 32);
          v[r][i] = (T)__longlong_as_double((long long)b);
        }
      }
  }
  // store / load this thread's cells of the plane whose columns start at `taddr` (warp-uniform)
  PERKS_DEVINL static void store(uint32_t taddr, const T (&v)[R][V]) {
    uint32_t w[WPT];
    pack(v, w);
#pragma unroll
    for (int g = 0; g < WPT / 8; g++) {
      uint32_t c[8];
#pragma unroll
      for (int j = 0; j < 8; j++) c[j] = w[g * 8 + j];
      tmem_st8(taddr + 8 * g, c);
    }
    tmem_wait_st();
  }
  PERKS_DEVINL static void load(uint32_t taddr, T (&v)[R][V]) {
    uint32_t w[WPT];
#pragma unroll
    for (int g = 0; g < WPT / 8; g++) {
      uint32_t c[8];
      tmem_ld8(taddr + 8 * g, c);
      tmem_wait_ld_dep(c);  // ties the registers to the wait: no use can be hoisted above it
#pragma unroll
      for (int j = 0; j < 8; j++) w[g * 8 + j] = c[j];
    }
    unpack(w, v);
  }
};

}  // namespace perks
