// dist.cuh — device side of the multi-GPU slab exchange (P:324 suggests running the
// boundary with communication overlapped with a PERKS interior).
//
// Each rank owns a z-slab.  Library-owned ghost planes G[4][ny][nx] (index = parity*2 + side; side 0
// holds plane -1 from the lower neighbour, side 1 plane nz from the upper neighbour) and two u64
// arrival counters C[2] (0: cells received from the lower neighbour, 1: from the upper) live on
// every rank.  Exchange e carries the neighbour's plane of x^{xbase... } and lands in parity e & 1.
// A producer CTA stores its tile of the face plane straight into the neighbour's ghost plane
// (NVLink P2P when the neighbour is another GPU), fences at system scope and adds the number of
// cells it wrote to the neighbour's counter with a system-scope release.  A consumer waits (system
// scope acquire) until its counter reaches (e + 1) * nx * ny, i.e. every cell of exchange e arrived.
// Counting cells instead of messages makes producer and consumer tilings independent.
#pragma once
#include "common.cuh"

namespace perks {

// Per-launch view of the exchange (plain POD, passed by value).  All zero = single GPU.
struct DistK {
  const unsigned long long *ctr;                 // local counters [2]
  unsigned long long *peer_ctr_lo, *peer_ctr_hi; // lower neighbour's C[1], upper neighbour's C[0]
  void *send_lo, *send_hi;                       // lower / upper neighbour's ghost base G
  int has_lo, has_hi;
};

PERKS_DEVINL unsigned long long ld_acquire_sys_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
PERKS_DEVINL void red_release_sys_add_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
PERKS_DEVINL void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }
PERKS_DEVINL void wait_counter_sys(const unsigned long long *p, unsigned long long target) {
  if (ld_acquire_sys_u64(p) >= target) return;
  const unsigned long long t0 = globaltimer_ns();
  unsigned n = 0;
  while (ld_acquire_sys_u64(p) < target) {
    if ((++n & 255u) == 0 && globaltimer_ns() - t0 > PERKS_WATCHDOG_NS) __trap();
  }
}

// Called by ALL threads of the CTA after they stored their part of a face plane into a neighbour's
// ghost plane: make the stores visible system wide, then one releasing add of `cells`.
PERKS_DEVINL void signal_counter_sys(unsigned long long *peer_ctr, unsigned long long cells) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) red_release_sys_add_u64(peer_ctr, cells);
}

}  // namespace perks
