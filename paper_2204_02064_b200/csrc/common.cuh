// common.cuh — device helpers shared by every kernel of the PERKS stencil library (sm_100a).
// Product code: nothing here is shared with oracle/ (the CPU oracle is independent C).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#ifndef PERKS_DEVINL
#define PERKS_DEVINL __device__ __forceinline__
#endif

namespace perks {

// --------------------------------------------------------------------- arithmetic
// Reading R5: first term one rounded multiply, later terms one fused multiply-add each.
// The _rn intrinsics pin the rounding (no contraction/reassociation by the compiler).
PERKS_DEVINL float mul_rn(float a, float b) { return __fmul_rn(a, b); }
PERKS_DEVINL double mul_rn(double a, double b) { return __dmul_rn(a, b); }
PERKS_DEVINL float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
PERKS_DEVINL double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

// Packed FP32 pairs (sm_100a FFMA2 / FMUL2, PTX fma.rn.f32x2 / mul.rn.f32x2): two cells of one
// chain term in one instruction, each lane rounded exactly as fma_rn / mul_rn (so the results stay
// bit-identical to the scalar chain, reading R5).  B200 runs FFMA2 at the same FMA-pipe rate as
// two FFMAs (profiles/r02_ffma2_probe.txt: 127.5 vs 124.4 FMA/clk/SM) but in HALF the issue slots:
// the stencil bodies are issue-bound, so the freed slots go to loads, stores and bookkeeping.
#ifndef PERKS_FFMA2
#define PERKS_FFMA2 1
#endif
// 64-bit register pairs of two fp32 cells.
using f32x2 = unsigned long long;
PERKS_DEVINL f32x2 pack2(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
PERKS_DEVINL void unpack2(f32x2 p, float &a, float &b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(p)); }
// w*a + c per lane (one rounding each); the weight is broadcast to both lanes
PERKS_DEVINL f32x2 fma2_rn(float w, f32x2 a, f32x2 c) {
  f32x2 r;
  asm("{\n.reg .b64 pw;\nmov.b64 pw, {%1, %1};\nfma.rn.f32x2 %0, pw, %2, %3;\n}" : "=l"(r) : "f"(w), "l"(a), "l"(c));
  return r;
}
// (w.lo*a + c.lo, w.hi*a + c.hi): a weight pair times one broadcast cell
PERKS_DEVINL f32x2 fma2_bc_rn(f32x2 w, float a, f32x2 c) {
  f32x2 r;
  asm("{\n.reg .b64 pa;\nmov.b64 pa, {%2, %2};\nfma.rn.f32x2 %0, %1, pa, %3;\n}" : "=l"(r) : "l"(w), "f"(a), "l"(c));
  return r;
}
PERKS_DEVINL f32x2 mul2_rn(float w, f32x2 a) {
  f32x2 r;
  asm("{\n.reg .b64 pw;\nmov.b64 pw, {%1, %1};\nmul.rn.f32x2 %0, pw, %2;\n}" : "=l"(r) : "f"(w), "l"(a));
  return r;
}

// A register copy the compiler cannot see through.  Used when a register-cached value is moved
// into the stencil's sliding window: the cached SSA value then dies at the copy, so ptxas can
// write the new value back into the same physical register instead of keeping a second copy of
// the whole register cache alive ("imperfect register reuse by the compiler").
PERKS_DEVINL float opaque_copy(float v) {
  float r;
  asm volatile("mov.b32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
PERKS_DEVINL double opaque_copy(double v) {
  double r;
  asm volatile("mov.b64 %0, %1;" : "=d"(r) : "d"(v));
  return r;
}

// --------------------------------------------------------------------- warp shuffles
// Neighbour-lane exchange by inline PTX: the compiler cannot prove convergence after the
// mbarrier-wait asm blocks and would guard every __shfl_*_sync with a BRA.DIV fallback; these
// are always called by full, converged warps.
PERKS_DEVINL uint32_t shfl_up1_u32(uint32_t v) {
  uint32_t r;
  asm("shfl.sync.up.b32 %0, %1, 1, 0, -1;\n" : "=r"(r) : "r"(v));
  return r;
}
PERKS_DEVINL uint32_t shfl_down1_u32(uint32_t v) {
  uint32_t r;
  asm("shfl.sync.down.b32 %0, %1, 1, 31, -1;\n" : "=r"(r) : "r"(v));
  return r;
}
PERKS_DEVINL float shfl_up1(float v) { return __uint_as_float(shfl_up1_u32(__float_as_uint(v))); }
PERKS_DEVINL float shfl_down1(float v) { return __uint_as_float(shfl_down1_u32(__float_as_uint(v))); }
PERKS_DEVINL double shfl_up1(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const uint32_t lo = shfl_up1_u32((uint32_t)b), hi = shfl_up1_u32((uint32_t)(b >> 32));
  return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
}
PERKS_DEVINL double shfl_down1(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const uint32_t lo = shfl_down1_u32((uint32_t)b), hi = shfl_down1_u32((uint32_t)(b >> 32));
  return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
}

// --------------------------------------------------------------------- vectors
template <typename T, int V> struct VecT;
template <> struct VecT<float, 1> { using type = float; };
template <> struct VecT<float, 2> { using type = float2; };
template <> struct VecT<float, 4> { using type = float4; };
template <> struct VecT<double, 1> { using type = double; };
template <> struct VecT<double, 2> { using type = double2; };

template <typename T, int V>
PERKS_DEVINL void vload(T (&v)[V], const T *p) {
  if constexpr (V * sizeof(T) > 16) {  // several 16-byte vectors
    constexpr int C = 16 / (int)sizeof(T);
#pragma unroll
    for (int j = 0; j < V / C; j++) {
      T w[C];
      vload<T, C>(w, p + j * C);
#pragma unroll
      for (int i = 0; i < C; i++) v[j * C + i] = w[i];
    }
  } else {
    using VT = typename VecT<T, V>::type;
    VT t = *reinterpret_cast<const VT *>(p);
    const T *s = reinterpret_cast<const T *>(&t);
#pragma unroll
    for (int i = 0; i < V; i++) v[i] = s[i];
  }
}
template <typename T, int V>
PERKS_DEVINL void vstore(T *p, const T (&v)[V]) {
  if constexpr (V * sizeof(T) > 16) {
    constexpr int C = 16 / (int)sizeof(T);
#pragma unroll
    for (int j = 0; j < V / C; j++) {
      T w[C];
#pragma unroll
      for (int i = 0; i < C; i++) w[i] = v[j * C + i];
      vstore<T, C>(p + j * C, w);
    }
  } else {
    using VT = typename VecT<T, V>::type;
    VT t;
    T *d = reinterpret_cast<T *>(&t);
#pragma unroll
    for (int i = 0; i < V; i++) d[i] = v[i];
    *reinterpret_cast<VT *>(p) = t;
  }
}
// L2-only (bypass L1) loads for data produced by other CTAs during the same launch.
template <typename T> PERKS_DEVINL T ld_cg(const T *p) { return __ldcg(p); }
template <typename T> PERKS_DEVINL void st_cg(T *p, T v) { __stcg(p, v); }

// --------------------------------------------------------------------- cp.async
PERKS_DEVINL uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte async copy global->shared, L2 only; src_bytes < 16 zero-fills the rest.
PERKS_DEVINL void cp_async16(void *sdst, const void *gsrc, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sdst)),
               "l"(gsrc), "r"(src_bytes)
               : "memory");
}
PERKS_DEVINL void cp_async8(void *sdst, const void *gsrc, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(sdst)),
               "l"(gsrc), "r"(src_bytes)
               : "memory");
}
PERKS_DEVINL void cp_async4(void *sdst, const void *gsrc, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(sdst)),
               "l"(gsrc), "r"(src_bytes)
               : "memory");
}
template <int BYTES> PERKS_DEVINL void cp_async(void *sdst, const void *gsrc, bool valid) {
  if constexpr (BYTES == 16) cp_async16(sdst, gsrc, valid ? 16 : 0);
  else if constexpr (BYTES == 8) cp_async8(sdst, gsrc, valid ? 8 : 0);
  else cp_async4(sdst, gsrc, valid ? 4 : 0);
}
// Bulk L2 prefetch of [p, p+bytes) (16-byte aligned address and size; sm_90+).
PERKS_DEVINL void prefetch_l2(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
PERKS_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> PERKS_DEVINL void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// --------------------------------------------------------------------- device-wide sync
PERKS_DEVINL unsigned ld_acquire_gpu(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PERKS_DEVINL unsigned ld_relaxed_gpu(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PERKS_DEVINL void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }
PERKS_DEVINL void st_release_gpu(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
PERKS_DEVINL void red_release_gpu(unsigned *p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// ---- tagged ("LL") exchange words: a value and the step tag that produced it travel in ONE
// naturally aligned 8-byte store, so a consumer that reads a matching tag also reads the matching
// value (single-copy atomicity of aligned 8-byte accesses) — no flag, no fence, no membar on the
// critical path of the per-step halo exchange.  fp64 values use two words (one per 32-bit half).
struct LLWord {
  unsigned v, tag;
};
PERKS_DEVINL void st_ll(LLWord *p, unsigned v, unsigned tag) {
  asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};\n" ::"l"(p), "r"(v), "r"(tag) : "memory");
}
PERKS_DEVINL LLWord ld_ll(const LLWord *p) {
  LLWord w;
  asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];\n" : "=r"(w.v), "=r"(w.tag) : "l"(p) : "memory");
  return w;
}
// GPU-scope relaxed variants (exchange between CTAs of one launch on one device): the value/tag
// pair still travels in one single-copy-atomic 8-byte access, without the system-scope ordering
// of volatile accesses (which compile to .STRONG.SYS and serialise in the memory system).
PERKS_DEVINL void st_llg(LLWord *p, unsigned v, unsigned tag) {
  asm volatile("st.relaxed.gpu.global.v2.u32 [%0], {%1, %2};\n" ::"l"(p), "r"(v), "r"(tag) : "memory");
}
PERKS_DEVINL LLWord ld_llg(const LLWord *p) {
  LLWord w;
  asm volatile("ld.relaxed.gpu.global.v2.u32 {%0, %1}, [%2];\n" : "=r"(w.v), "=r"(w.tag) : "l"(p) : "memory");
  return w;
}
template <typename T> struct LLG;
template <> struct LLG<float> {
  static constexpr int WORDS = 1;
  PERKS_DEVINL static void put(LLWord *p, float x, unsigned tag) { st_llg(p, __float_as_uint(x), tag); }
  PERKS_DEVINL static bool get(const LLWord *p, unsigned tag, float &x) {
    LLWord w = ld_llg(p);
    x = __uint_as_float(w.v);
    return w.tag == tag;
  }
};
template <> struct LLG<double> {
  static constexpr int WORDS = 2;
  PERKS_DEVINL static void put(LLWord *p, double x, unsigned tag) {
    const unsigned long long b = __double_as_longlong(x);
    st_llg(p, (unsigned)b, tag);
    st_llg(p + 1, (unsigned)(b >> 32), tag);
  }
  PERKS_DEVINL static bool get(const LLWord *p, unsigned tag, double &x) {
    const LLWord a = ld_llg(p), b = ld_llg(p + 1);
    x = __longlong_as_double((long long)(((unsigned long long)b.v << 32) | a.v));
    return a.tag == tag && b.tag == tag;
  }
};

template <typename T> struct LL;
template <> struct LL<float> {
  static constexpr int WORDS = 1;
  PERKS_DEVINL static void put(LLWord *p, float x, unsigned tag) { st_ll(p, __float_as_uint(x), tag); }
  // returns true when every word carries `tag`
  PERKS_DEVINL static bool get(const LLWord *p, unsigned tag, float &x) {
    LLWord w = ld_ll(p);
    x = __uint_as_float(w.v);
    return w.tag == tag;
  }
};
template <> struct LL<double> {
  static constexpr int WORDS = 2;
  PERKS_DEVINL static void put(LLWord *p, double x, unsigned tag) {
    const unsigned long long b = __double_as_longlong(x);
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "r"((unsigned)b),
                 "r"(tag), "r"((unsigned)(b >> 32)), "r"(tag)
                 : "memory");
  }
  PERKS_DEVINL static bool get(const LLWord *p, unsigned tag, double &x) {
    unsigned lo, t0, hi, t1;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(lo), "=r"(t0), "=r"(hi), "=r"(t1)
                 : "l"(p)
                 : "memory");
    x = __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
    return t0 == tag && t1 == tag;
  }
};

PERKS_DEVINL unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
  return t;
}

#ifndef PERKS_WATCHDOG_NS
#define PERKS_WATCHDOG_NS 10000000000ull  // 10 s: a lost neighbour becomes a trap, not a hang
#endif

// Spin (one thread) until *p >= target, acquiring at system scope.
// Watchdog for device-side spins: after PERKS_WATCHDOG_NS a lost peer/CTA becomes a reported
// trap (the caller's next synchronisation fails with cudaErrorLaunchFailure) instead of a hang.
__device__ __noinline__ inline void watchdog_fire(const char *what, unsigned a, unsigned b) {
  printf("perks watchdog: %s stuck (block %d thread %d, %u %u)\n", what, (int)blockIdx.x, (int)threadIdx.x, a, b);
  __trap();
}

// Grid barrier on a monotonically increasing 32-bit counter ctr[0] (ctr[1] = its value at launch,
// set by reset_grid_barrier).  Barrier n (n = 1, 2, ...) completes when every CTA has arrived n
// times: ctr[0] reaches ctr[1] + n * gridDim.x.  Counter and target wrap modulo 2^32 together and are
// compared wrap-safely (the signed difference): CTAs are at most one barrier apart, so the counter
// never trails the target by 2^31 and any step count (steps is int64) is safe.
// CTA-level __syncthreads + one releasing arrive per CTA + acquiring spin (P:1068 grid.sync).
PERKS_DEVINL bool grid_barrier_pending(const unsigned *ctr, unsigned target) {
  return (int)(ld_acquire_gpu(ctr) - target) < 0;
}
PERKS_DEVINL void grid_barrier(unsigned *ctr, unsigned n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = ld_relaxed_gpu(ctr + 1) + n * gridDim.x;
    red_release_gpu(ctr, 1u);
    if (grid_barrier_pending(ctr, target)) {
      const unsigned long long t0 = globaltimer_ns();
      unsigned k = 0;
      while (grid_barrier_pending(ctr, target))
        if ((++k & 1023u) == 0 && globaltimer_ns() - t0 > PERKS_WATCHDOG_NS)
          watchdog_fire("grid barrier", ld_acquire_gpu(ctr), target);
    }
  }
  __syncthreads();
}

}  // namespace perks
