// k2d_cluster.cu — variant (c) PERKS for SMALL 2D domains: the whole domain lives in the
// registers of ONE thread-block cluster (up to 16 CTAs on 16 SMs) for all T steps.
//
// Small domains are latency bound, not bandwidth bound: the host loop pays a
// launch gap per step and a 148-CTA grid barrier costs ~1.2 us, while the domain (C1: 128 KiB)
// fits on a few SMs.  So this kernel keeps the time loop inside one cluster launch (Fig. 3 right,
// P:288) and replaces grid.sync by the cluster hardware barrier
// (barrier.cluster.arrive.release / wait.acquire, ~0.2 us).  Every cell is cached in registers
// (reg_cache, Fig. 6; "cache inter-step data in registers"): warp w of CTA c
// owns R consecutive rows, each lane V consecutive x cells; one warp spans the whole x extent, so
// x-neighbours come from warp shuffles only.  The rows above/below a warp's segment are the halo
// (P:348): the producing warp PUSHES its edge row into the consumer's shared-memory halo buffer —
// a local st.shared for a warp of the same CTA, a distributed-shared-memory st.shared::cluster
// for the neighbouring CTA — so every halo read is a local shared-memory load.
//
// One cluster barrier per step suffices: halo buffers are double-buffered by step parity, and the
// barrier is split-phase — a warp computes its two edge rows first, pushes them, arrives, then
// computes its inner rows (registers only) while the other CTAs catch up, then waits.
//
// The compute body is the canonical FMA chain (reading R5), so results are bit-identical to the
// other variants and the oracle.
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "internal.h"
#include "shapes.cuh"

namespace perks {

PERKS_DEVINL unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
PERKS_DEVINL unsigned cluster_nctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
  return r;
}
PERKS_DEVINL void cluster_arrive_release() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
PERKS_DEVINL void cluster_wait_acquire() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
PERKS_DEVINL void cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory"); }
PERKS_DEVINL void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory"); }
// Shared-memory address of `local_addr` in the CTA of cluster rank `rank`.
PERKS_DEVINL uint32_t map_rank(uint32_t local_addr, unsigned rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
PERKS_DEVINL void st_cluster(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;\n" ::"r"(addr), "f"(v) : "memory");
}
PERKS_DEVINL void st_cluster(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}

constexpr int KC_R = 4;  // rows per warp

// Shared memory: halo[par][warp][side][32*V]; side 0 = row above the warp's segment, 1 = below.
template <typename T, int S, int V, int WY>
__global__ void __launch_bounds__(32 * WY, 1) perks2d_cluster_kernel(const T *__restrict__ in,
                                                                 T *__restrict__ out, int nx, int ny,
                                                                 int64_t steps, Coef<T, Shape<S>::N> c) {
  constexpr int R = KC_R, W = 32 * V;
  constexpr bool BOX = has_corners<S>();
  __shared__ __align__(16) T halo[2][WY][2][W];
  const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
  const unsigned rank = cluster_ctarank(), ncta = cluster_nctarank();
  const int y0 = ((int)rank * WY + wy) * R;  // first row of this warp
  const int x = lane * V;

  // Every CTA of the cluster must have started before anyone writes its shared memory (DSMEM):
  // arrive now, wait just before the first push, so the barrier overlaps the prologue loads.
  cluster_arrive_relaxed();

  // ---- prologue: the whole domain into registers (one-time load half of 2·D_cache)
  T cur[R][V];
#pragma unroll
  for (int r = 0; r < R; r++)
#pragma unroll
    for (int i = 0; i < V; i++) {
      const int y = y0 + r, xx = x + i;
      cur[r][i] = (y < ny && xx < nx) ? in[(size_t)y * nx + xx] : T(0);
    }
  // frame predicates (reading R1)
  unsigned rowint = 0, colint = 0;
#pragma unroll
  for (int r = 0; r < R; r++) rowint |= (y0 + r >= 1 && y0 + r <= ny - 2) ? 1u << r : 0u;
#pragma unroll
  for (int i = 0; i < V; i++) colint |= (x + i >= 1 && x + i <= nx - 2) ? 1u << i : 0u;

  // push targets of my top row (-> the warp above, its "below" halo) and bottom row (-> the warp
  // below, its "above" halo); at the cluster's ends there is no consumer (frame rows)
  const bool has_up = wy > 0 || rank > 0;
  const bool has_dn = wy < WY - 1 || rank + 1 < ncta;
  const unsigned up_rank = wy > 0 ? rank : rank - 1, dn_rank = wy < WY - 1 ? rank : rank + 1;
  const int up_w = wy > 0 ? wy - 1 : WY - 1, dn_w = wy < WY - 1 ? wy + 1 : 0;
  const uint32_t up_base = map_rank(smem_u32(&halo[0][up_w][1][x]), has_up ? up_rank : rank);
  const uint32_t dn_base = map_rank(smem_u32(&halo[0][dn_w][0][x]), has_dn ? dn_rank : rank);
  constexpr uint32_t PAR_BYTES = (uint32_t)(WY * 2 * W * sizeof(T));
  auto push = [&](int pb, const T (&top)[V], const T (&bot)[V]) {
#pragma unroll
    for (int i = 0; i < V; i++) {
      if (has_up) st_cluster(up_base + pb * PAR_BYTES + i * (uint32_t)sizeof(T), top[i]);
      if (has_dn) st_cluster(dn_base + pb * PAR_BYTES + i * (uint32_t)sizeof(T), bot[i]);
    }
  };
  cluster_wait();  // all CTAs of the cluster are running (their halo buffers exist)
  push(0, cur[0], cur[R - 1]);
  cluster_arrive_release();
  cluster_wait_acquire();

  // neighbourhood of one row: w[0] = x-1, w[1..V] = own cells, w[V+1] = x+V
  auto widen = [&](T (&w)[V + 2], const T (&v)[V]) {
    const T l = __shfl_up_sync(0xffffffffu, v[V - 1], 1);
    const T rr = __shfl_down_sync(0xffffffffu, v[0], 1);
    w[0] = lane == 0 ? T(0) : l;         // x = -1 does not exist (x = 0 is frame)
    w[V + 1] = lane == 31 ? T(0) : rr;   // x = W is outside the domain
#pragma unroll
    for (int i = 0; i < V; i++) w[i + 1] = v[i];
  };
  auto load_halo = [&](T (&w)[V + 2], const T *h) {
    T v[V];
#pragma unroll
    for (int i = 0; i < V; i++) v[i] = h[x + i];
    widen(w, v);
  };
  // new value of row r from rows (a: r-1, b: r, d: r+1), frame-selected
  auto row_update = [&](int r, const T (&a)[V + 2], const T (&b)[V + 2], const T (&d)[V + 2], T (&nv)[V]) {
#pragma unroll
    for (int i = 0; i < V; i++) {
      T acc;
#pragma unroll
      for (int p = 0; p < Shape<S>::N; p++) {
        const int dy = Shape<S>::dy(p), dx = Shape<S>::dx(p);
        const T val = dy < 0 ? a[i + 1 + dx] : (dy > 0 ? d[i + 1 + dx] : b[i + 1 + dx]);
        acc = (p == 0) ? mul_rn(c.w[0], val) : fma_rn(c.w[p], val, acc);
      }
      nv[i] = (((rowint >> r) & (colint >> i)) & 1u) ? acc : b[i + 1];
    }
  };
  (void)BOX;

  for (int64_t t = 0; t < steps; t++) {
    const int par = (int)(t & 1);
    T nv[R][V];
    {
      // edge rows first (they read the halo written before the last barrier)
      T wa[V + 2], wb[V + 2], wd[V + 2];
      load_halo(wa, halo[par][wy][0]);
      widen(wb, cur[0]);
      if constexpr (R > 1) widen(wd, cur[1]); else load_halo(wd, halo[par][wy][1]);
      row_update(0, wa, wb, wd, nv[0]);
      if constexpr (R > 1) {
        widen(wa, cur[R - 2]);
        widen(wb, cur[R - 1]);
        load_halo(wd, halo[par][wy][1]);
        row_update(R - 1, wa, wb, wd, nv[R - 1]);
      }
    }
    push(par ^ 1, nv[0], nv[R - 1]);
    cluster_arrive_release();
    // inner rows: registers only, overlapping the barrier
#pragma unroll
    for (int r = 1; r < R - 1; r++) {
      T wa[V + 2], wb[V + 2], wd[V + 2];
      widen(wa, cur[r - 1]);
      widen(wb, cur[r]);
      widen(wd, cur[r + 1]);
      row_update(r, wa, wb, wd, nv[r]);
    }
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
      for (int i = 0; i < V; i++) cur[r][i] = nv[r][i];
    cluster_wait_acquire();
  }

  // ---- epilogue: registers to `out` (store half of 2·D_cache)
#pragma unroll
  for (int r = 0; r < R; r++)
#pragma unroll
    for (int i = 0; i < V; i++) {
      const int y = y0 + r, xx = x + i;
      if (y < ny && xx < nx) out[(size_t)y * nx + xx] = cur[r][i];
    }
}

// ------------------------------------------------------------------ host side
namespace {
constexpr int KC_MAX_CLUSTER = 16;

template <typename T, int S, int V> void *kc_ptr(int wy) {
  if (wy == 1) return (void *)perks2d_cluster_kernel<T, S, V, 1>;
  if (wy == 2) return (void *)perks2d_cluster_kernel<T, S, V, 2>;
  if (wy == 4) return (void *)perks2d_cluster_kernel<T, S, V, 4>;
  return (void *)perks2d_cluster_kernel<T, S, V, 8>;
}
template <typename T, int S> void *kc_ptr_v(int v, int wy) {
  if (v == 2) return kc_ptr<T, S, 2>(wy);
  if constexpr (sizeof(T) == 4) {
    if (v == 8) return kc_ptr<T, S, 8>(wy);
  }
  return kc_ptr<T, S, 4>(wy);  // f64 is capped at V = 4 (register budget)
}
void *kc_kernel(const Problem &p, int v, int wy) {
  if (p.dtype == PERKS_F32)
    return p.shape == SHAPE_2D5 ? kc_ptr_v<float, SHAPE_2D5>(v, wy) : kc_ptr_v<float, SHAPE_2D9>(v, wy);
  return p.shape == SHAPE_2D5 ? kc_ptr_v<double, SHAPE_2D5>(v, wy) : kc_ptr_v<double, SHAPE_2D9>(v, wy);
}
}  // namespace

// Plan the cluster kernel: returns !ok if the domain does not fit one cluster's registers.
Plan plan_perks2d_cluster(const Problem &p) {
  Plan pl;
  pl.variant = PERKS_PERKS;
  if (p.ndim != 2 || (p.shape != SHAPE_2D5 && p.shape != SHAPE_2D9) || p.bc != PERKS_BC_FRAME) {
    pl.why = "perks2d_cluster: needs 2D 5pt/9pt FRAME";
    return pl;
  }
  if (env_int("PERKS_NO_CLUSTER", 0)) { pl.why = "disabled"; return pl; }
  // lane width V: smallest of {2,4,8} with 32*V >= nx (f64 capped at 4: register budget)
  const int vmax = p.dtype == PERKS_F64 ? 4 : 8;
  int v = 2;
  while (v < vmax && 32 * v < p.nx) v *= 2;
  if (32 * v < p.nx) { pl.why = "perks2d_cluster: nx too wide"; return pl; }
  // warps per CTA: smallest WY whose cluster (<= 16 CTAs) covers ny
  int wy = -1, csize = 0;
  const int force_wy = env_int("PERKS_KC_WY", 0);  // sweeps only
  for (int w : {1, 2, 4, 8}) {
    if (force_wy && w != force_wy) continue;
    const int64_t rows = (int64_t)w * KC_R;
    const int64_t cs = (p.ny + rows - 1) / rows;
    if (cs <= KC_MAX_CLUSTER) { wy = w; csize = (int)cs; break; }
  }
  if (wy < 0) { pl.why = "perks2d_cluster: ny too tall"; return pl; }
  void *k = kc_kernel(p, v, wy);
  if (csize > 8 && cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    pl.why = "perks2d_cluster: non-portable cluster size refused";
    return pl;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize);
  cfg.blockDim = dim3(32 * wy);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, k, &cfg) != cudaSuccess || nclusters < 1) {
    cudaGetLastError();
    pl.why = "perks2d_cluster: cluster not schedulable";
    return pl;
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  pl.cfg = (v << 8) | wy;
  pl.grid = csize;
  pl.block = 32 * wy;
  pl.ctas_per_sm = 1;
  pl.tile[0] = 32 * v; pl.tile[1] = wy * KC_R; pl.tile[2] = 1;
  pl.regs = fa.numRegs;
  pl.smem = (int)fa.sharedSizeBytes;
  pl.units = csize;
  pl.cached_reg = (int64_t)csize * wy * KC_R * 32 * v;
  pl.cached_smem = 0;
  pl.dram_bytes_step = 0.0;  // resident: only the one-time 2·D_cache term
  pl.halo_bytes_step = (double)p.elem() * 2.0 * (csize - 1) * (double)p.nx;  // DSMEM, not L2
  pl.ws_bytes = 0;
  snprintf(pl.name, sizeof(pl.name), "perks2d_cluster_%s_%s_v%d_w%d_c%d", p.shape == SHAPE_2D5 ? "5pt" : "9pt",
           p.dtype == PERKS_F32 ? "f32" : "f64", v, wy, csize);
  pl.ok = true;
  return pl;
}

template <typename T, int S>
static cudaError_t launch_kc(const Problem &p, const Plan &pl, const T *in, T *out, int64_t steps,
                             cudaStream_t s) {
  Coef<T, Shape<S>::N> c;
  for (int i = 0; i < Shape<S>::N; i++) c.w[i] = sizeof(T) == 4 ? (T)p.wf[i] : (T)p.wd[i];
  const int v = pl.cfg >> 8, wy = pl.cfg & 0xff;
  void *k = kc_kernel(p, v, wy);
  int nx = (int)p.nx, ny = (int)p.ny;
  void *args[] = {(void *)&in, (void *)&out, (void *)&nx, (void *)&ny, (void *)&steps, (void *)&c};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(pl.block);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = pl.grid;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, k, args);
}

cudaError_t run_perks2d_cluster(const Problem &p, const Plan &pl, const void *in, void *out,
                                int64_t steps, cudaStream_t s) {
  if (p.dtype == PERKS_F32) {
    if (p.shape == SHAPE_2D5) return launch_kc<float, SHAPE_2D5>(p, pl, (const float *)in, (float *)out, steps, s);
    return launch_kc<float, SHAPE_2D9>(p, pl, (const float *)in, (float *)out, steps, s);
  }
  if (p.shape == SHAPE_2D5) return launch_kc<double, SHAPE_2D5>(p, pl, (const double *)in, (double *)out, steps, s);
  return launch_kc<double, SHAPE_2D9>(p, pl, (const double *)in, (double *)out, steps, s);
}

}  // namespace perks
