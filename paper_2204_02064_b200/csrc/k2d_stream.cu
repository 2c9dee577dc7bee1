// k2d_stream.cu — 2D stencil step kernels without on-chip caching across steps:
//   (a) host-loop: one launch per time step (Fig. 3 left);
//   (b) persistent: the time loop inside one cooperative launch with a grid barrier between
//       steps (Fig. 3 right; grid.sync P:1068) — no caching, so every step still
//       reads and writes the whole domain through L2/HBM.
// Both use the same compute body (the paper keeps "the compute portion" unchanged):
// one warp owns a strip of 32*V consecutive x cells and RW rows.  It loads RW+2 rows (one halo
// row above and below) as 128-bit vectors, gets x-neighbours with warp shuffles (lanes 0/31
// load the strip's halo columns), and applies the canonical FMA chain (reading R5).
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "internal.h"
#include "shapes.cuh"

namespace perks {

template <typename T, int S, int V, int RW>
PERKS_DEVINL void strip2d(const T *__restrict__ src, T *__restrict__ dst, int nx, int ny, int xs,
                          int ys, const Coef<T, Shape<S>::N> &c, int lane) {
  constexpr int NR = RW + 2;
  T v[NR][V];
  T el[NR], er[NR];
  const int x = xs + lane * V;
  const bool xin = x < nx;  // V > 1 requires nx % V == 0 (host guarantees), so all-or-nothing
#pragma unroll
  for (int j = 0; j < NR; j++) {
    const int y = ys - 1 + j;
    const bool yin = (y >= 0) && (y < ny);
    const T *row = src + (size_t)(yin ? y : 0) * nx;
    if (yin && xin) {
      vload<T, V>(v[j], row + x);
    } else {
#pragma unroll
      for (int i = 0; i < V; i++) v[j][i] = T(0);
    }
    el[j] = (lane == 0 && yin && xs >= 1) ? row[xs - 1] : T(0);
    er[j] = (lane == 31 && yin && xs + 32 * V < nx) ? row[xs + 32 * V] : T(0);
  }
  // neighbourhood rows: nb[j][0] = x-1, nb[j][1..V] = own cells, nb[j][V+1] = x+V
  T nb[NR][V + 2];
#pragma unroll
  for (int j = 0; j < NR; j++) {
    T l = __shfl_up_sync(0xffffffffu, v[j][V - 1], 1);
    T r = __shfl_down_sync(0xffffffffu, v[j][0], 1);
    nb[j][0] = lane == 0 ? el[j] : l;
    nb[j][V + 1] = lane == 31 ? er[j] : r;
#pragma unroll
    for (int i = 0; i < V; i++) nb[j][i + 1] = v[j][i];
  }
#pragma unroll
  for (int rr = 0; rr < RW; rr++) {
    const int y = ys + rr;
    if (y >= ny) break;  // warp-uniform
    const bool yint = (y >= 1) && (y <= ny - 2);
    T out[V];
#pragma unroll
    for (int i = 0; i < V; i++) {
      T acc;
#pragma unroll
      for (int p = 0; p < Shape<S>::N; p++) {
        const T val = nb[rr + 1 + Shape<S>::dy(p)][i + 1 + Shape<S>::dx(p)];
        acc = (p == 0) ? mul_rn(c.w[0], val) : fma_rn(c.w[p], val, acc);
      }
      const int xi = x + i;
      const bool inter = yint && xi >= 1 && xi <= nx - 2;
      out[i] = inter ? acc : nb[rr + 1][i + 1];
    }
    if (xin) vstore<T, V>(dst + (size_t)y * nx + x, out);
  }
}

constexpr int K2D_THREADS = 256;
constexpr int K2D_WARPS = K2D_THREADS / 32;

template <typename T, int S, int V, int RW>
__global__ void __launch_bounds__(K2D_THREADS) hostloop2d_kernel(const T *__restrict__ src,
                                                                 T *__restrict__ dst, int nx,
                                                                 int ny, int sx, int nstrips,
                                                                 Coef<T, Shape<S>::N> c) {
  const int w = blockIdx.x * K2D_WARPS + (threadIdx.x >> 5);
  if (w >= nstrips) return;  // whole warp exits together
  const int lane = threadIdx.x & 31;
  strip2d<T, S, V, RW>(src, dst, nx, ny, (w % sx) * 32 * V, (w / sx) * RW, c, lane);
}

// Destination of step t for a run of `steps` steps: the last step lands in `out`.
template <typename T>
PERKS_DEVINL T *step_dst(T *out, T *tmp, int64_t t, int64_t steps) {
  return ((steps - 1 - t) & 1) == 0 ? out : tmp;
}

template <typename T, int S, int V, int RW>
__global__ void __launch_bounds__(K2D_THREADS) persistent2d_kernel(
    const T *__restrict__ in, T *out, T *tmp, int nx, int ny, int sx, int nstrips, int64_t steps,
    unsigned *bar, Coef<T, Shape<S>::N> c) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * K2D_WARPS + (threadIdx.x >> 5);
  const int nw = gridDim.x * K2D_WARPS;
  for (int64_t t = 0; t < steps; t++) {
    const T *src = t == 0 ? in : step_dst(out, tmp, t - 1, steps);
    T *dst = step_dst(out, tmp, t, steps);
    for (int s = gw; s < nstrips; s += nw)
      strip2d<T, S, V, RW>(src, dst, nx, ny, (s % sx) * 32 * V, (s / sx) * RW, c, lane);
    if (t + 1 < steps) grid_barrier(bar, (unsigned)(t + 1));
  }
}

// ------------------------------------------------------------------ host side

namespace {
constexpr int RW2D = 8;

template <typename T, int S, int V>
void *kernel_ptr(bool persistent) {
  return persistent ? (void *)persistent2d_kernel<T, S, V, RW2D>
                    : (void *)hostloop2d_kernel<T, S, V, RW2D>;
}

void *pick_kernel(const Problem &p, int V, bool persistent) {
  // instantiate: f32 V in {4,1}, f64 V in {2,1}, shapes 2d5pt / 2d9pt
#define PK(T, S, VV) \
  if (V == VV) return kernel_ptr<T, S, VV>(persistent);
  if (p.dtype == PERKS_F32) {
    if (p.shape == SHAPE_2D5) { PK(float, SHAPE_2D5, 4) PK(float, SHAPE_2D5, 1) }
    if (p.shape == SHAPE_2D9) { PK(float, SHAPE_2D9, 4) PK(float, SHAPE_2D9, 1) }
  } else {
    if (p.shape == SHAPE_2D5) { PK(double, SHAPE_2D5, 2) PK(double, SHAPE_2D5, 1) }
    if (p.shape == SHAPE_2D9) { PK(double, SHAPE_2D9, 2) PK(double, SHAPE_2D9, 1) }
  }
#undef PK
  return nullptr;
}

int vec_width(const Problem &p) {
  const int vmax = p.dtype == PERKS_F32 ? 4 : 2;
  return (p.nx % vmax == 0) ? vmax : 1;
}
}  // namespace

Plan plan_stream2d(const Problem &p, perks_variant v) {
  Plan pl;
  pl.variant = v;
  if (p.ndim != 2 || (p.shape != SHAPE_2D5 && p.shape != SHAPE_2D9) || p.bc != PERKS_BC_FRAME) {
    pl.why = "stream2d: needs 2D 5pt/9pt FRAME";
    return pl;
  }
  const bool persistent = v == PERKS_PERSISTENT;
  const int V = vec_width(p);
  void *k = pick_kernel(p, V, persistent);
  if (!k) { pl.why = "stream2d: no instantiation"; return pl; }
  const int sx = (int)((p.nx + 32 * V - 1) / (32 * V));
  const int sy = (int)((p.ny + RW2D - 1) / RW2D);
  pl.units = (int64_t)sx * sy;
  pl.block = K2D_THREADS;
  pl.tile[0] = 32 * V; pl.tile[1] = RW2D; pl.tile[2] = 1;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  pl.regs = fa.numRegs;
  pl.smem = (int)fa.sharedSizeBytes;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, K2D_THREADS, 0);
  pl.ctas_per_sm = occ;
  const int64_t blocks_needed = (pl.units + K2D_WARPS - 1) / K2D_WARPS;
  if (persistent) {
    pl.grid = (int)std::min<int64_t>((int64_t)occ * p.num_sms, blocks_needed);
    if (pl.grid < 1) pl.grid = 1;
  } else {
    pl.grid = (int)blocks_needed;
  }
  const double S = (double)p.elem();
  pl.dram_bytes_step = 2.0 * S * (double)p.cells();
  pl.halo_bytes_step = S * (double)p.nx * 2.0 * sy;  // re-read halo rows (L2)
  pl.ws_bytes = align256((size_t)p.cells() * p.elem()) + (persistent ? 256 : 0);
  snprintf(pl.name, sizeof(pl.name), "%s2d_%s_%s_v%d_rw%d", persistent ? "persistent" : "hostloop",
           p.shape == SHAPE_2D5 ? "5pt" : "9pt", p.dtype == PERKS_F32 ? "f32" : "f64", V, RW2D);
  pl.ok = true;
  return pl;
}

template <typename T, int N>
static Coef<T, N> make_coef(const Problem &p) {
  Coef<T, N> c;
  for (int i = 0; i < N; i++) c.w[i] = sizeof(T) == 4 ? (T)p.wf[i] : (T)p.wd[i];
  return c;
}

template <typename T, int S>
static cudaError_t launch2d(const Problem &p, const Plan &pl, int V, const T *in, T *out, T *tmp,
                            unsigned *bar, int64_t steps, cudaStream_t s) {
  auto c = make_coef<T, Shape<S>::N>(p);
  const int nx = (int)p.nx, ny = (int)p.ny;
  const int sx = (int)((p.nx + 32 * V - 1) / (32 * V));
  const int nstrips = (int)pl.units;
  if (pl.variant == PERKS_HOSTLOOP) {
    void *k = pick_kernel(p, V, false);
    for (int64_t t = 0; t < steps; t++) {
      const T *src = t == 0 ? in : ((((steps - 1 - (t - 1)) & 1) == 0) ? out : tmp);
      T *dst = (((steps - 1 - t) & 1) == 0) ? out : tmp;
      void *args[] = {(void *)&src, (void *)&dst, (void *)&nx, (void *)&ny, (void *)&sx,
                      (void *)&nstrips, (void *)&c};
      cudaError_t e = cudaLaunchKernel(k, dim3(pl.grid), dim3(pl.block), args, 0, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  void *k = pick_kernel(p, V, true);
  cudaError_t e = reset_grid_barrier(bar, s);
  if (e != cudaSuccess) return e;
  void *args[] = {(void *)&in, (void *)&out, (void *)&tmp, (void *)&nx, (void *)&ny, (void *)&sx,
                  (void *)&nstrips, (void *)&steps, (void *)&bar, (void *)&c};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(pl.block);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, k, args);
}

cudaError_t run_stream2d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws,
                         int64_t steps, cudaStream_t s) {
  const int V = vec_width(p);
  char *w = (char *)ws;
  void *tmp = w;
  unsigned *bar = (unsigned *)(w + align256((size_t)p.cells() * p.elem()));
  if (p.dtype == PERKS_F32) {
    if (p.shape == SHAPE_2D5)
      return launch2d<float, SHAPE_2D5>(p, pl, V, (const float *)in, (float *)out, (float *)tmp, bar, steps, s);
    return launch2d<float, SHAPE_2D9>(p, pl, V, (const float *)in, (float *)out, (float *)tmp, bar, steps, s);
  }
  if (p.shape == SHAPE_2D5)
    return launch2d<double, SHAPE_2D5>(p, pl, V, (const double *)in, (double *)out, (double *)tmp, bar, steps, s);
  return launch2d<double, SHAPE_2D9>(p, pl, V, (const double *)in, (double *)out, (double *)tmp, bar, steps, s);
}

}  // namespace perks
