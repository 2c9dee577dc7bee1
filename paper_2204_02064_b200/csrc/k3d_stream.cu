// k3d_stream.cu — 3D stencil kernels without cross-step caching:
//   (a) host-loop: one launch per step, one (tile, z-chunk) unit per CTA  (Fig. 3 left)
//   (b) persistent: one cooperative launch; CTAs loop over units; grid barrier per step
// Compute body: stream3d.cuh (plane streaming).
#include <algorithm>
#include <cstdio>

#include "internal.h"
#include "stream3d.cuh"

namespace perks {

template <typename T> struct G3Sel;
template <> struct G3Sel<float> { using G = Geo3D<float, 4, 2, 8, 4>; };
template <> struct G3Sel<double> { using G = Geo3D<double, 2, 2, 8, 4>; };

constexpr int K3D_THREADS = 256;
static_assert(G3Sel<float>::G::NT == K3D_THREADS && G3Sel<double>::G::NT == K3D_THREADS, "3D block size");

struct Units3 {
  int tx, ty, nzc, zc;
};

PERKS_DEVINL void unit_coords(const Units3 &u, int id, int tile_x, int tile_y, int &x0, int &y0,
                              int &zs) {
  const int t = id % (u.tx * u.ty);
  const int zc = id / (u.tx * u.ty);
  x0 = (t % u.tx) * tile_x;
  y0 = (t / u.tx) * tile_y;
  zs = zc * u.zc;
}

template <typename T, int S>
__global__ void __launch_bounds__(K3D_THREADS) hostloop3d_kernel(const T *__restrict__ src,
                                                                     T *__restrict__ dst, Dom3 d,
                                                                     Units3 u,
                                                                     Coef<T, Shape<S>::N> c) {
  using G = typename G3Sel<T>::G;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *smem = reinterpret_cast<T *>(smem_raw);
  int x0, y0, zs;
  unit_coords(u, blockIdx.x, G::TX, G::TY, x0, y0, zs);
  const int ze = min(zs + u.zc, d.nz);
  stream_unit<T, S, G>(smem, src, dst, d, x0, y0, zs, ze, c);
}

template <typename T>
PERKS_DEVINL T *step_dst3(T *out, T *tmp, int64_t t, int64_t steps) {
  return ((steps - 1 - t) & 1) == 0 ? out : tmp;
}

template <typename T, int S>
__global__ void __launch_bounds__(K3D_THREADS) persistent3d_kernel(
    const T *__restrict__ in, T *out, T *tmp, Dom3 d, Units3 u, int64_t steps, unsigned *bar,
    Coef<T, Shape<S>::N> c) {
  using G = typename G3Sel<T>::G;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *smem = reinterpret_cast<T *>(smem_raw);
  const int nunits = u.tx * u.ty * u.nzc;
  for (int64_t t = 0; t < steps; t++) {
    const T *src = t == 0 ? in : step_dst3(out, tmp, t - 1, steps);
    T *dst = step_dst3(out, tmp, t, steps);
    for (int id = blockIdx.x; id < nunits; id += gridDim.x) {
      int x0, y0, zs;
      unit_coords(u, id, G::TX, G::TY, x0, y0, zs);
      const int ze = min(zs + u.zc, d.nz);
      __syncthreads();  // slots of the previous unit are free
      stream_unit<T, S, G>(smem, src, dst, d, x0, y0, zs, ze, c);
    }
    if (t + 1 < steps) grid_barrier(bar, (unsigned)((t + 1) * gridDim.x));
  }
}

// ------------------------------------------------------------------ host side
namespace {
template <typename T> void *kptr3(int shape, bool persistent) {
  if (shape == SHAPE_3D7)
    return persistent ? (void *)persistent3d_kernel<T, SHAPE_3D7> : (void *)hostloop3d_kernel<T, SHAPE_3D7>;
  if (shape == SHAPE_3D27)
    return persistent ? (void *)persistent3d_kernel<T, SHAPE_3D27> : (void *)hostloop3d_kernel<T, SHAPE_3D27>;
  return nullptr;
}
void *pick3(const Problem &p, bool persistent) {
  return p.dtype == PERKS_F32 ? kptr3<float>(p.shape, persistent) : kptr3<double>(p.shape, persistent);
}
template <typename T> size_t smem3() { return (size_t)G3Sel<T>::G::NS * G3Sel<T>::G::SLOT_BYTES; }
template <typename T> void geo3(int &tx, int &ty, int &nt) {
  tx = G3Sel<T>::G::TX; ty = G3Sel<T>::G::TY; nt = G3Sel<T>::G::NT;
}
}  // namespace

Plan plan_stream3d(const Problem &p, perks_variant v) {
  Plan pl;
  pl.variant = v;
  if (p.ndim != 3 || (p.shape != SHAPE_3D7 && p.shape != SHAPE_3D27) || p.bc != PERKS_BC_FRAME) {
    pl.why = "stream3d: needs 3D 7pt/27pt FRAME";
    return pl;
  }
  const bool persistent = v == PERKS_PERSISTENT;
  void *k = pick3(p, persistent);
  const size_t smem = p.dtype == PERKS_F32 ? smem3<float>() : smem3<double>();
  int TX, TY, NT;
  if (p.dtype == PERKS_F32) geo3<float>(TX, TY, NT); else geo3<double>(TX, TY, NT);
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    pl.why = "cudaFuncSetAttribute"; return pl;
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem);
  const int tx = (int)((p.nx + TX - 1) / TX), ty = (int)((p.ny + TY - 1) / TY);
  const int resident = std::max(1, occ * p.num_sms);
  // z chunks: about two waves of units for the host loop; exactly one wave for the persistent
  // kernel (one unit per CTA per step, so no CTA idles at the tail)
  const int tiles = tx * ty;
  int nzc = persistent ? std::max(1, resident / tiles) : std::max(1, (2 * resident + tiles - 1) / tiles);
  nzc = std::min<int>(nzc, (int)std::max<int64_t>(1, p.nz / 8));
  const int zc = (int)((p.nz + nzc - 1) / nzc);
  nzc = (int)((p.nz + zc - 1) / zc);
  pl.units = (int64_t)tiles * nzc;
  pl.zchunk = zc;
  pl.block = NT;
  pl.tile[0] = TX; pl.tile[1] = TY; pl.tile[2] = zc;
  pl.regs = fa.numRegs;
  pl.smem = (int)smem;
  pl.ctas_per_sm = occ;
  pl.grid = persistent ? (int)std::min<int64_t>(pl.units, resident) : (int)pl.units;
  const double S = (double)p.elem();
  pl.dram_bytes_step = 2.0 * S * (double)p.cells();
  pl.halo_bytes_step = S * (double)p.nz * (2.0 * TX * ty * tx + 2.0 * TY * ty * tx) +
                       S * 2.0 * nzc * (double)p.nx * p.ny;
  pl.ws_bytes = align256((size_t)p.cells() * p.elem()) + (persistent ? 256 : 0);
  snprintf(pl.name, sizeof(pl.name), "%s3d_%s_%s_t%dx%d_z%d", persistent ? "persistent" : "hostloop",
           p.shape == SHAPE_3D7 ? "7pt" : "27pt", p.dtype == PERKS_F32 ? "f32" : "f64", TX, TY, zc);
  pl.ok = true;
  return pl;
}

template <typename T, int S>
static cudaError_t launch3d(const Problem &p, const Plan &pl, const T *in, T *out, T *tmp,
                            unsigned *bar, int64_t steps, cudaStream_t s) {
  using G = typename G3Sel<T>::G;
  Coef<T, Shape<S>::N> c;
  for (int i = 0; i < Shape<S>::N; i++) c.w[i] = sizeof(T) == 4 ? (T)p.wf[i] : (T)p.wd[i];
  Dom3 d{(int)p.nx, (int)p.ny, (int)p.nz};
  Units3 u{(int)((p.nx + G::TX - 1) / G::TX), (int)((p.ny + G::TY - 1) / G::TY), 0, pl.zchunk};
  u.nzc = (int)((p.nz + u.zc - 1) / u.zc);
  const size_t smem = (size_t)G::NS * G::SLOT_BYTES;
  if (pl.variant == PERKS_HOSTLOOP) {
    void *k = (void *)hostloop3d_kernel<T, S>;
    for (int64_t t = 0; t < steps; t++) {
      const T *src = t == 0 ? in : ((((steps - t) & 1) == 0) ? out : tmp);
      T *dst = (((steps - 1 - t) & 1) == 0) ? out : tmp;
      void *args[] = {(void *)&src, (void *)&dst, (void *)&d, (void *)&u, (void *)&c};
      cudaError_t e = cudaLaunchKernel(k, dim3(pl.grid), dim3(G::NT), args, smem, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  void *k = (void *)persistent3d_kernel<T, S>;
  cudaError_t e = cudaMemsetAsync(bar, 0, 256, s);
  if (e != cudaSuccess) return e;
  void *args[] = {(void *)&in, (void *)&out, (void *)&tmp, (void *)&d, (void *)&u, (void *)&steps,
                  (void *)&bar, (void *)&c};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(G::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, k, args);
}

cudaError_t run_stream3d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws,
                         int64_t steps, cudaStream_t s) {
  char *w = (char *)ws;
  unsigned *bar = (unsigned *)(w + align256((size_t)p.cells() * p.elem()));
  if (p.dtype == PERKS_F32) {
    if (p.shape == SHAPE_3D7)
      return launch3d<float, SHAPE_3D7>(p, pl, (const float *)in, (float *)out, (float *)w, bar, steps, s);
    return launch3d<float, SHAPE_3D27>(p, pl, (const float *)in, (float *)out, (float *)w, bar, steps, s);
  }
  if (p.shape == SHAPE_3D7)
    return launch3d<double, SHAPE_3D7>(p, pl, (const double *)in, (double *)out, (double *)w, bar, steps, s);
  return launch3d<double, SHAPE_3D27>(p, pl, (const double *)in, (double *)out, (double *)w, bar, steps, s);
}

}  // namespace perks
