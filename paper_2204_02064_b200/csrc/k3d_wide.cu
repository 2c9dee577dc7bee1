// k3d_wide.cu — host-loop (a), persistent (b) and PERKS (c) for GENERAL 3D point sets: any list of
// <= 64 offsets of radius <= 3, in any order (Table II 3d13pt, the radius-2 star, runs
// with a compile-time point set).  The FMA chain follows the list order (reading R5), so results
// are bit-identical to the oracle and across variants.
//
// One CTA computes a 32 x 8 x 8 output block from a shared-memory copy of the block plus its r-wide
// halo shell (loaded from L2/HBM each step); 256 threads sweep the block x-fastest.  A double-buffered cp.async
// variant of the persistent kernel was measured slower (3d13pt f64 256^3: 231.9 vs 200.8 us/step —
// it halves occupancy).  (c) runs the
// persistent kernel with an empty on-chip cache split — the 3D policy of k3d_stream.cu, measured
// there: on B200 the 126 MB L2 serves what an on-chip plane cache would.
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "internal.h"

namespace perks {

constexpr int KW3_THREADS = 256, KW3_TX = 32, KW3_TY = 8, KW3_TZ = 8, KW3_MAXR = 3;

template <typename T> struct WideCoef3 {
  int n;
  int8_t dx[kMaxPoints2D], dy[kMaxPoints2D], dz[kMaxPoints2D];
  T w[kMaxPoints2D];
};

// Compile-time point sets: PS 1 = 3d13pt (the radius-2 star: centre + two points per half-axis),
// (dz,dy,dx) lexicographic.  PS 0 = any other list.
template <int PS> struct WideSet3;
template <> struct WideSet3<1> {
  static constexpr int R = 2, N = 13;
  // (dz, dy, dx) of point p, lexicographic
  static constexpr __host__ __device__ int dz(int p) { return p < 2 ? p - 2 : p < 11 ? 0 : p - 10; }
  static constexpr __host__ __device__ int dy(int p) { return p < 2 || p >= 11 ? 0 : p < 4 ? p - 4 : p < 9 ? 0 : p - 8; }
  static constexpr __host__ __device__ int dx(int p) { return p >= 4 && p < 9 ? p - 6 : 0; }
};

template <typename T, int PS>
__device__ __forceinline__ T cell3(const T *s, int PX, int PXY, int r, int lx, int ly, int lz, int x, int y, int z,
                                   int nx, int ny, int nz, const WideCoef3<T> &c) {
  if constexpr (PS == 0) {
    const T *ctr = s + (size_t)(lz + r) * PXY + (ly + r) * PX + (lx + r);
    if (x < r || x >= nx - r || y < r || y >= ny - r || z < r || z >= nz - r) return *ctr;
    T acc = mul_rn(c.w[0], ctr[c.dz[0] * PXY + c.dy[0] * PX + c.dx[0]]);
    for (int p = 1; p < c.n; p++) acc = fma_rn(c.w[p], ctr[c.dz[p] * PXY + c.dy[p] * PX + c.dx[p]], acc);
    return acc;
  } else {
    using WS = WideSet3<PS>;
    constexpr int R = WS::R, QX = KW3_TX + 2 * R, QXY = QX * (KW3_TY + 2 * R);
    const T *ctr = s + (lz + R) * QXY + (ly + R) * QX + (lx + R);
    if (x < R || x >= nx - R || y < R || y >= ny - R || z < R || z >= nz - R) return *ctr;
    T acc = mul_rn(c.w[0], ctr[WS::dz(0) * QXY + WS::dy(0) * QX + WS::dx(0)]);
#pragma unroll
    for (int p = 1; p < WS::N; p++) acc = fma_rn(c.w[p], ctr[WS::dz(p) * QXY + WS::dy(p) * QX + WS::dx(p)], acc);
    return acc;
  }
}

// One block of one step: src -> shared memory (zero outside the domain) -> dst.
template <typename T, int PS>
__device__ void block3(const T *__restrict__ src, T *__restrict__ dst, int nx, int ny, int nz, int bx, int by,
                       int bz, int r, const WideCoef3<T> &c, T *s) {
  const int PX = KW3_TX + 2 * r, PY = KW3_TY + 2 * r, PZ = KW3_TZ + 2 * r, PXY = PX * PY;
  const int x0 = bx * KW3_TX, y0 = by * KW3_TY, z0 = bz * KW3_TZ;
  for (int i = threadIdx.x; i < PXY * PZ; i += blockDim.x) {
    const int lz = i / PXY, rem = i % PXY, ly = rem / PX, lx = rem % PX;
    const int x = x0 - r + lx, y = y0 - r + ly, z = z0 - r + lz;
    s[i] = (x >= 0 && x < nx && y >= 0 && y < ny && z >= 0 && z < nz)
               ? __ldcg(src + ((size_t)z * ny + y) * nx + x) : T(0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < KW3_TX * KW3_TY * KW3_TZ; i += blockDim.x) {
    const int lz = i / (KW3_TX * KW3_TY), rem = i % (KW3_TX * KW3_TY), ly = rem / KW3_TX, lx = rem % KW3_TX;
    const int x = x0 + lx, y = y0 + ly, z = z0 + lz;
    if (x < nx && y < ny && z < nz)
      dst[((size_t)z * ny + y) * nx + x] = cell3<T, PS>(s, PX, PXY, r, lx, ly, lz, x, y, z, nx, ny, nz, c);
  }
  __syncthreads();
}

struct Blocks3 {
  int bx, by, bz;
};

template <typename T, int PS>
__global__ void __launch_bounds__(KW3_THREADS) wide3_hostloop_kernel(const T *__restrict__ src, T *__restrict__ dst,
                                                                     int nx, int ny, int nz, Blocks3 b, int r,
                                                                     const __grid_constant__ WideCoef3<T> c) {
  extern __shared__ __align__(16) unsigned char kw3_smem[];
  const int id = blockIdx.x;
  block3<T, PS>(src, dst, nx, ny, nz, id % b.bx, (id / b.bx) % b.by, id / (b.bx * b.by), r, c,
                reinterpret_cast<T *>(kw3_smem));
}

template <typename T, int PS>
__global__ void __launch_bounds__(KW3_THREADS) wide3_persistent_kernel(const T *__restrict__ in, T *out, T *tmp,
                                                                       int nx, int ny, int nz, Blocks3 b, int r,
                                                                       int64_t steps, unsigned *bar,
                                                                       const __grid_constant__ WideCoef3<T> c) {
  extern __shared__ __align__(16) unsigned char kw3_smem[];
  const int nb = b.bx * b.by * b.bz;
  for (int64_t t = 0; t < steps; t++) {
    const T *src = t == 0 ? in : ((((steps - t) & 1) == 0) ? out : tmp);
    T *dst = (((steps - 1 - t) & 1) == 0) ? out : tmp;
    for (int id = blockIdx.x; id < nb; id += gridDim.x)
      block3<T, PS>(src, dst, nx, ny, nz, id % b.bx, (id / b.bx) % b.by, id / (b.bx * b.by), r, c,
                    reinterpret_cast<T *>(kw3_smem));
    if (t + 1 < steps) grid_barrier(bar, (unsigned)((t + 1) * gridDim.x));
  }
}

// ------------------------------------------------------------------ host side
namespace {
int radius3d(const Problem &p) {
  int r = 0;
  for (int i = 0; i < p.npts; i++)
    r = std::max(r, std::max(std::abs(p.off[i][0]), std::max(std::abs(p.off[i][1]), std::abs(p.off3z[i]))));
  return r;
}
int wide3_preset(const Problem &p) {
  if (p.npts != WideSet3<1>::N) return 0;
  for (int q = 0; q < WideSet3<1>::N; q++)
    if (p.off[q][0] != WideSet3<1>::dx(q) || p.off[q][1] != WideSet3<1>::dy(q) || p.off3z[q] != WideSet3<1>::dz(q))
      return 0;
  return 1;
}
template <typename T> WideCoef3<T> make_coef3(const Problem &p) {
  WideCoef3<T> c{};
  c.n = p.npts;
  for (int i = 0; i < p.npts; i++) {
    c.dx[i] = (int8_t)p.off[i][0];
    c.dy[i] = (int8_t)p.off[i][1];
    c.dz[i] = (int8_t)p.off3z[i];
    c.w[i] = sizeof(T) == 4 ? (T)p.wf[i] : (T)p.wd[i];
  }
  return c;
}
template <typename T> void *wk3(bool hostloop, int ps) {
  if (hostloop) return ps == 1 ? (void *)wide3_hostloop_kernel<T, 1> : (void *)wide3_hostloop_kernel<T, 0>;
  return ps == 1 ? (void *)wide3_persistent_kernel<T, 1> : (void *)wide3_persistent_kernel<T, 0>;
}
size_t smem3(int r, size_t S) {
  return (size_t)(KW3_TX + 2 * r) * (KW3_TY + 2 * r) * (KW3_TZ + 2 * r) * S;
}
}  // namespace

Plan plan_wide3d(const Problem &p, perks_variant v) {
  Plan pl;
  pl.variant = v;
  const int r = radius3d(p);
  if (p.ndim != 3 || p.shape != SHAPE_G3D || p.bc != PERKS_BC_FRAME || r > KW3_MAXR) {
    pl.why = "wide3d: 3D FRAME point sets of radius <= 3";
    return pl;
  }
  const bool f32 = p.dtype == PERKS_F32, hostloop = v == PERKS_HOSTLOOP;
  const int ps = wide3_preset(p);
  void *k = f32 ? wk3<float>(hostloop, ps) : wk3<double>(hostloop, ps);
  const size_t smem = smem3(r, p.elem());
  if (smem > (size_t)p.max_smem_optin) { pl.why = "wide3d: block does not fit shared memory"; return pl; }
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    pl.why = "cudaFuncSetAttribute";
    return pl;
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, KW3_THREADS, smem);
  if (occ < 1) { pl.why = "wide3d: not resident"; return pl; }
  const int bx = (int)((p.nx + KW3_TX - 1) / KW3_TX), by = (int)((p.ny + KW3_TY - 1) / KW3_TY),
            bz = (int)((p.nz + KW3_TZ - 1) / KW3_TZ);
  const int64_t blocks = (int64_t)bx * by * bz;
  pl.units = blocks;
  pl.grid = hostloop ? (int)blocks : (int)std::min<int64_t>(blocks, (int64_t)occ * p.num_sms);
  pl.block = KW3_THREADS;
  pl.ctas_per_sm = occ;
  pl.tile[0] = KW3_TX; pl.tile[1] = KW3_TY; pl.tile[2] = KW3_TZ;
  pl.regs = fa.numRegs;
  pl.smem = (int)smem;
  pl.cfg = ps;
  pl.family = 5;  // (wide 3D)
  const double S = (double)p.elem();
  pl.dram_bytes_step = 2.0 * S * (double)p.cells();
  pl.halo_bytes_step = S * (double)blocks *
                       ((double)smem3(r, 1) - (double)KW3_TX * KW3_TY * KW3_TZ);
  pl.ws_bytes = align256((size_t)p.cells() * p.elem()) + (hostloop ? 0 : 256);
  snprintf(pl.name, sizeof(pl.name), "%s3d_wide_r%d_%dpt%s_%s%s", v == PERKS_PERKS ? "perks" : hostloop ? "hostloop" : "persistent",
           r, p.npts, ps ? "" : "_any", f32 ? "f32" : "f64", v == PERKS_PERKS ? "_c0" : "");
  pl.ok = true;
  return pl;
}

namespace {
template <typename T>
cudaError_t run_wide3_t(const Problem &p, const Plan &pl, const T *in, T *out, void *ws, int64_t steps,
                        cudaStream_t s) {
  const WideCoef3<T> c = make_coef3<T>(p);
  int r = radius3d(p);
  int nx = (int)p.nx, ny = (int)p.ny, nz = (int)p.nz;
  Blocks3 b{(nx + KW3_TX - 1) / KW3_TX, (ny + KW3_TY - 1) / KW3_TY, (nz + KW3_TZ - 1) / KW3_TZ};
  T *tmp = (T *)ws;
  void *k = wk3<T>(pl.variant == PERKS_HOSTLOOP, pl.cfg);
  if (pl.variant == PERKS_HOSTLOOP) {
    for (int64_t t = 0; t < steps; t++) {
      const T *src = t == 0 ? in : ((((steps - t) & 1) == 0) ? out : tmp);
      T *dst = (((steps - 1 - t) & 1) == 0) ? out : tmp;
      void *args[] = {(void *)&src, (void *)&dst, (void *)&nx, (void *)&ny, (void *)&nz, (void *)&b, (void *)&r,
                      (void *)&c};
      cudaError_t e = cudaLaunchKernel(k, dim3(pl.grid), dim3(KW3_THREADS), args, pl.smem, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  unsigned *bar = (unsigned *)((char *)ws + align256((size_t)p.cells() * p.elem()));
  cudaError_t e = cudaMemsetAsync(bar, 0, 256, s);
  if (e != cudaSuccess) return e;
  void *args[] = {(void *)&in, (void *)&out, (void *)&tmp, (void *)&nx, (void *)&ny, (void *)&nz, (void *)&b,
                  (void *)&r, (void *)&steps, (void *)&bar, (void *)&c};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(KW3_THREADS);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, k, args);
}
}  // namespace

cudaError_t run_wide3d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws, int64_t steps,
                       cudaStream_t s) {
  if (p.dtype == PERKS_F32) return run_wide3_t<float>(p, pl, (const float *)in, (float *)out, ws, steps, s);
  return run_wide3_t<double>(p, pl, (const double *)in, (double *)out, ws, steps, s);
}

}  // namespace perks
