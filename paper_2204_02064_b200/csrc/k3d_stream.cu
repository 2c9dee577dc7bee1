// k3d_stream.cu — 3D stencil kernels without cross-step caching:
//   (a) host-loop: one launch per step, one (tile, z-chunk) unit per CTA  (Fig. 3 left)
//   (b) persistent: one cooperative launch; CTAs loop over units; grid barrier per step
// Compute body and plane loaders: stream3d.cuh (plane streaming; TMA boxes on sm_100a).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "internal.h"
#include "stream3d.cuh"

namespace perks {

#ifndef PERKS_S3D_R
#define PERKS_S3D_R 2
#endif
#ifndef PERKS_S3D_NS
#define PERKS_S3D_NS 4
#endif
template <typename T> struct G3Sel;
template <> struct G3Sel<float> { using G = Geo3D<float, 4, PERKS_S3D_R, 8, PERKS_S3D_NS>; };
template <> struct G3Sel<double> { using G = Geo3D<double, 2, PERKS_S3D_R, 8, PERKS_S3D_NS>; };

constexpr int K3D_THREADS = 256;
static_assert(G3Sel<float>::G::NT == K3D_THREADS && G3Sel<double>::G::NT == K3D_THREADS, "3D block size");

struct Units3 {
  int tx, ty, nzc, zc;
  int rev;  // zig-zag experiment: 1 = reversed unit order (odd steps)
};

PERKS_DEVINL void unit_coords(const Units3 &u, int id, int tile_x, int tile_y, int &x0, int &y0,
                              int &zs) {
  const int t = id % (u.tx * u.ty);
  const int zc = id / (u.tx * u.ty);
  x0 = (t % u.tx) * tile_x;
  y0 = (t / u.tx) * tile_y;
  zs = zc * u.zc;
}

template <class G> PERKS_DEVINL uint64_t *ring_bars(unsigned char *smem) {
  return reinterpret_cast<uint64_t *>(smem + (size_t)G::NS * G::SLOT_BYTES);
}

template <typename T, int S, bool TMA>
__global__ void __launch_bounds__(K3D_THREADS) hostloop3d_kernel(const T *__restrict__ src,
                                                                 const __grid_constant__ Maps3 maps,
                                                                 int src_idx, T *__restrict__ dst,
                                                                 Dom3 d, Units3 u,
                                                                 Coef<T, Shape<S>::N> c) {
  using G = typename G3Sel<T>::G;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Ring<T, G, TMA> ring;
  ring.init(reinterpret_cast<T *>(smem_raw), ring_bars<G>(smem_raw), 0);
  int x0, y0, zs;
  const int nunits = u.tx * u.ty * u.nzc;
  unit_coords(u, u.rev ? nunits - 1 - (int)blockIdx.x : (int)blockIdx.x, G::TX, G::TY, x0, y0, zs);
  const int ze = min(zs + u.zc, d.nz);
  stream_unit<T, S, G, TMA>(ring, src, &maps.box[src_idx], dst, d, x0, y0, zs, ze, c);
}

template <typename T, int S, bool TMA>
__global__ void __launch_bounds__(K3D_THREADS) persistent3d_kernel(
    const T *__restrict__ in, T *out, T *tmp, const __grid_constant__ Maps3 maps, Dom3 d, Units3 u,
    int64_t steps, unsigned *bar, Coef<T, Shape<S>::N> c) {
  using G = typename G3Sel<T>::G;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Ring<T, G, TMA> ring;
  ring.init(reinterpret_cast<T *>(smem_raw), ring_bars<G>(smem_raw), 0);
  const int nunits = u.tx * u.ty * u.nzc;
  for (int64_t t = 0; t < steps; t++) {
    const bool src_out = t > 0 && ((steps - t) & 1) == 0;
    const T *src = t == 0 ? in : (src_out ? out : tmp);
    const int src_idx = t == 0 ? 0 : (src_out ? 1 : 2);
    T *dst = ((steps - 1 - t) & 1) == 0 ? out : tmp;
    for (int id = blockIdx.x; id < nunits; id += gridDim.x) {
      int x0, y0, zs;
      unit_coords(u, (u.rev && (t & 1)) ? nunits - 1 - id : id, G::TX, G::TY, x0, y0, zs);
      const int ze = min(zs + u.zc, d.nz);
      __syncthreads();  // slots of the previous unit are free
      stream_unit<T, S, G, TMA>(ring, src, &maps.box[src_idx], dst, d, x0, y0, zs, ze, c);
    }
    if (t + 1 < steps) grid_barrier(bar, (unsigned)((t + 1) * gridDim.x));
  }
}

// ------------------------------------------------------------------ TMA descriptors (host)
namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;
}  // namespace

bool tma_available() {
  std::call_once(g_encode_once, [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

// 3D map of a dense [nz][ny][nx] buffer with box {bx, by, 1}; OOB cells read as zero.
bool encode_map3(CUtensorMap *m, const Problem &p, const void *base, int bx, int by) {
  if (!tma_available()) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)p.nx, (cuuint64_t)p.ny, (cuuint64_t)p.nz};
  const cuuint64_t strides[2] = {(cuuint64_t)(p.nx * p.elem()), (cuuint64_t)(p.nx * p.ny * p.elem())};
  const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, p.dtype == PERKS_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        3, const_cast<void *>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// TMA needs 16-byte aligned row strides (and 16-byte aligned bases, checked by run()).
bool use_tma3(const Problem &p) {
  return ((p.nx * (int64_t)p.elem()) % 16) == 0 && env_int("PERKS_NO_TMA", 0) == 0 && tma_available();
}

bool make_maps3(const Problem &p, int P, int ROWS, const void *in, const void *out, const void *tmp,
                Maps3 *m) {
  const void *b[3] = {in, out, tmp ? tmp : out};
  for (int i = 0; i < 3; i++) {
    if (!encode_map3(&m->box[i], p, b[i], P, ROWS)) return false;
    if (!encode_map3(&m->row[i], p, b[i], P, 1)) return false;
  }
  return true;
}

// ------------------------------------------------------------------ host side
namespace {
template <typename T> void *kptr3(int shape, bool persistent, bool tma) {
#define K3(S)                                                                                   \
  if (shape == S) {                                                                             \
    if (persistent) return tma ? (void *)persistent3d_kernel<T, S, true> : (void *)persistent3d_kernel<T, S, false>; \
    return tma ? (void *)hostloop3d_kernel<T, S, true> : (void *)hostloop3d_kernel<T, S, false>; \
  }
  K3(SHAPE_3D7)
  K3(SHAPE_3D27)
#undef K3
  return nullptr;
}
void *pick3(const Problem &p, bool persistent) {
  const bool tma = use_tma3(p);
  return p.dtype == PERKS_F32 ? kptr3<float>(p.shape, persistent, tma) : kptr3<double>(p.shape, persistent, tma);
}
template <typename T> size_t smem3() {
  using G = typename G3Sel<T>::G;
  return (size_t)G::NS * G::SLOT_BYTES + (size_t)G::NS * sizeof(uint64_t);
}
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
  pl.cfg = use_tma3(p) ? 1 : 0;
  const double S = (double)p.elem();
  pl.dram_bytes_step = 2.0 * S * (double)p.cells();
  pl.halo_bytes_step = S * (double)p.nz * (2.0 * TX * ty * tx + 2.0 * TY * ty * tx) +
                       S * 2.0 * nzc * (double)p.nx * p.ny;
  pl.ws_bytes = align256((size_t)p.cells() * p.elem()) + (persistent ? 256 : 0);
  snprintf(pl.name, sizeof(pl.name), "%s3d_%s_%s_t%dx%d_z%d%s", persistent ? "persistent" : "hostloop",
           p.shape == SHAPE_3D7 ? "7pt" : "27pt", p.dtype == PERKS_F32 ? "f32" : "f64", TX, TY, zc,
           pl.cfg ? "_tma" : "_cpasync");
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
  Units3 u{(int)((p.nx + G::TX - 1) / G::TX), (int)((p.ny + G::TY - 1) / G::TY), 0, pl.zchunk, 0};
  const int zigzag = env_int("PERKS_ZIGZAG", 0);
  u.nzc = (int)((p.nz + u.zc - 1) / u.zc);
  const size_t smem = (size_t)pl.smem;
  const bool tma = pl.cfg == 1;
  Maps3 maps;
  std::memset(&maps, 0, sizeof(maps));
  if (tma && !make_maps3(p, G::P, G::ROWS, in, out, tmp, &maps)) return cudaErrorInvalidValue;
  if (pl.variant == PERKS_HOSTLOOP) {
    void *k = tma ? (void *)hostloop3d_kernel<T, S, true> : (void *)hostloop3d_kernel<T, S, false>;
    for (int64_t t = 0; t < steps; t++) {
      const bool src_out = t > 0 && ((steps - t) & 1) == 0;
      const T *src = t == 0 ? in : (src_out ? out : tmp);
      int src_idx = t == 0 ? 0 : (src_out ? 1 : 2);
      u.rev = zigzag && (t & 1);
      T *dst = (((steps - 1 - t) & 1) == 0) ? out : tmp;
      void *args[] = {(void *)&src, (void *)&maps, (void *)&src_idx, (void *)&dst, (void *)&d,
                      (void *)&u, (void *)&c};
      cudaError_t e = cudaLaunchKernel(k, dim3(pl.grid), dim3(G::NT), args, smem, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  void *k = tma ? (void *)persistent3d_kernel<T, S, true> : (void *)persistent3d_kernel<T, S, false>;
  u.rev = zigzag;
  cudaError_t e = cudaMemsetAsync(bar, 0, 256, s);
  if (e != cudaSuccess) return e;
  void *args[] = {(void *)&in, (void *)&out, (void *)&tmp, (void *)&maps, (void *)&d, (void *)&u,
                  (void *)&steps, (void *)&bar, (void *)&c};
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
