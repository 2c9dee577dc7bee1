// k3d_stream.cu — the 3D stencil kernels of all three variants:
//   (a) host-loop: one launch per step, one (tile, z-chunk) unit per CTA  (Fig. 3 left)
//   (b) persistent: one cooperative launch; CTAs loop over units; grid barrier per step
//   (c) PERKS: the persistent kernel plus an on-chip plane cache (§3.3): each
//       CTA keeps `nc` interior planes of its unit resident in shared memory across steps.  "Planes
//       that already have the data cached from the previous time step do not load from global
//       memory": a cached plane reloads only its one-cell halo ring (halo cells are never
//       cached) and publishes only its tile perimeter (TB-boundary cells "continue to
//       store and load from global memory").  Cached planes are spread evenly through the
//       unit so the HBM stream never pauses, and every tile of a z-chunk caches the same planes.
//       The first/last plane of each unit is never cached (other units read it as z-halo).
// Compute body and plane pipelines: stream3d.cuh (plane streaming; TMA on sm_100a).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

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
// Warp-specialised geometries (consumer warps + 1 producer warp, CTAs per SM), chosen per problem
// by the planner (profiles/r01_ws_geometry_sweep.txt): WSG 0 = 8 warps x 2 CTAs/SM (best while the
// domain is within a few L2 sizes, C3/C4); WSG 1 = 4 warps x 3 CTAs/SM (more independent plane
// streams in flight: best for domains far larger than L2, C5).
constexpr int wsg_nwarp(int g) { return g == 0 ? 8 : 4; }
constexpr int wsg_minb(int g) { return g == 0 ? 2 : 3; }
template <typename T, bool WS, int WSG = 0> struct GS { using G = typename G3Sel<T>::G; };
template <typename T, int WSG> struct GS<T, true, WSG> {
  using G = Geo3D<T, 16 / (int)sizeof(T), PERKS_S3D_R, wsg_nwarp(WSG), PERKS_S3D_NS>;
};

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

// Threads per CTA: warp-specialised kernels add one producer warp (stream3d.cuh WsPipe).  The
// host loop (a) keeps the single-role ring (TMA issued by thread 0, CTA barrier per plane) at 4-5
// CTAs per SM, measured faster for one-unit-per-launch CTAs (profiles/r01_ws_pipeline_sweep.txt);
// the persistent kernel (b) uses the warp-specialised pipeline, measured faster when a CTA
// streams long units back to back.
#ifndef PERKS_S3D_HWS
#define PERKS_S3D_HWS 0
#endif
#ifndef PERKS_S3D_MINB
#define PERKS_S3D_MINB 4
#endif
template <bool TMA> constexpr bool host_ws() { return TMA && PERKS_S3D_HWS; }
template <bool WS, int WSG = 0> constexpr int k3d_threads() { return WS ? 32 * wsg_nwarp(WSG) + 32 : K3D_THREADS; }

template <typename T, int S, bool TMA, bool DIST>
__global__ void __launch_bounds__(k3d_threads<host_ws<TMA>()>(), (TMA && !DIST) ? PERKS_S3D_MINB : 2) hostloop3d_kernel(const T *__restrict__ src,
                                                                 const __grid_constant__ Maps3 maps,
                                                                 int src_idx, T *__restrict__ dst,
                                                                 Dom3 d, Units3 u,
                                                                 Coef<T, Shape<S>::N> c, const __grid_constant__ DistK dk,
                                                                 unsigned long long e) {
  using G = typename GS<T, host_ws<TMA>()>::G;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  int x0, y0, zs;
  const int nunits = u.tx * u.ty * u.nzc;
  unit_coords(u, u.rev ? nunits - 1 - (int)blockIdx.x : (int)blockIdx.x, G::TX, G::TY, x0, y0, zs);
  const int ze = min(zs + u.zc, d.nz);
  const DistStep ds{&dk, &maps.ghost, e, (unsigned long long)d.nx * d.ny};
  if constexpr (host_ws<TMA>()) {
    WsPipe<T, G> pp;
    pp.init(reinterpret_cast<T *>(smem_raw), ring_bars<G>(smem_raw));
    stream_unit_ws<T, S, G, DIST>(pp, src, &maps.box[src_idx], dst, d, x0, y0, zs, ze, c, ds);
  } else {
    Ring<T, G, TMA> ring;
    ring.init(reinterpret_cast<T *>(smem_raw), ring_bars<G>(smem_raw), 0);
    stream_unit<T, S, G, TMA, DIST>(ring, src, &maps.box[src_idx], dst, d, x0, y0, zs, ze, c, ds);
  }
}

// Cache geometry of a PERKS launch (CACHE kernels only).
struct Cache3 {
  int nc;  // shared-memory plane slots per CTA
};

// Slot map of a unit [zs, ze): cmap[j] = cache slot of plane zs + j, or -1.  nc slots spread
// evenly over the interior planes zs+1 .. ze-2 (the unit's first/last plane is never cached).
PERKS_DEVINL int cache_slot_of(int j, int len, int nc) {
  const int elig = len - 2, jj = j - 1;
  if (nc <= 0 || jj < 0 || jj >= elig) return -1;
  const int a = (jj * nc) / elig, b = ((jj + 1) * nc) / elig;
  return b != a ? a : -1;
}

template <typename T, int S, bool TMA, bool DIST, bool CACHE, int WSG>
__global__ void __launch_bounds__(k3d_threads<TMA, WSG>(), DIST ? 1 : wsg_minb(WSG)) persistent3d_kernel(
    const T *__restrict__ in, T *out, T *tmp, const __grid_constant__ Maps3 maps, Dom3 d, Units3 u,
    int64_t steps, unsigned *bar, Coef<T, Shape<S>::N> c, const __grid_constant__ DistK dk,
    unsigned long long xbase, Cache3 ch) {
  using G = typename GS<T, TMA, WSG>::G;
  static_assert(!CACHE || TMA, "the PERKS cache runs on the warp-specialised TMA pipeline");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Ring<T, G, TMA> ring;
  WsPipe<T, G> pp;
  if constexpr (TMA) pp.init(reinterpret_cast<T *>(smem_raw), ring_bars<G>(smem_raw));
  else ring.init(reinterpret_cast<T *>(smem_raw), ring_bars<G>(smem_raw), 0);
  const int nunits = u.tx * u.ty * u.nzc;

  // ---- PERKS: the CTA's first unit hosts the cache
  T *cache = reinterpret_cast<T *>(smem_raw + (size_t)G::NS * G::SLOT_BYTES + 128);
  short *cmap = reinterpret_cast<short *>(cache + (size_t)ch.nc * G::SLOT);
  int cx0 = 0, cy0 = 0, czs = 0, cze = 0;
  const bool consumer = (int)(threadIdx.x >> 5) < G::NWARP;
  if constexpr (CACHE) {
    if (blockIdx.x < nunits) {
      unit_coords(u, blockIdx.x, G::TX, G::TY, cx0, cy0, czs);
      cze = min(czs + u.zc, d.nz);
    }
    const int nc = min(ch.nc, max(0, cze - czs - 2));
    for (int j = threadIdx.x; j < cze - czs; j += blockDim.x) cmap[j] = (short)cache_slot_of(j, cze - czs, nc);
    __syncthreads();
    // prologue: cached planes from `in` (the one-time load half of 2·D_cache)
    for (int q = czs + 1; q < cze - 1 && consumer; q++) {
      const int sl = cmap[q - czs];
      if (sl >= 0) issue_plane<T, G>(cache + (size_t)sl * G::SLOT, in, d, q, cx0, cy0, false);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
  }
  const CacheView<T> cv{cache, cmap, czs, cze};

  for (int64_t t = 0; t < steps; t++) {
    const bool src_out = t > 0 && ((steps - t) & 1) == 0;
    const T *src = t == 0 ? in : (src_out ? out : tmp);
    const int src_idx = t == 0 ? 0 : (src_out ? 1 : 2);
    T *dst = ((steps - 1 - t) & 1) == 0 ? out : tmp;
    const DistStep ds{&dk, &maps.ghost, xbase + (unsigned long long)t, (unsigned long long)d.nx * d.ny};
    if (TMA && threadIdx.x == 0) fence_proxy_async_global();  // last step's stores -> TMA reads
    for (int id = blockIdx.x; id < nunits; id += gridDim.x) {
      int x0, y0, zs;
      // (the zig-zag unit-order experiment never applies to PERKS: the cache belongs to a unit)
      unit_coords(u, (!CACHE && u.rev && (t & 1)) ? nunits - 1 - id : id, G::TX, G::TY, x0, y0, zs);
      const int ze = min(zs + u.zc, d.nz);
      if constexpr (TMA) {
        if (CACHE && id == (int)blockIdx.x)
          stream_unit_ws<T, S, G, DIST, CACHE>(pp, src, &maps.box[src_idx], dst, d, x0, y0, zs, ze, c, ds, cv);
        else
          stream_unit_ws<T, S, G, DIST, false>(pp, src, &maps.box[src_idx], dst, d, x0, y0, zs, ze, c, ds);
      } else {
        __syncthreads();  // slots of the previous unit are free
        stream_unit<T, S, G, TMA, DIST>(ring, src, &maps.box[src_idx], dst, d, x0, y0, zs, ze, c, ds);
      }
    }
    if (t + 1 < steps) grid_barrier(bar, (unsigned)((t + 1) * gridDim.x));
  }

  if constexpr (CACHE) {  // epilogue: cached planes to `out` (store half of 2·D_cache)
    __syncthreads();
    ThreadTile<G> ct;
    ct.init(d, cx0, cy0);
    for (int q = czs + 1; q < cze - 1 && consumer; q++) {
      const int sl = cmap[q - czs];
      if (sl < 0) continue;
      T v[G::R][G::V];
      read_own<T, G>(cache + (size_t)sl * G::SLOT, v);
      store_cells<T, G>(out, d, ct, q, v);
    }
  }
}

// Multi-GPU prologue: exchange xbase = the run's INPUT face planes.  blockIdx.y = side (0: plane 0
// to the lower neighbour's ghost side 1; 1: plane nz-1 to the upper neighbour's ghost side 0);
// each CTA copies 8 rows.  Before overwriting the neighbour's ghost parity, wait until that
// neighbour's last exchange of the previous run arrived (it was produced after the neighbour's
// last ghost read, so the slot is free: no write-after-read across runs).
template <typename T>
__global__ void __launch_bounds__(256) dist_prologue_kernel(const T *__restrict__ in, DistK dk, int nx,
                                                            int ny, int nz, unsigned long long xbase) {
  const int side = blockIdx.y;
  if (side == 0 ? !dk.has_lo : !dk.has_hi) return;
  const unsigned long long plane = (unsigned long long)nx * ny;
  if (threadIdx.x == 0) wait_counter_sys(dk.ctr + side, xbase * plane);
  __syncthreads();
  const int y0 = blockIdx.x * 8, y1 = min(y0 + 8, ny);
  const T *srcp = in + (side == 0 ? (size_t)0 : (size_t)(nz - 1) * plane) + (size_t)y0 * nx;
  T *dstp = reinterpret_cast<T *>(side == 0 ? dk.send_lo : dk.send_hi) +
            (size_t)((xbase & 1) * 2 + (side == 0 ? 1 : 0)) * plane + (size_t)y0 * nx;
  const int n16 = (int)((size_t)(y1 - y0) * nx * sizeof(T) / 16);  // nx*S % 16 == 0 (planner)
  const uint4 *s4 = reinterpret_cast<const uint4 *>(srcp);
  uint4 *d4 = reinterpret_cast<uint4 *>(dstp);
  for (int i = threadIdx.x; i < n16; i += blockDim.x) d4[i] = s4[i];
  signal_counter_sys(side == 0 ? dk.peer_ctr_lo : dk.peer_ctr_hi, (unsigned long long)(y1 - y0) * nx);
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
                Maps3 *m, const void *ghost) {
  const void *b[3] = {in, out, tmp ? tmp : out};
  for (int i = 0; i < 3; i++) {
    if (!encode_map3(&m->box[i], p, b[i], P, ROWS)) return false;
    if (!encode_map3(&m->row[i], p, b[i], P, 1)) return false;
  }
  if (ghost) {  // G[4][ny][nx]
    Problem g = p;
    g.nz = 4;
    if (!encode_map3(&m->ghost, g, ghost, P, ROWS)) return false;
  }
  return true;
}

Dom3 make_dom3(const Problem &p) {
  Dom3 d{(int)p.nx, (int)p.ny, (int)p.nz, 1, (int)p.nz - 2};
  if (p.rank > 0) d.zlo = 0;                  // lower face has a neighbour: interior (R12)
  if (p.rank < p.nranks - 1) d.zhi = (int)p.nz - 1;
  return d;
}

DistK make_distk(const DistRun *dr) {
  DistK k{};
  if (!dr) return k;
  k.ctr = dr->ctr;
  k.has_lo = dr->has_lo;
  k.has_hi = dr->has_hi;
  k.send_lo = dr->lo_ghost;
  k.send_hi = dr->hi_ghost;
  k.peer_ctr_lo = dr->lo_ctr ? dr->lo_ctr + 1 : nullptr;  // I am the lower neighbour's upper
  k.peer_ctr_hi = dr->hi_ctr ? dr->hi_ctr + 0 : nullptr;
  return k;
}

cudaError_t launch_dist_prologue(const Problem &p, const void *in, const DistRun &dr, cudaStream_t s) {
  if (!dr.has_lo && !dr.has_hi) return cudaSuccess;
  DistK k = make_distk(&dr);
  int nx = (int)p.nx, ny = (int)p.ny, nz = (int)p.nz;
  unsigned long long xb = dr.xbase;
  dim3 grid((unsigned)((ny + 7) / 8), 2);
  if (p.dtype == PERKS_F32)
    dist_prologue_kernel<float><<<grid, 256, 0, s>>>((const float *)in, k, nx, ny, nz, xb);
  else
    dist_prologue_kernel<double><<<grid, 256, 0, s>>>((const double *)in, k, nx, ny, nz, xb);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ host side
namespace {
// persistent kernel pointer for (shape, TMA, DIST, CACHE, WSG)
template <typename T, int S, bool DIST, bool CACHE> void *pk_w(int wsg) {
  return wsg == 1 ? (void *)persistent3d_kernel<T, S, true, DIST, CACHE, 1>
                  : (void *)persistent3d_kernel<T, S, true, DIST, CACHE, 0>;
}
template <typename T, int S> void *pk_s(bool tma, bool dist, bool cache, int wsg) {
  if (!tma) return (void *)persistent3d_kernel<T, S, false, false, false, 0>;
  if (dist) return cache ? pk_w<T, S, true, true>(wsg) : pk_w<T, S, true, false>(wsg);
  return cache ? pk_w<T, S, false, true>(wsg) : pk_w<T, S, false, false>(wsg);
}
template <typename T> void *pk(int shape, bool tma, bool dist, bool cache, int wsg) {
  return shape == SHAPE_3D7 ? pk_s<T, SHAPE_3D7>(tma, dist, cache, wsg) : pk_s<T, SHAPE_3D27>(tma, dist, cache, wsg);
}
void *persist_ptr(const Problem &p, bool tma, bool cache, int wsg) {
  const bool dist = p.nranks > 1;
  return p.dtype == PERKS_F32 ? pk<float>(p.shape, tma, dist, cache, wsg) : pk<double>(p.shape, tma, dist, cache, wsg);
}
template <typename T> void *kptr3d(int shape, bool persistent) {  // multi-GPU host-loop kernels (TMA)
  (void)persistent;
  return shape == SHAPE_3D7 ? (void *)hostloop3d_kernel<T, SHAPE_3D7, true, true>
                            : (void *)hostloop3d_kernel<T, SHAPE_3D27, true, true>;
}
template <typename T> void *kptr3(int shape, bool persistent, bool tma) {
#define K3(S)                                                                                   \
  if (shape == S) {                                                                             \
    (void)persistent; \
    return tma ? (void *)hostloop3d_kernel<T, S, true, false> : (void *)hostloop3d_kernel<T, S, false, false>; \
  }
  K3(SHAPE_3D7)
  K3(SHAPE_3D27)
#undef K3
  return nullptr;
}
// host-loop kernel pointer
void *pick3(const Problem &p, bool persistent) {
  const bool tma = use_tma3(p);
  if (p.nranks > 1) return p.dtype == PERKS_F32 ? kptr3d<float>(p.shape, persistent) : kptr3d<double>(p.shape, persistent);
  return p.dtype == PERKS_F32 ? kptr3<float>(p.shape, persistent, tma) : kptr3<double>(p.shape, persistent, tma);
}
template <typename T, bool WS, int WSG> void geo3_t(int &tx, int &ty, int &nt, size_t &slot, size_t &ring,
                                                  int &P, int &ROWS) {
  using G = typename GS<T, WS, WSG>::G;
  tx = G::TX; ty = G::TY; nt = G::NT + (WS ? 32 : 0); slot = G::SLOT_BYTES;
  ring = (size_t)G::NS * G::SLOT_BYTES + 2 * (size_t)G::NS * sizeof(uint64_t);
  P = G::P; ROWS = G::ROWS;
}
struct Geo3Info { int TX, TY, NT, P, ROWS; size_t slot, ring; };
template <typename T> Geo3Info geo3(bool ws, int wsg) {
  Geo3Info g;
  if (!ws) geo3_t<T, false, 0>(g.TX, g.TY, g.NT, g.slot, g.ring, g.P, g.ROWS);
  else if (wsg == 1) geo3_t<T, true, 1>(g.TX, g.TY, g.NT, g.slot, g.ring, g.P, g.ROWS);
  else geo3_t<T, true, 0>(g.TX, g.TY, g.NT, g.slot, g.ring, g.P, g.ROWS);
  return g;
}
}  // namespace


// Plan (a) host loop, (b) persistent or (c) PERKS for a 3D problem.
Plan plan_stream3d(const Problem &p, perks_variant v) {
  Plan pl;
  pl.variant = v;
  if (p.ndim != 3 || (p.shape != SHAPE_3D7 && p.shape != SHAPE_3D27) || p.bc != PERKS_BC_FRAME) {
    pl.why = "stream3d: needs 3D 7pt/27pt FRAME";
    return pl;
  }
  const bool tma = use_tma3(p);
  if (p.nranks > 1 && !tma) { pl.why = "stream3d: multi-GPU slabs need TMA (nx*S % 16 == 0)"; return pl; }
  const bool cache = v == PERKS_PERKS;
  if (cache && !tma) { pl.why = "perks3d: needs TMA (nx*S % 16 == 0)"; return pl; }
  const bool persistent = v != PERKS_HOSTLOOP;
  const bool ws = tma && persistent;  // warp-specialised pipeline (persistent kernels)
  // WS geometry: 4 warps x 3 CTAs/SM once one buffer is >= 16 L2 sizes (more plane streams in
  // flight for DRAM-latency-bound streaming), else 8 warps x 2 CTAs/SM
  int wsg = ((double)p.cells() * p.elem() >= 16.0 * (double)p.l2_bytes) ? 1 : 0;
  if (env_int("PERKS_WSG", -1) >= 0) wsg = env_int("PERKS_WSG", 0) ? 1 : 0;
  if (!ws) wsg = 0;
  void *k = persistent ? persist_ptr(p, tma, cache, wsg) : pick3(p, false);
  const Geo3Info gi = p.dtype == PERKS_F32 ? geo3<float>(ws, wsg) : geo3<double>(ws, wsg);
  const size_t ring = gi.ring, slot = gi.slot;
  const int TX = gi.TX, TY = gi.TY, NT = gi.NT;
  const int tx = (int)((p.nx + TX - 1) / TX), ty = (int)((p.ny + TY - 1) / TY);
  const int tiles = tx * ty;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  size_t smem = ring;
  int occ = 0, nc = 0;
  if (!cache) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      cudaGetLastError();
      pl.why = "cudaFuncSetAttribute"; return pl;
    }
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem);
  } else {
    // PERKS: the shared memory the ring leaves at `cps` CTAs per SM caches planes (
    // minimal occupancy that keeps the HBM stream saturated: 2 CTAs/SM measured best)
    const int force_cps = env_int("PERKS_P3D_CPS", 0);
    for (int cps = force_cps > 0 ? force_cps : wsg_minb(wsg); cps >= 1; cps--) {
      const size_t budget = std::min<size_t>((size_t)p.max_smem_optin, (size_t)p.smem_per_sm / cps - 1024);
      const size_t fixed = ring + 128 + align256((size_t)p.nz * sizeof(short));
      nc = budget > fixed ? (int)((budget - fixed) / slot) : 0;
      const int forced = env_int("PERKS_P3D_NSM", -1);
      if (forced >= 0) nc = std::min(nc, forced);
      smem = fixed + (size_t)nc * slot;
      if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem);
      if (occ >= cps) { occ = cps; break; }
    }
  }
  if (occ < 1) { pl.why = "stream3d: not co-resident"; return pl; }
  const int resident = occ * p.num_sms;
  // z chunks: about two waves of units for the host loop; exactly one wave for the persistent
  // kernels (one unit per CTA per step, so no CTA idles at the tail)
  int nzc = std::max(1, (2 * resident + tiles - 1) / tiles);
  nzc = std::min<int>(nzc, (int)std::max<int64_t>(1, p.nz / 8));
  if (persistent) {
    // persistent kernels: pick the z-chunking that minimises the busiest CTA's planes per step,
    // ceil(units / grid) * (chunk + 2 halo planes), with grid <= resident CTAs (load balance over
    // 148 SMs: e.g. C3 64 tiles x 4 chunks on 256 CTAs; C5 1024 tiles x 2 chunks)
    int64_t best = -1;
    for (int n = 1; n <= std::max<int64_t>(1, p.nz / 4); n++) {
      const int64_t zcn = (p.nz + n - 1) / n, nn = (p.nz + zcn - 1) / zcn;
      if (nn != n) continue;
      const int64_t un = (int64_t)tiles * n, g = std::min<int64_t>(un, resident);
      const int64_t cost = ((un + g - 1) / g) * (zcn + 2);
      if (best < 0 || cost < best) { best = cost; nzc = n; }
    }
  }
  if (persistent && env_int("PERKS_S3D_NZC", 0) > 0) nzc = std::min<int>(env_int("PERKS_S3D_NZC", 0), (int)p.nz);  // sweeps
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
  pl.cfg = tma ? 1 : 0;
  pl.family = cache ? 2 : 0;  // (2: PERKS 3D, supports multi-GPU slabs)
  pl.wsg = wsg;
  pl.nc = cache ? std::min(nc, std::max(0, zc - 2)) : 0;
  const double S = (double)p.elem();
  // cached cells: every CTA's first unit caches nc planes of its tile (last z-chunk may be shorter)
  int64_t cached = 0;
  if (cache) {
    for (int cz = 0; cz < nzc; cz++) {
      const int len = (int)std::min<int64_t>(zc, p.nz - (int64_t)cz * zc);
      cached += (int64_t)tiles * std::min(pl.nc, std::max(0, len - 2));
    }
    if (pl.units > pl.grid) cached = cached * pl.grid / pl.units;
    cached *= (int64_t)TX * TY;
    cached = std::min<int64_t>(cached, p.cells());
  }
  pl.cached_smem = cached;
  pl.dram_bytes_step = 2.0 * S * ((double)p.cells() - (double)cached);
  pl.halo_bytes_step = S * (double)p.nz * (2.0 * TX * ty * tx + 2.0 * TY * ty * tx) +
                       S * 2.0 * nzc * (double)p.nx * p.ny;
  pl.ws_bytes = align256((size_t)p.cells() * p.elem()) + (persistent ? 256 : 0);
  snprintf(pl.name, sizeof(pl.name), "%s3d_%s_%s_t%dx%d_z%d%s", cache ? "perks" : persistent ? "persistent" : "hostloop",
           p.shape == SHAPE_3D7 ? "7pt" : "27pt", p.dtype == PERKS_F32 ? "f32" : "f64", TX, TY, zc,
           cache ? "_c" : (pl.cfg ? "_tma" : "_cpasync"));
  if (cache) {
    char extra[24];
    snprintf(extra, sizeof(extra), "%d_%dcta", pl.nc, occ);
    strncat(pl.name, extra, sizeof(pl.name) - strlen(pl.name) - 1);
  }
  pl.ok = true;
  return pl;
}

namespace {
// Everything one 3D streaming launch needs, prepared once per run.
template <typename T, int S>
struct Launch3 {
  Coef<T, Shape<S>::N> c;
  Dom3 d;
  Units3 u;
  Maps3 maps;
  DistK dk;
  unsigned long long xbase = 0;
  const T *in;
  T *out, *tmp;
  unsigned *bar;
  size_t smem;
  bool tma;
  int grid;
  int zigzag;
  bool cache = false;
  Cache3 ch{0};
  int block = 0;
  int wsg = 0;

  cudaError_t setup(const Problem &p, const Plan &pl, const T *in_, T *out_, T *tmp_, unsigned *bar_,
                    const DistRun *dr) {
    for (int i = 0; i < Shape<S>::N; i++) c.w[i] = sizeof(T) == 4 ? (T)p.wf[i] : (T)p.wd[i];
    d = make_dom3(p);
    u = Units3{(int)((p.nx + pl.tile[0] - 1) / pl.tile[0]), (int)((p.ny + pl.tile[1] - 1) / pl.tile[1]), 0,
               pl.zchunk, 0};
    block = pl.block;
    u.nzc = (int)((p.nz + u.zc - 1) / u.zc);
    zigzag = env_int("PERKS_ZIGZAG", 0);  // experiment knob; off by default
    smem = (size_t)pl.smem;
    tma = pl.cfg == 1;
    grid = pl.grid;
    in = in_; out = out_; tmp = tmp_; bar = bar_;
    dk = make_distk(dr);
    xbase = dr ? dr->xbase : 0;
    dist = p.nranks > 1;
    cache = pl.family == 2;
    ch.nc = pl.nc;
    if (dist && !tma) return cudaErrorNotSupported;
    std::memset(&maps, 0, sizeof(maps));
    const bool ws = pl.variant != PERKS_HOSTLOOP && pl.cfg == 1;
    wsg = pl.wsg;
    const Geo3Info gi = geo3<T>(ws, wsg);
    const int P = gi.P, ROWS = gi.ROWS;
    if (tma && !make_maps3(p, P, ROWS, in, out, tmp, &maps, dr ? dr->ghost : nullptr))
      return cudaErrorInvalidValue;
    return cudaSuccess;
  }
  // host loop (a): the kernel of step t of `steps`
  bool dist = false;
  cudaError_t step(int64_t t, int64_t steps, cudaStream_t s) {
    void *k = dist ? (void *)hostloop3d_kernel<T, S, true, true>
                   : tma ? (void *)hostloop3d_kernel<T, S, true, false> : (void *)hostloop3d_kernel<T, S, false, false>;
    const bool src_out = t > 0 && ((steps - t) & 1) == 0;
    const T *src = t == 0 ? in : (src_out ? out : tmp);
    int src_idx = t == 0 ? 0 : (src_out ? 1 : 2);
    T *dst = (((steps - 1 - t) & 1) == 0) ? out : tmp;
    Units3 uu = u;
    uu.rev = zigzag && (t & 1);
    unsigned long long e = xbase + (unsigned long long)t;
    void *args[] = {(void *)&src, (void *)&maps, (void *)&src_idx, (void *)&dst, (void *)&d,
                    (void *)&uu, (void *)&c, (void *)&dk, (void *)&e};
    return cudaLaunchKernel(k, dim3(grid), dim3(block), args, smem, s);
  }
  // persistent (b): one launch; cooperative on a single GPU (co-residency guaranteed by the driver)
  cudaError_t persistent(int64_t steps, cudaStream_t s, bool cooperative) {
    void *k = pk_s<T, S>(tma, dist, cache, wsg);
    Units3 uu = u;
    uu.rev = zigzag;
    cudaError_t e = cudaMemsetAsync(bar, 0, 256, s);
    if (e != cudaSuccess) return e;
    void *args[] = {(void *)&in, (void *)&out, (void *)&tmp, (void *)&maps, (void *)&d, (void *)&uu,
                    (void *)&steps, (void *)&bar, (void *)&c, (void *)&dk, (void *)&xbase, (void *)&ch};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = cooperative ? 1 : 0;
    return cudaLaunchKernelExC(&cfg, k, args);
  }
};

template <typename T, int S>
cudaError_t run3(const Problem &p, const Plan &pl, const void *in, void *out, void *ws, int64_t steps,
                 cudaStream_t s, const DistRun *dr) {
  char *w = (char *)ws;
  unsigned *bar = (unsigned *)(w + align256((size_t)p.cells() * p.elem()));
  Launch3<T, S> L;
  cudaError_t e = L.setup(p, pl, (const T *)in, (T *)out, (T *)w, bar, dr);
  if (e != cudaSuccess) return e;
  if (dr && (e = launch_dist_prologue(p, in, *dr, s)) != cudaSuccess) return e;
  if (pl.variant == PERKS_HOSTLOOP) {
    for (int64_t t = 0; t < steps; t++)
      if ((e = L.step(t, steps, s)) != cudaSuccess) return e;
    return cudaSuccess;
  }
  return L.persistent(steps, s, !(dr && dr->noncoop));
}
}  // namespace

cudaError_t run_stream3d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws,
                         int64_t steps, cudaStream_t s, const DistRun *dr) {
  if (p.dtype == PERKS_F32)
    return p.shape == SHAPE_3D7 ? run3<float, SHAPE_3D7>(p, pl, in, out, ws, steps, s, dr)
                                : run3<float, SHAPE_3D27>(p, pl, in, out, ws, steps, s, dr);
  return p.shape == SHAPE_3D7 ? run3<double, SHAPE_3D7>(p, pl, in, out, ws, steps, s, dr)
                              : run3<double, SHAPE_3D27>(p, pl, in, out, ws, steps, s, dr);
}

namespace {
template <typename T, int S>
cudaError_t group3(const Problem *const *ps, const Plan *const *pls, const void *const *in,
                   void *const *out, void *const *ws, const DistRun *drs, int n, int64_t steps,
                   cudaStream_t s) {
  std::vector<Launch3<T, S>> L(n);
  for (int i = 0; i < n; i++) {
    char *w = (char *)ws[i];
    unsigned *bar = (unsigned *)(w + align256((size_t)ps[i]->cells() * ps[i]->elem()));
    cudaError_t e = L[i].setup(*ps[i], *pls[i], (const T *)in[i], (T *)out[i], (T *)w, bar, &drs[i]);
    if (e != cudaSuccess) return e;
  }
  for (int i = 0; i < n; i++) {
    cudaError_t e = launch_dist_prologue(*ps[i], in[i], drs[i], s);
    if (e != cudaSuccess) return e;
  }
  for (int64_t t = 0; t < steps; t++)
    for (int i = 0; i < n; i++) {
      cudaError_t e = L[i].step(t, steps, s);
      if (e != cudaSuccess) return e;
    }
  return cudaSuccess;
}
}  // namespace

cudaError_t run_stream3d_hostloop_group(const Problem *const *ps, const Plan *const *pls,
                                        const void *const *in, void *const *out, void *const *ws,
                                        const DistRun *drs, int n, int64_t steps, cudaStream_t s) {
  const Problem &p = *ps[0];
  if (p.dtype == PERKS_F32)
    return p.shape == SHAPE_3D7 ? group3<float, SHAPE_3D7>(ps, pls, in, out, ws, drs, n, steps, s)
                                : group3<float, SHAPE_3D27>(ps, pls, in, out, ws, drs, n, steps, s);
  return p.shape == SHAPE_3D7 ? group3<double, SHAPE_3D7>(ps, pls, in, out, ws, drs, n, steps, s)
                              : group3<double, SHAPE_3D27>(ps, pls, in, out, ws, drs, n, steps, s);
}

}  // namespace perks
