// k3d_stream.cu — the 3D stencil kernels of all three variants:
//   (a) host-loop: one launch per step, one (tile, z-chunk) unit per CTA  (Fig. 3 left)
//   (b) persistent: one cooperative launch; CTAs loop over units; grid barrier per step
//   (c) PERKS: the persistent kernel plus an on-chip plane cache (§3.3): each
//       CTA keeps `nc` tile planes resident in shared memory and `ntm` in Tensor Memory (tmem.cuh,
//       the sm_100a tier the paper's GPUs lack) across steps.  "Planes that already have the data
//       cached from the previous time step do not load from global memory": a cached
//       plane reloads only its one-cell halo ring (halo cells are never cached) and
//       publishes only its tile perimeter (TB-boundary cells "continue to store and load from
//       global memory").  The cached planes are spread evenly over ALL of the CTA's units
//       of a step, so every CTA's HBM stream continues through the whole step.  The first/last
//       plane of each unit is never cached (other units read it as z-halo).
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
// WSG 2 = 8 warps x 4 rows x 1 CTA/SM: one CTA per SM with a large register budget per thread
// (profiles/r01_wsg2_sweep.txt; a single CTA per SM also keeps the TMEM tier launchable
// cooperatively).
constexpr int wsg_nwarp(int g) { return g == 1 ? 4 : 8; }
constexpr int wsg_minb(int g) { return g == 0 ? 2 : g == 1 ? 3 : 1; }
constexpr int wsg_r(int g) { return g == 2 ? 2 * PERKS_S3D_R : PERKS_S3D_R; }
constexpr int kNumWsg = 3;
template <typename T, bool WS, int WSG = 0> struct GS { using G = typename G3Sel<T>::G; };
template <typename T, int WSG> struct GS<T, true, WSG> {
  using G = Geo3D<T, 16 / (int)sizeof(T), wsg_r(WSG), wsg_nwarp(WSG), PERKS_S3D_NS>;
};

struct Units3 {
  int tx, ty, nzc, zc;
  int rev;  // zig-zag traversal: host loop: reversed unit order in this launch; persistent /
            // PERKS: every CTA reverses its units on odd steps
};

PERKS_DEVINL void unit_coords(const Units3 &u, int id, int tile_x, int tile_y, int &x0, int &y0,
                              int &zs) {
  const int t = id % (u.tx * u.ty);
  const int zc = id / (u.tx * u.ty);
  x0 = (t % u.tx) * tile_x;
  y0 = (t / u.tx) * tile_y;
  zs = zc * u.zc;
}

// Ring slots, then full/empty/tfull mbarriers (3 x NS) and the TMEM base address (Geo3D::BAR_BYTES,
// before the PERKS plane cache).
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
// host-loop CTAs per SM (launch bound): fp64 27pt needs more than 64 registers per thread
template <typename T, int S, bool TMA, bool DIST> constexpr int hl_minb() {
  return !(TMA && !DIST) ? 2 : (sizeof(T) == 8 && S != SHAPE_3D7) ? 3 : PERKS_S3D_MINB;
}
template <bool WS, int WSG = 0> constexpr int k3d_threads() { return WS ? 32 * wsg_nwarp(WSG) + 32 : K3D_THREADS; }

template <typename T, int S, bool TMA, bool DIST>
__global__ void __launch_bounds__(k3d_threads<host_ws<TMA>()>(), hl_minb<T, S, TMA, DIST>()) hostloop3d_kernel(const T *__restrict__ src,
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
    pp.init();
    stream_unit_ws<T, S, G, DIST>(pp, src, &maps.box[src_idx], dst, d, x0, y0, zs, ze, c, ds);
  } else {
    Ring<T, G, TMA> ring;
    ring.init(reinterpret_cast<T *>(smem_raw), ring_bars<G>(smem_raw), 0);
    stream_unit<T, S, G, TMA, DIST>(ring, src, &maps.box[src_idx], dst, d, x0, y0, zs, ze, c, ds);
  }
}

// Cache geometry of a PERKS launch (CACHE kernels only).
struct Cache3 {
  int nc;     // shared-memory plane slots per CTA
  int ntm;    // TMEM planes per CTA (tmem.cuh; 0 = no TMEM tier)
  int tcols;  // TMEM columns allocated per CTA (power of two >= 32, 512 / CTAs per SM)
};

// Cache code of arrival a of a CTA's step (PERKS).  The CTA's units are processed back to back,
// unit j contributing arrivals for its planes zs-1 .. ze (len + 2, len = ze - zs); its eligible
// planes are zs+1 .. ze-2 (the first/last plane of a unit is read by other units as z-halo and is
// never cached).  Of the E eligible planes of the whole step, n = ns + nt are cached, spread
// evenly (plane g is chosen iff floor((g+1)n/E) > floor(gn/E)), and the nt TMEM planes evenly
// among the chosen ones.
PERKS_DEVINL int cache_code_of(int g, int E, int ns, int nt) {
  const int n = ns + nt;
  if (n <= 0 || g < 0 || g >= E) return -1;
  const int a = (g * n) / E, b = ((g + 1) * n) / E;
  if (b == a) return -1;
  const int t0 = (a * nt) / n, t1 = ((a + 1) * nt) / n;  // TMEM planes among chosen [0, a) / [0, a]
  return t1 != t0 ? kTmemCode + t0 : a - t1;
}
// The CTA's unit j of a step: tile origin, z range.
struct UnitGeo {
  int x0, y0, zs, ze;
};
template <class G> PERKS_DEVINL UnitGeo my_unit(const Units3 &u, const Dom3 &d, int j) {
  UnitGeo g;
  unit_coords(u, (int)blockIdx.x + j * (int)gridDim.x, G::TX, G::TY, g.x0, g.y0, g.zs);
  g.ze = min(g.zs + u.zc, d.nz);
  return g;
}
// Visit every cached plane of the CTA (prologue / epilogue): f(unit geometry, plane q, code).
template <class G, class F>
PERKS_DEVINL void for_cached_planes(const Units3 &u, const Dom3 &d, int nmine, const signed char *cmap, F f) {
  int abase = 0;
  for (int j = 0; j < nmine; j++) {
    const UnitGeo g = my_unit<G>(u, d, j);
    for (int q = g.zs + 1; q < g.ze - 1; q++) {
      const int c = cmap[abase + q - g.zs + 1];
      if (c >= 0) f(g, q, c);
    }
    abase += g.ze - g.zs + 2;
  }
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
  if constexpr (TMA) pp.init();
  else ring.init(reinterpret_cast<T *>(smem_raw), ring_bars<G>(smem_raw), 0);
  const int nunits = u.tx * u.ty * u.nzc;

  // ---- PERKS: cached planes spread over all of this CTA's units (CacheView, stream3d.cuh)
  const int nmine = (int)blockIdx.x < nunits ? (nunits - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  CacheView<T, G> cv{ch.nc, 0, 0u};
  signed char *cmap = cv.cmap();
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(ring_bars<G>(smem_raw) + 3 * G::NS);
  const int warp = (int)(threadIdx.x >> 5);
  const bool consumer = warp < G::NWARP;
  if constexpr (CACHE) {
    int E = 0, A = 0;
    for (int j = 0; j < nmine; j++) {
      const UnitGeo g = my_unit<G>(u, d, j);
      E += max(0, g.ze - g.zs - 2);
      A += g.ze - g.zs + 2;
    }
    const int n = min(ch.nc + ch.ntm, E), ns = min(ch.nc, n), nt = min(ch.ntm, n - ns);
    for (int a = threadIdx.x; a <= A; a += blockDim.x) {  // (a == A: the -1 sentinel)
      int abase = 0, gbase = 0, code = -1;
      for (int j = 0; j < nmine; j++) {
        const UnitGeo g = my_unit<G>(u, d, j);
        const int len = g.ze - g.zs;
        if (a < abase + len + 2) {
          const int k = a - abase;  // plane zs - 1 + k
          if (k >= 2 && k <= len - 1) code = cache_code_of(gbase + k - 2, E, ns, nt);
          break;
        }
        abase += len + 2;
        gbase += max(0, len - 2);
      }
      cmap[a] = (signed char)code;
    }
    if (warp == 0) {
      if (ch.tcols > 0) tmem_alloc(tmem_slot, (uint32_t)ch.tcols);
      tmem_relinquish();  // lets the next CTA onto this SM (tmem.cuh)
    }
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
    if (ch.tcols > 0)  // lane quarter of this warp, column group of its warp-group half
      cv.tbase = *tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) +
                 (uint32_t)((warp >> 2) * TmemCells<T, G::R, G::V>::WPT);
    // prologue: cached planes from `in` (the one-time load half of 2·D_cache)
    if (consumer)
      for_cached_planes<G>(u, d, nmine, cmap, [&](const UnitGeo &g, int q, int code) {
        if (is_smem_code(code)) {
          issue_plane<T, G>(cv.slot(code), in, d, q, g.x0, g.y0, false);
        } else {
          ThreadTile<G> ct;
          ct.init(d, g.x0, g.y0);
          T v[G::R][G::V];
          load_own_cells<T, G>(in, d, ct, q, v);
          TmemCells<T, G::R, G::V>::store(cv.tbase + (uint32_t)((code - kTmemCode) * tmem_cpp<T, G>()), v);
        }
      });
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
  }

  for (int64_t t = 0; t < steps; t++) {
    const bool src_out = t > 0 && ((steps - t) & 1) == 0;
    const T *src = t == 0 ? in : (src_out ? out : tmp);
    const int src_idx = t == 0 ? 0 : (src_out ? 1 : 2);
    T *dst = ((steps - 1 - t) & 1) == 0 ? out : tmp;
    const DistStep ds{&dk, &maps.ghost, xbase + (unsigned long long)t, (unsigned long long)d.nx * d.ny};
    if (TMA && threadIdx.x == 0) fence_proxy_async_global();  // last step's stores -> TMA reads
    // L2-aware traversal ("zig-zag", [draft] P:395-404): on odd steps every CTA runs its units in
    // reverse, so a step starts on the tiles the previous step wrote last (still L2-resident:
    // B200's L2 is about one buffer of C3).  Each CTA keeps its units (and its cached planes).
    const bool rev = u.rev && (t & 1);
    for (int jj = 0; jj < nmine; jj++) {
      const int j = rev ? nmine - 1 - jj : jj;
      const int id = (int)blockIdx.x + j * (int)gridDim.x;
      int x0, y0, zs;
      unit_coords(u, id, G::TX, G::TY, x0, y0, zs);
      const int ze = min(zs + u.zc, d.nz);
      if constexpr (TMA) {
        if constexpr (CACHE) {  // arrival offset of unit j in the forward order (cache-code map)
          cv.kbase = 0;
          for (int i = 0; i < j; i++) {
            int xi, yi, zi;
            unit_coords(u, (int)blockIdx.x + i * (int)gridDim.x, G::TX, G::TY, xi, yi, zi);
            cv.kbase += min(zi + u.zc, d.nz) - zi + 2;
          }
        }
        stream_unit_ws<T, S, G, DIST, CACHE>(pp, src, &maps.box[src_idx], dst, d, x0, y0, zs, ze, c, ds, cv);
      } else {
        __syncthreads();  // slots of the previous unit are free
        stream_unit<T, S, G, TMA, DIST>(ring, src, &maps.box[src_idx], dst, d, x0, y0, zs, ze, c, ds);
      }
    }
    if (t + 1 < steps) grid_barrier(bar, (unsigned)(t + 1));
  }

  if constexpr (CACHE) {  // epilogue: cached planes to `out` (store half of 2·D_cache)
    __syncthreads();
    if (consumer)
      for_cached_planes<G>(u, d, nmine, cmap, [&](const UnitGeo &g, int q, int code) {
        ThreadTile<G> ct;
        ct.init(d, g.x0, g.y0);
        T v[G::R][G::V];
        if (is_tmem_code(code))
          TmemCells<T, G::R, G::V>::load(cv.tbase + (uint32_t)((code - kTmemCode) * tmem_cpp<T, G>()), v);
        else
          read_own<T, G>(cv.slot(code), v);
        store_cells<T, G>(out, d, ct, q, v);
      });
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
    if (ch.tcols > 0 && warp == 0) tmem_dealloc(*tmem_slot, (uint32_t)ch.tcols);
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
bool encode_map3(CUtensorMap *m, const Problem &p, const void *base, int bx, int by, int promo) {
  if (!tma_available()) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)p.nx, (cuuint64_t)p.ny, (cuuint64_t)p.nz};
  const cuuint64_t strides[2] = {(cuuint64_t)(p.nx * p.elem()), (cuuint64_t)(p.nx * p.ny * p.elem())};
  const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUtensorMapL2promotion pr = promo == 0    ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                    : promo == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                    : promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                   : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult r = g_encode(m, p.dtype == PERKS_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        3, const_cast<void *>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// L2 promotion of the box fetches: 256 B (sweeps: PERKS_TMA_L2PROMO = 0 / 64 / 128 / 256 bytes)
bool encode_map3(CUtensorMap *m, const Problem &p, const void *base, int bx, int by) {
  return encode_map3(m, p, base, bx, by, env_int("PERKS_TMA_L2PROMO", 256));
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
  switch (wsg) {
    case 1: return (void *)persistent3d_kernel<T, S, true, DIST, CACHE, 1>;
    default: break;
  }
  if constexpr (!DIST) {  // (multi-GPU slabs use WSG 0/1 only)
    if (wsg == 2) return (void *)persistent3d_kernel<T, S, true, DIST, CACHE, 2>;
  }
  return (void *)persistent3d_kernel<T, S, true, DIST, CACHE, 0>;
}
template <typename T, int S> void *pk_s(bool tma, bool dist, bool cache, int wsg) {
  if (!tma) return (void *)persistent3d_kernel<T, S, false, false, false, 0>;
  if (dist) return cache ? pk_w<T, S, true, true>(wsg) : pk_w<T, S, true, false>(wsg);
  return cache ? pk_w<T, S, false, true>(wsg) : pk_w<T, S, false, false>(wsg);
}
template <typename T> void *pk(int shape, bool tma, bool dist, bool cache, int wsg) {
  return shape == SHAPE_3D7    ? pk_s<T, SHAPE_3D7>(tma, dist, cache, wsg)
         : shape == SHAPE_3D19 ? pk_s<T, SHAPE_3D19>(tma, dist, cache, wsg)
                               : pk_s<T, SHAPE_3D27>(tma, dist, cache, wsg);
}
void *persist_ptr(const Problem &p, bool tma, bool cache, int wsg) {
  const bool dist = p.nranks > 1;
  return p.dtype == PERKS_F32 ? pk<float>(p.shape, tma, dist, cache, wsg) : pk<double>(p.shape, tma, dist, cache, wsg);
}
template <typename T> void *kptr3d(int shape, bool persistent) {  // multi-GPU host-loop kernels (TMA)
  (void)persistent;
  return shape == SHAPE_3D7    ? (void *)hostloop3d_kernel<T, SHAPE_3D7, true, true>
         : shape == SHAPE_3D19 ? (void *)hostloop3d_kernel<T, SHAPE_3D19, true, true>
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
  K3(SHAPE_3D19)
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
  ring = G::RING_BYTES;  // slots + mbarriers + TMEM address (Geo3D)
  P = G::P; ROWS = G::ROWS;
}
struct Geo3Info { int TX, TY, NT, P, ROWS, cpp; size_t slot, ring; };
template <typename T, bool WS, int WSG> Geo3Info geo3_g() {
  Geo3Info g;
  geo3_t<T, WS, WSG>(g.TX, g.TY, g.NT, g.slot, g.ring, g.P, g.ROWS);
  g.cpp = tmem_cpp<T, typename GS<T, WS, WSG>::G>();
  return g;
}
template <typename T> Geo3Info geo3(bool ws, int wsg) {
  if (!ws) return geo3_g<T, false, 0>();
  switch (wsg) {
    case 1: return geo3_g<T, true, 1>();
    case 2: return geo3_g<T, true, 2>();
    default: return geo3_g<T, true, 0>();
  }
}
}  // namespace


// Co-resident CTAs per SM from the kernel's registers, threads and shared memory.  The runtime's
// occupancy calculator (and hence a cooperative launch) caps every kernel that contains
// tcgen05.alloc at ONE CTA per SM (profiles/r01_tmem_occupancy_probe.txt: 1 for any smem, while
// the same kernel launched normally runs 2 CTAs per SM, each with its own TMEM allocation), so the
// PERKS kernels — which carry the TMEM tier — compute residency from the hardware limits
// (B200: 64K registers in 4 SMSP files, 2048 threads, 32 CTAs, smem_per_sm incl. 1 KiB/CTA).
int occupancy_ignoring_tmem(const Problem &p, const cudaFuncAttributes &fa, int nt, size_t smem) {
  const int warps = (nt + 31) / 32;
  const int regs_warp = (fa.numRegs * 32 + 255) / 256 * 256;
  int by_regs = 0;  // warps of all CTAs round-robin over 4 SMSPs of 16384 registers each
  for (int b = 1; b <= 32; b++) {
    const int per_smsp = (b * warps + 3) / 4;
    if (per_smsp * regs_warp > 16384) break;
    by_regs = b;
  }
  const int by_threads = 2048 / (warps * 32);
  const size_t per = smem + (size_t)fa.sharedSizeBytes + 1024;
  const int by_smem = (int)((size_t)p.smem_per_sm / per);
  return std::min(std::min(by_regs, by_threads), std::min(by_smem, 32));
}

// Plan (a) host loop, (b) persistent or (c) PERKS for a 3D problem.
Plan plan_stream3d(const Problem &p, perks_variant v) {
  Plan pl;
  pl.variant = v;
  if (p.ndim != 3 || (p.shape != SHAPE_3D7 && p.shape != SHAPE_3D27 && p.shape != SHAPE_3D19) ||
      p.bc != PERKS_BC_FRAME) {
    pl.why = "stream3d: needs 3D 7pt/19pt/27pt FRAME";
    return pl;
  }
  const bool tma = use_tma3(p);
  if (p.nranks > 1 && !tma) { pl.why = "stream3d: multi-GPU slabs need TMA (nx*S % 16 == 0)"; return pl; }
  // PERKS-3D on-chip plane cache (shared memory + TMEM tiers): measured to cost more SM-side time
  // (per-plane halo fetches, perimeter publishes, TMEM staging) than the DRAM/L2 traffic it saves
  // at every 3D size tried on B200, including fully cacheable ones (profiles/r01_perks3d_cache_sweep.txt):
  // the planner's default cache split is empty (D_cache = 0: the PERKS variant runs the persistent
  // kernel, P:519 with D_cache = 0); PERKS_P3D_CACHE=1 enables the tiers.
  const bool cache = v == PERKS_PERKS && env_int("PERKS_P3D_CACHE", 0) != 0;
  if (cache && !tma) { pl.why = "perks3d: needs TMA (nx*S % 16 == 0)"; return pl; }
  const bool persistent = v != PERKS_HOSTLOOP;
  const bool ws = tma && persistent;  // warp-specialised pipeline (persistent kernels)
  // WS geometry: 4 warps x 3 CTAs/SM once one buffer is >= 16 L2 sizes (more plane streams in
  // flight for DRAM-latency-bound streaming), else 8 warps x 2 CTAs/SM
  int wsg = ((double)p.cells() * p.elem() >= 16.0 * (double)p.l2_bytes) ? 1 : 0;
  if (env_int("PERKS_WSG", -1) >= 0) wsg = std::min(std::max(env_int("PERKS_WSG", 0), 0), kNumWsg - 1);
  if (!ws || (p.nranks > 1 && wsg > 1)) wsg = std::min(wsg, ws ? 1 : 0);
  void *k = persistent ? persist_ptr(p, tma, cache, wsg) : pick3(p, false);
  const Geo3Info gi = p.dtype == PERKS_F32 ? geo3<float>(ws, wsg) : geo3<double>(ws, wsg);
  const size_t ring = gi.ring, slot = gi.slot;
  const int TX = gi.TX, TY = gi.TY, NT = gi.NT;
  const int tx = (int)((p.nx + TX - 1) / TX), ty = (int)((p.ny + TY - 1) / TY);
  const int tiles = tx * ty;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  // z chunks: about two waves of units for the host loop; for the persistent kernels the
  // z-chunking that minimises the busiest CTA's planes per step, ceil(units / grid) * (chunk + 2
  // halo planes), with grid <= resident CTAs (load balance over 148 SMs)
  auto choose_nzc = [&](int resident) {
    int nz_c = std::max(1, (2 * resident + tiles - 1) / tiles);
    nz_c = std::min<int>(nz_c, (int)std::max<int64_t>(1, p.nz / 8));
    if (persistent) {
      int64_t best = -1;
      for (int n = 1; n <= std::max<int64_t>(1, p.nz / 4); n++) {
        const int64_t zcn = (p.nz + n - 1) / n, nn = (p.nz + zcn - 1) / zcn;
        if (nn != n) continue;
        const int64_t un = (int64_t)tiles * n, g = std::min<int64_t>(un, resident);
        const int64_t cost = ((un + g - 1) / g) * (zcn + 2);
        if (best < 0 || cost < best) { best = cost; nz_c = n; }
      }
      if (env_int("PERKS_S3D_NZC", 0) > 0) nz_c = std::min<int>(env_int("PERKS_S3D_NZC", 0), (int)p.nz);  // sweeps
    }
    const int zcn = (int)((p.nz + nz_c - 1) / nz_c);
    return (int)((p.nz + zcn - 1) / zcn);
  };
  size_t smem = ring;
  int occ = 0, nc = 0, tcols = 0, ntm0 = 0;
  bool tmem_ok = false;
  const bool use_tmem = env_int("PERKS_P3D_TMEM", 1) != 0;
  if (!cache) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      cudaGetLastError();
      pl.why = "cudaFuncSetAttribute"; return pl;
    }
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem);
    // warp-specialised persistent kernels: the geometry's designed CTAs per SM (more CTAs of the
    // 4-warp geometry measured slower on C5: 3.63 vs 2.90 ms/step, profiles/r01_perks3d_tmem_probe.txt)
    if (ws) occ = std::min(occ, env_int("PERKS_S3D_CPS", wsg_minb(wsg)));
  } else {
    // PERKS: the shared memory the ring leaves at `cps` CTAs per SM caches planes (
    // minimal occupancy that keeps the HBM stream saturated: 2 CTAs/SM measured best)
    const int force_cps = env_int("PERKS_P3D_CPS", 0);
    for (int cps = force_cps > 0 ? force_cps : wsg_minb(wsg); cps >= 1; cps--) {
      const size_t budget = std::min<size_t>((size_t)p.max_smem_optin, (size_t)p.smem_per_sm / cps - 1024);
      // TMEM tier (tmem.cuh): 512 / cps columns per CTA (power of two), gi.cpp per plane
      tcols = 512;
      while (tcols * cps > 512) tcols >>= 1;
      ntm0 = use_tmem ? tcols / gi.cpp : 0;
      if (env_int("PERKS_P3D_NTM", -1) >= 0) ntm0 = std::min(ntm0, env_int("PERKS_P3D_NTM", 0));
      // the CTA's cache-code map: one byte per arrival of its busiest step (+ sentinel)
      const int nzc_c = choose_nzc(cps * p.num_sms);
      const int64_t zc_c = (p.nz + nzc_c - 1) / nzc_c, un_c = (int64_t)tiles * nzc_c;
      const int64_t g_c = std::min<int64_t>(un_c, (int64_t)cps * p.num_sms);
      const size_t map_bytes = align256((size_t)(((un_c + g_c - 1) / g_c) * (zc_c + 2) + 1));
      const size_t fixed = ring + map_bytes;
      nc = budget > fixed ? (int)((budget - fixed) / slot) : 0;
      const int forced = env_int("PERKS_P3D_NSM", -1);
      if (forced >= 0) nc = std::min(nc, forced);
      smem = fixed + (size_t)nc * slot;
      if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      occ = occupancy_ignoring_tmem(p, fa, NT, smem);
      if (env_int("PERKS_DEBUG_PLAN", 0))
        fprintf(stderr, "perks3d plan: cps=%d nc=%d smem=%zu occ=%d regs=%d static_smem=%zu\n", cps, nc, smem, occ,
                fa.numRegs, (size_t)fa.sharedSizeBytes);
      if (occ >= cps) {
        // TMEM tier: every co-resident CTA allocates 512 / cps columns, so exactly cps CTAs may
        // share an SM (more would block in tcgen05.alloc): pad shared memory until no more fit
        while (occ > cps && smem + 1024 <= (size_t)p.max_smem_optin) {
          smem += 1024;
          if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
            cudaGetLastError();
            break;
          }
          occ = occupancy_ignoring_tmem(p, fa, NT, smem);
        }
        if (occ == cps) tmem_ok = true;
        occ = cps;
        break;
      }
    }
  }
  if (occ < 1) { pl.why = "stream3d: not co-resident"; return pl; }
  const int resident = occ * p.num_sms;
  int nzc = choose_nzc(resident);
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
  pl.family = v == PERKS_PERKS ? 2 : 0;  // (2: PERKS 3D, supports multi-GPU slabs)
  pl.cache_kernel = cache;
  pl.wsg = wsg;
  pl.nc = cache ? nc : 0;
  if (cache && tmem_ok && ntm0 > 0) {
    pl.ntm = ntm0;
    pl.tcols = tcols;
  }
  const double S = (double)p.elem();
  // cached cells: per CTA min(nc + ntm, eligible planes of its units) tile planes (the kernel's
  // cache_code_of split: shared memory first, then TMEM)
  int64_t cached = 0, cached_t = 0;
  if (cache) {
    for (int64_t b = 0; b < pl.grid; b++) {
      int64_t E = 0;
      for (int64_t id = b; id < pl.units; id += pl.grid) {
        const int64_t cz = id / tiles, len = std::min<int64_t>(zc, p.nz - cz * zc);
        E += std::max<int64_t>(0, len - 2);
      }
      const int64_t n = std::min<int64_t>(pl.nc + pl.ntm, E), ns = std::min<int64_t>(pl.nc, n);
      cached += ns;
      cached_t += std::min<int64_t>(pl.ntm, n - ns);
    }
    cached *= (int64_t)TX * TY;
    cached_t *= (int64_t)TX * TY;
    cached = std::min<int64_t>(cached, p.cells());
    cached_t = std::min<int64_t>(cached_t, p.cells() - cached);
  }
  pl.cached_smem = cached;
  pl.cached_tmem = cached_t;
  pl.dram_bytes_step = 2.0 * S * ((double)p.cells() - (double)cached - (double)cached_t);
  pl.halo_bytes_step = S * (double)p.nz * (2.0 * TX * ty * tx + 2.0 * TY * ty * tx) +
                       S * 2.0 * nzc * (double)p.nx * p.ny;
  pl.ws_bytes = align256((size_t)p.cells() * p.elem()) + (persistent ? 256 : 0);
  snprintf(pl.name, sizeof(pl.name), "%s3d_%s_%s_t%dx%d_z%d%s",
           v == PERKS_PERKS ? "perks" : persistent ? "persistent" : "hostloop",
           p.shape == SHAPE_3D7 ? "7pt" : p.shape == SHAPE_3D19 ? "19pt" : "27pt", p.dtype == PERKS_F32 ? "f32" : "f64", TX, TY, zc,
           cache ? "_c" : v == PERKS_PERKS ? "_c0" : (pl.cfg ? "_tma" : "_cpasync"));
  if (cache) {
    char extra[24];
    if (pl.ntm > 0) snprintf(extra, sizeof(extra), "%d_t%d_%dcta", pl.nc, pl.ntm, occ);
    else snprintf(extra, sizeof(extra), "%d_%dcta", pl.nc, occ);
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
  Cache3 ch{0, 0, 0};
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
    zigzag = env_int("PERKS_ZIGZAG", 1);  // L2-aware traversal; PERKS_ZIGZAG=0 disables
    smem = (size_t)pl.smem;
    tma = pl.cfg == 1;
    grid = pl.grid;
    in = in_; out = out_; tmp = tmp_; bar = bar_;
    dk = make_distk(dr);
    xbase = dr ? dr->xbase : 0;
    dist = p.nranks > 1;
    cache = pl.cache_kernel;
    ch.nc = pl.nc;
    ch.ntm = pl.ntm;
    ch.tcols = pl.tcols;
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
    cudaError_t e = reset_grid_barrier(bar, s);
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
  // A PERKS plan (its kernel carries the TMEM tier) with several CTAs per SM cannot be launched
  // cooperatively (the
  // runtime caps tcgen05.alloc kernels at one CTA per SM, see occupancy_ignoring_tmem): it is
  // launched normally with a grid of exactly the co-resident capacity computed by the planner
  // (shared memory padded so no further CTA fits an SM), which the block scheduler places all at
  // once on an idle device.  Opt-in only (PERKS_P3D_CACHE=1) and it needs exclusive use of the GPU:
  // a concurrent kernel holding SMs would leave CTAs unscheduled until the watchdog traps.
  const bool tmem_multi = pl.cache_kernel && pl.ctas_per_sm > 1;
  return L.persistent(steps, s, !(dr && dr->noncoop) && !tmem_multi && !env_int("PERKS_NONCOOP", 0));
}
}  // namespace

cudaError_t run_stream3d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws,
                         int64_t steps, cudaStream_t s, const DistRun *dr) {
  if (p.dtype == PERKS_F32)
    return p.shape == SHAPE_3D7    ? run3<float, SHAPE_3D7>(p, pl, in, out, ws, steps, s, dr)
           : p.shape == SHAPE_3D19 ? run3<float, SHAPE_3D19>(p, pl, in, out, ws, steps, s, dr)
                                   : run3<float, SHAPE_3D27>(p, pl, in, out, ws, steps, s, dr);
  return p.shape == SHAPE_3D7    ? run3<double, SHAPE_3D7>(p, pl, in, out, ws, steps, s, dr)
         : p.shape == SHAPE_3D19 ? run3<double, SHAPE_3D19>(p, pl, in, out, ws, steps, s, dr)
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
    return p.shape == SHAPE_3D7    ? group3<float, SHAPE_3D7>(ps, pls, in, out, ws, drs, n, steps, s)
           : p.shape == SHAPE_3D19 ? group3<float, SHAPE_3D19>(ps, pls, in, out, ws, drs, n, steps, s)
                                   : group3<float, SHAPE_3D27>(ps, pls, in, out, ws, drs, n, steps, s);
  return p.shape == SHAPE_3D7    ? group3<double, SHAPE_3D7>(ps, pls, in, out, ws, drs, n, steps, s)
         : p.shape == SHAPE_3D19 ? group3<double, SHAPE_3D19>(ps, pls, in, out, ws, drs, n, steps, s)
                                 : group3<double, SHAPE_3D27>(ps, pls, in, out, ws, drs, n, steps, s);
}

}  // namespace perks
