// k3d_perks.cu — variant (c) PERKS for 3D stencils: persistent plane streaming with an on-chip
// plane cache and zig-zag (L2-aware) traversal.
//
// The time loop runs inside one persistent launch with a device-wide barrier per step (Fig. 3
// right; grid.sync P:1068).  Work = xy tile x z-plane "plane-tiles"; the tiles x nz
// plane-tiles are split into exactly `grid` contiguous runs (one per CTA, CPS CTAs per SM, so all
// 148 SMs stay busy whatever the tile count), each run being 1-2 z-segments of a tile column.
// "2D planes are loaded one after the other in shared memory, and each thread computes the cells
// in a vertical direction": planes arrive through a TMA ring; output plane o is computed
// when planes o-1, o, o+1 are resident, with the canonical FMA chain (reading R5) — so results are
// bit-identical to variants (a)/(b) and the oracle in either traversal direction.
//
// Caching (§3.3, Fig. 6 Source/Destination switch P:1056-1064): each CTA keeps
// `nc` interior planes of its longest segment resident in shared memory for all steps, spread
// evenly through the segment so the HBM stream never pauses.  A cached plane reloads only its
// one-cell halo ring ("planes that already have the data cached from the previous time step do not
// load from global memory"; halo cells are never cached) and publishes only its
// tile perimeter to the global buffer (TB-boundary cells "continue to store and load from global
// memory").  The first/last plane of every segment is never cached, so z-halo planes other
// segments read are always in global memory.
//
// Zig-zag traversal ([draft] P:395-404, "zig-zag ... caching" for "future GPUs designs with large
// capacity L2"): even steps stream every segment upward, odd steps downward (and the CTA's
// segments in reverse order), so the planes written last in step t — still in the 126 MB L2 — are
// the first ones read in step t+1.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "internal.h"
#include "stream3d.cuh"

#ifndef PERKS_P3_NS
#define PERKS_P3_NS 4     // ring slots (NS-1 planes in flight)
#endif
#ifndef PERKS_P3_R
#define PERKS_P3_R 2      // rows per thread
#endif
#ifndef PERKS_P3_NWARP
#define PERKS_P3_NWARP 8
#endif
#ifndef PERKS_P3_CPS
#define PERKS_P3_CPS 2    // CTAs per SM
#endif

namespace perks {

template <typename T> struct GP3 {
  using G = Geo3D<T, 16 / (int)sizeof(T), PERKS_P3_R, PERKS_P3_NWARP, PERKS_P3_NS>;
};
constexpr int KP3_THREADS = 32 * PERKS_P3_NWARP;

bool use_tma3(const Problem &p);
bool make_maps3(const Problem &p, int P, int ROWS, const void *in, const void *out, const void *tmp,
                Maps3 *m, const void *ghost);
Dom3 make_dom3(const Problem &p);
DistK make_distk(const DistRun *dr);

struct P3Work {
  int tx, ty;            // xy tiles
  long long W;           // plane-tiles = tx * ty * nz
  int nc;                // shared-memory cache slots per CTA
  int k;                 // sub-runs ("units") per CTA: the granularity of the zig-zag order
  int zigzag;            // 1 = reverse the unit order every other step
};

// The pieces of a CTA's plane-tile run [lo, hi) (in (tile, z) order): cut at tile-column
// boundaries and at the k equal sub-run boundaries.  Returns the piece count; fills piece idx.
PERKS_DEVINL int run_pieces(long long lo, long long hi, int nz, int k, int idx, int &tile, int &zs,
                            int &ze) {
  int n = 0, i = 1;
  long long pos = lo;
  while (pos < hi) {
    long long sb = lo + (long long)i * (hi - lo) / k;
    while (sb <= pos && i < k) sb = lo + (long long)(++i) * (hi - lo) / k;
    if (sb <= pos) sb = hi;
    const long long tb = (pos / nz + 1) * nz;
    const long long end = min(min(sb, tb), hi);
    if (n == idx) {
      tile = (int)(pos / nz);
      zs = (int)(pos % nz);
      ze = (int)(zs + (end - pos));
    }
    n++;
    pos = end;
  }
  return n;
}

template <typename T, int S, bool DIST>
__global__ void __launch_bounds__(KP3_THREADS, DIST ? 1 : PERKS_P3_CPS) perks3d_kernel(
    const T *__restrict__ in, T *out, T *tmp, const __grid_constant__ Maps3 maps, Dom3 d, P3Work w,
    int64_t steps, unsigned *bar, Coef<T, Shape<S>::N> c, const __grid_constant__ DistK dk,
    unsigned long long xbase) {
  using G = typename GP3<T>::G;
  constexpr int NS = G::NS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T *ring_slots = reinterpret_cast<T *>(smem_raw);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)NS * G::SLOT_BYTES);
  T *cache = reinterpret_cast<T *>(smem_raw + (size_t)NS * G::SLOT_BYTES + 128);
  short *cmap = reinterpret_cast<short *>(cache + (size_t)w.nc * G::SLOT);
  Ring<T, G, true> ring;
  ring.init(ring_slots, bars, 2 * G::TY);

  const long long lo = (long long)blockIdx.x * w.W / gridDim.x;
  const long long hi = (long long)(blockIdx.x + 1) * w.W / gridDim.x;
  int tl, zs, ze;
  const int np = run_pieces(lo, hi, d.nz, w.k, -1, tl, zs, ze);
  // the cached piece = the CTA's longest; nc slots spread evenly over its interior planes (the
  // first/last plane of every piece is never cached: other pieces read them as z-halo)
  int cpiece = 0, clen = -1;
  for (int i = 0; i < np; i++) {
    run_pieces(lo, hi, d.nz, w.k, i, tl, zs, ze);
    if (ze - zs > clen) { clen = ze - zs; cpiece = i; }
  }
  int ctile, czs, cze;
  run_pieces(lo, hi, d.nz, w.k, cpiece, ctile, czs, cze);
  const int elig = max(0, cze - czs - 2);
  const int nc = min(w.nc, elig);
  for (int j = threadIdx.x; j < cze - czs; j += blockDim.x) {
    const int jj = j - 1;
    int v = -1;
    if (nc > 0 && jj >= 0 && jj < elig) {
      const int a = (jj * nc) / elig, b = ((jj + 1) * nc) / elig;
      v = b != a ? a : -1;
    }
    cmap[j] = (short)v;
  }
  __syncthreads();
  const CacheView<T> cv{cache, cmap, czs, cze};
  const int cx0 = (ctile % w.tx) * G::TX, cy0 = (ctile / w.tx) * G::TY;

  // ---- prologue: cached planes from `in` (one-time load half of 2·D_cache)
  for (int q = czs + 1; q < cze - 1; q++) {
    const int sl = cmap[q - czs];
    if (sl >= 0) issue_plane<T, G>(cache + (size_t)sl * G::SLOT, in, d, q, cx0, cy0, false);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  const unsigned long long plane_cells = (unsigned long long)d.nx * d.ny;
  for (int64_t t = 0; t < steps; t++) {
    const bool src_out = t > 0 && ((steps - t) & 1) == 0;
    const T *src = t == 0 ? in : (src_out ? out : tmp);
    const int si = t == 0 ? 0 : (src_out ? 1 : 2);
    T *dst = ((steps - 1 - t) & 1) == 0 ? out : tmp;
    const CUtensorMap *boxmap = &maps.box[si];
    const DistStep ds{&dk, &maps.ghost, xbase + (unsigned long long)t, plane_cells};
    const bool rev = w.zigzag && (t & 1);
    if (threadIdx.x == 0) fence_proxy_async_global();  // last step's generic stores -> TMA reads
    for (int i = 0; i < np; i++) {
      const int idx = rev ? np - 1 - i : i;
      run_pieces(lo, hi, d.nz, w.k, idx, tl, zs, ze);
      const int x0 = (tl % w.tx) * G::TX, y0 = (tl / w.tx) * G::TY;
      __syncthreads();  // the previous piece's ring slots are free
      if (idx == cpiece)
        stream_unit<T, S, G, true, DIST, true>(ring, src, boxmap, dst, d, x0, y0, zs, ze, c, ds, true, cv);
      else
        stream_unit<T, S, G, true, DIST, false>(ring, src, boxmap, dst, d, x0, y0, zs, ze, c, ds, true);
    }
    if (t + 1 < steps) grid_barrier(bar, (unsigned)((t + 1) * gridDim.x));
  }

  // ---- epilogue: cached planes to `out` (store half of 2·D_cache); the last step's dst is out
  __syncthreads();
  ThreadTile<G> ct;
  ct.init(d, cx0, cy0);
  for (int q = czs + 1; q < cze - 1; q++) {
    const int sl = cmap[q - czs];
    if (sl < 0) continue;
    T v[G::R][G::V];
    read_own<T, G>(cache + (size_t)sl * G::SLOT, v);
    store_cells<T, G>(out, d, ct, q, v);
  }
}

// ------------------------------------------------------------------ host side
namespace {
template <typename T> void *kp3(int shape, bool dist) {
  if (shape == SHAPE_3D7) return dist ? (void *)perks3d_kernel<T, SHAPE_3D7, true> : (void *)perks3d_kernel<T, SHAPE_3D7, false>;
  return dist ? (void *)perks3d_kernel<T, SHAPE_3D27, true> : (void *)perks3d_kernel<T, SHAPE_3D27, false>;
}
void *kp3p(const Problem &p) {
  const bool dist = p.nranks > 1;
  return p.dtype == PERKS_F32 ? kp3<float>(p.shape, dist) : kp3<double>(p.shape, dist);
}
struct P3Geo {
  int TX, TY, NT, P, ROWS, NS;
  size_t slot_bytes;
};
template <typename T> P3Geo p3geo() {
  using G = typename GP3<T>::G;
  return P3Geo{G::TX, G::TY, G::NT, G::P, G::ROWS, G::NS, G::SLOT_BYTES};
}
P3Geo p3geo_of(const Problem &p) { return p.dtype == PERKS_F32 ? p3geo<float>() : p3geo<double>(); }

// cached plane-tiles of the whole grid (host replica of the kernel's piece logic)
int64_t cached_planes(const P3Work &w, int nz, int grid) {
  int64_t tot = 0;
  for (int cta = 0; cta < grid; cta++) {
    const long long lo = (long long)cta * w.W / grid, hi = (long long)(cta + 1) * w.W / grid;
    int best = 0, i = 1;
    long long pos = lo;
    while (pos < hi) {
      long long sb = lo + (long long)i * (hi - lo) / w.k;
      while (sb <= pos && i < w.k) sb = lo + (long long)(++i) * (hi - lo) / w.k;
      if (sb <= pos) sb = hi;
      const long long end = std::min(std::min(sb, (pos / nz + 1) * nz), hi);
      best = std::max(best, (int)(end - pos));
      pos = end;
    }
    tot += std::min(w.nc, std::max(0, best - 2));
  }
  return tot;
}
}  // namespace

Plan plan_perks3d(const Problem &p) {
  Plan pl;
  pl.variant = PERKS_PERKS;
  if (p.ndim != 3 || (p.shape != SHAPE_3D7 && p.shape != SHAPE_3D27) || p.bc != PERKS_BC_FRAME) {
    pl.why = "perks3d: needs 3D 7pt/27pt FRAME";
    return pl;
  }
  if (!use_tma3(p)) { pl.why = "perks3d: needs TMA (nx*S % 16 == 0)"; return pl; }
  const P3Geo g = p3geo_of(p);
  void *k = kp3p(p);
  const int cps = PERKS_P3_CPS;
  P3Work w{};
  w.tx = (int)((p.nx + g.TX - 1) / g.TX);
  w.ty = (int)((p.ny + g.TY - 1) / g.TY);
  w.W = (long long)w.tx * w.ty * p.nz;
  w.zigzag = env_int("PERKS_ZIGZAG", 1) ? 1 : 0;
  w.k = w.zigzag ? std::max(1, env_int("PERKS_P3D_K", 2)) : 1;
  int grid = (int)std::min<long long>(w.W, (long long)cps * p.num_sms);
  // cache budget: the shared memory the ring leaves (CPS CTAs per SM)
  const size_t cmap_bytes = align256((size_t)p.nz * sizeof(short));
  const size_t ring = (size_t)g.NS * g.slot_bytes + 128 + cmap_bytes;
  const size_t per_cta = std::min<size_t>((size_t)p.max_smem_optin, (size_t)p.smem_per_sm / cps - 1024);
  int nc = per_cta > ring ? (int)((per_cta - ring) / g.slot_bytes) : 0;
  const int forced = env_int("PERKS_P3D_NSM", -1);
  if (forced >= 0) nc = std::min(nc, forced);
  w.nc = nc;
  const size_t smem = ring + (size_t)nc * g.slot_bytes;
  if (ring > per_cta) { pl.why = "perks3d: nz too large for the plane map"; return pl; }
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    pl.why = "cudaFuncSetAttribute"; return pl;
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, g.NT, smem);
  if (occ < 1) { pl.why = "perks3d: not co-resident"; return pl; }
  grid = std::min(grid, occ * p.num_sms);  // (the multi-GPU build may fit fewer CTAs per SM)
  pl.grid = grid;
  pl.block = g.NT;
  pl.ctas_per_sm = std::min(cps, occ);
  pl.tile[0] = g.TX; pl.tile[1] = g.TY; pl.tile[2] = (int)((w.W + grid - 1) / grid);
  pl.regs = fa.numRegs;
  pl.smem = (int)smem;
  pl.units = grid;
  pl.cfg = (w.k << 17) | (w.zigzag << 16) | nc;
  pl.family = 2;  // supports multi-GPU slabs
  const int64_t cplanes = cached_planes(w, (int)p.nz, grid);
  pl.cached_reg = 0;
  pl.cached_smem = std::min<int64_t>(cplanes * g.TX * g.TY, p.cells());
  const double S = (double)p.elem();
  pl.dram_bytes_step = 2.0 * S * ((double)p.cells() - (double)pl.cached_smem);
  pl.halo_bytes_step = S * (double)cplanes * 2.0 * 2.0 * (g.TX + g.TY);
  pl.ws_bytes = align256((size_t)p.cells() * p.elem()) + 256;
  snprintf(pl.name, sizeof(pl.name), "perks3d_%s_%s_t%dx%d_c%d_s%d_k%d%s", p.shape == SHAPE_3D7 ? "7pt" : "27pt",
           p.dtype == PERKS_F32 ? "f32" : "f64", g.TX, g.TY, pl.ctas_per_sm, nc, w.k, w.zigzag ? "_zz" : "");
  pl.ok = true;
  return pl;
}

template <typename T, int S>
static cudaError_t launch_p3(const Problem &p, const Plan &pl, const T *in, T *out, void *ws,
                             int64_t steps, cudaStream_t s, const DistRun *dr) {
  const P3Geo g = p3geo<T>();
  Coef<T, Shape<S>::N> c;
  for (int i = 0; i < Shape<S>::N; i++) c.w[i] = sizeof(T) == 4 ? (T)p.wf[i] : (T)p.wd[i];
  Dom3 d = make_dom3(p);
  P3Work w{};
  w.tx = (int)((p.nx + g.TX - 1) / g.TX);
  w.ty = (int)((p.ny + g.TY - 1) / g.TY);
  w.W = (long long)w.tx * w.ty * p.nz;
  w.nc = pl.cfg & 0xffff;
  w.zigzag = (pl.cfg >> 16) & 1;
  w.k = pl.cfg >> 17;
  T *tmp = (T *)ws;
  unsigned *bar = (unsigned *)((char *)ws + align256((size_t)p.cells() * p.elem()));
  Maps3 maps;
  std::memset(&maps, 0, sizeof(maps));
  if (!make_maps3(p, g.P, g.ROWS, in, out, tmp, &maps, dr ? dr->ghost : nullptr)) return cudaErrorInvalidValue;
  DistK dk = make_distk(dr);
  unsigned long long xbase = dr ? dr->xbase : 0;
  cudaError_t e = cudaMemsetAsync(bar, 0, 256, s);
  if (e != cudaSuccess) return e;
  if (dr && (e = launch_dist_prologue(p, in, *dr, s)) != cudaSuccess) return e;
  void *k = kp3p(p);
  void *args[] = {(void *)&in, (void *)&out, (void *)&tmp, (void *)&maps, (void *)&d, (void *)&w,
                  (void *)&steps, (void *)&bar, (void *)&c, (void *)&dk, (void *)&xbase};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(g.NT);
  cfg.dynamicSmemBytes = (size_t)pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = (dr && dr->noncoop) ? 0 : 1;
  return cudaLaunchKernelExC(&cfg, k, args);
}

cudaError_t run_perks3d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws,
                        int64_t steps, cudaStream_t s, const DistRun *dr) {
  if (p.dtype == PERKS_F32) {
    if (p.shape == SHAPE_3D7) return launch_p3<float, SHAPE_3D7>(p, pl, (const float *)in, (float *)out, ws, steps, s, dr);
    return launch_p3<float, SHAPE_3D27>(p, pl, (const float *)in, (float *)out, ws, steps, s, dr);
  }
  if (p.shape == SHAPE_3D7) return launch_p3<double, SHAPE_3D7>(p, pl, (const double *)in, (double *)out, ws, steps, s, dr);
  return launch_p3<double, SHAPE_3D27>(p, pl, (const double *)in, (double *)out, ws, steps, s, dr);
}

}  // namespace perks
