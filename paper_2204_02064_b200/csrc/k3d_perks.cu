// k3d_perks.cu — variant (c) PERKS for 3D stencils: partially cached plane streaming.
//
// The baseline's plane-streaming body (stream3d.cuh, "2D planes are loaded one after the other in
// shared memory") runs inside one persistent cooperative launch with a grid barrier per
// step (Fig. 3 right).  Each CTA (1 per SM) owns a fixed unit = xy tile x z-chunk for all
// steps and keeps some of the unit's planes resident across steps:
//   * REG planes   — the thread's V x R cells of NRP planes in registers (reg_cache, Fig. 6);
//   * SMEM planes  — whole tile planes (with their halo ring) in shared memory (sm_cache);
//   * GLOBAL planes— everything else, streamed from/to HBM every step exactly as in (a)/(b).
// "Planes that already have the data cached from the previous time step do not load from global
// memory": a cached plane only fetches its one-cell halo ring (halo cells are never cached,
// P:348-355), and its new values stay on chip; only its tile perimeter is written back each step so
// neighbouring tiles can read it as their halo (the TB-boundary cells "continue to store and load
// from global memory").  The first and last plane of every unit are never cached, so the
// z-halo planes other units read are always in global memory.  DRAM bytes per step:
// 2·S·(cells - cached) + perimeter traffic (A_gm).
//
// Concurrency: with one CTA per SM, the ring must keep ~B_gm/148 x latency ~ 44 KB of
// planes in flight, so the ring is NS = 8 slots deep; the remaining shared memory caches planes.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "internal.h"
#include "stream3d.cuh"

#ifndef PERKS_P3D_NS
#define PERKS_P3D_NS 5
#endif
#ifndef PERKS_P3D_R
#define PERKS_P3D_R 4
#endif
#ifndef PERKS_P3D_NWARP
#define PERKS_P3D_NWARP 8
#endif
#ifndef PERKS_P3D_NRP
#define PERKS_P3D_NRP 4
#endif
#ifndef PERKS_P3D_MINB
#define PERKS_P3D_MINB 1
#endif

namespace perks {

template <typename T> struct GP3Sel;
template <> struct GP3Sel<float> {
  using G = Geo3D<float, 4, PERKS_P3D_R, PERKS_P3D_NWARP, PERKS_P3D_NS>;
  static constexpr int NRP = PERKS_P3D_NRP;
};
template <> struct GP3Sel<double> {
  using G = Geo3D<double, 2, PERKS_P3D_R, PERKS_P3D_NWARP, PERKS_P3D_NS>;
  static constexpr int NRP = PERKS_P3D_NRP;
};
constexpr int KP3_THREADS = 32 * PERKS_P3D_NWARP;

bool use_tma3(const Problem &p);
bool make_maps3(const Problem &p, int P, int ROWS, const void *in, const void *out, const void *tmp,
                Maps3 *m, const void *ghost);
Dom3 make_dom3(const Problem &p);

struct P3Units {
  int tx, ty, nzc, zc;  // tiles in x/y, z-chunks, planes per chunk
  int nsm;              // SMEM planes cached in the CTA's first unit
  int nreg;             // REG planes cached (0 or NRP)
};

// Publish the tile-perimeter cells of a cached plane o to dst (so neighbours' halo rings read the
// current values next step) — only threads owning perimeter cells store.
template <typename T, class G>
PERKS_DEVINL void publish_perimeter(T *__restrict__ dst, const Dom3 &d, int o, int x0, int y0,
                                    const T (&v)[G::R][G::V]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x = x0 + lane * G::V;
  T *base = dst + (size_t)o * d.nx * d.ny;
  const int xl = min(x0 + G::TX, d.nx) - 1;  // last tile column inside the domain
#pragma unroll
  for (int r = 0; r < G::R; r++) {
    const int y = y0 + warp * G::R + r;
    if (y >= d.ny) break;
    const bool edge_row = (warp == 0 && r == 0) || (warp == G::NWARP - 1 && r == G::R - 1) ||
                          y == d.ny - 1;
    if (edge_row) {
#pragma unroll
      for (int i = 0; i < G::V; i++)
        if (x + i < d.nx) base[(size_t)y * d.nx + x + i] = v[r][i];
    } else {
      if (lane == 0 && x < d.nx) base[(size_t)y * d.nx + x] = v[r][0];
      if (xl >= x && xl < x + G::V) {
#pragma unroll
        for (int i = 0; i < G::V; i++)
          if (x + i == xl) base[(size_t)y * d.nx + x + i] = v[r][i];
      }
    }
  }
}

// Thread's V x R interior cells of a slot <-> registers.
template <typename T, class G>
PERKS_DEVINL void slot_put(T *slot, const T (&v)[G::R][G::V]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < G::R; r++)
    vstore<T, G::V>(slot + (warp * G::R + r + 1) * G::P + G::PAD + lane * G::V, v[r]);
}
template <typename T, class G>
PERKS_DEVINL void slot_get(const T *slot, T (&v)[G::R][G::V]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < G::R; r++)
    vload<T, G::V>(v[r], slot + (warp * G::R + r + 1) * G::P + G::PAD + lane * G::V);
}
template <typename T, class G>
PERKS_DEVINL void copy_cells(T (&a)[G::R][G::V], const T (&b)[G::R][G::V]) {
#pragma unroll
  for (int r = 0; r < G::R; r++)
#pragma unroll
    for (int i = 0; i < G::V; i++) a[r][i] = b[r][i];
}

template <typename T, int S, bool TMA>
__global__ void __launch_bounds__(KP3_THREADS, PERKS_P3D_MINB) perks3d_kernel(
    const T *__restrict__ in, T *out, T *tmp, const __grid_constant__ Maps3 maps, Dom3 d,
    P3Units u, int64_t steps, unsigned *bar, Coef<T, Shape<S>::N> c) {
  using G = typename GP3Sel<T>::G;
  constexpr int NRP = GP3Sel<T>::NRP;
  constexpr int NS = G::NS, D = NS - 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T *ring_slots = reinterpret_cast<T *>(smem_raw);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)NS * G::SLOT_BYTES);
  T *smc = reinterpret_cast<T *>(smem_raw + (size_t)NS * G::SLOT_BYTES + 128);  // SMEM planes
  const int nunits = u.tx * u.ty * u.nzc;
  Ring<T, G, TMA> ring;
  ring.init(ring_slots, bars, TMA ? 2 * G::TY : 0);

  // the CTA's first unit (the cached one)
  const int t0 = blockIdx.x % (u.tx * u.ty), zc0 = blockIdx.x / (u.tx * u.ty);
  const int x0 = (t0 % u.tx) * G::TX, y0 = (t0 / u.tx) * G::TY;
  const int zs = zc0 * u.zc, ze = min(zs + u.zc, d.nz);
  const int len = ze - zs;                         // the last chunk may be shorter
  const int zr0 = zs + 1;                          // first REG plane
  const int nreg = (len - 2 >= NRP) ? u.nreg : 0;  // 0 or NRP
  const int zm0 = zr0 + nreg;                      // first SMEM plane
  const int nsm = min(u.nsm, max(0, len - 2 - nreg));
  auto kind = [&](int q) { return (q >= zr0 && q < zr0 + nreg) ? 1 : (q >= zm0 && q < zm0 + nsm) ? 2 : 0; };
  auto smbuf = [&](int q) { return smc + (size_t)(q - zm0) * G::SLOT; };
  ThreadTile<G> tt;
  tt.init(d, x0, y0);

  T reg[NRP > 0 ? NRP : 1][G::R][G::V];
  // ---- prologue: cached planes from `in` (one-time load half of 2·D_cache)
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x = x0 + lane * G::V;
#pragma unroll
    for (int j = 0; j < NRP; j++) {
#pragma unroll
      for (int r = 0; r < G::R; r++) {
        const int y = y0 + warp * G::R + r;
#pragma unroll
        for (int i = 0; i < G::V; i++)
          reg[j][r][i] = (j < nreg && y < d.ny && x + i < d.nx)
                             ? in[((size_t)(zr0 + j) * d.ny + y) * d.nx + x + i] : T(0);
      }
    }
    for (int q = zm0; q < zm0 + nsm; q++) issue_plane<T, G>(smbuf(q), in, d, q, x0, y0, false);
    cp_async_commit();
    cp_async_wait<0>();
  }
  __syncthreads();

  for (int64_t t = 0; t < steps; t++) {
    const bool src_out = t > 0 && ((steps - t) & 1) == 0;
    const T *src = t == 0 ? in : (src_out ? out : tmp);
    const int si = t == 0 ? 0 : (src_out ? 1 : 2);
    T *dst = ((steps - 1 - t) & 1) == 0 ? out : tmp;
    const CUtensorMap *boxmap = &maps.box[si];
    {
      const int q0 = zs - 1, narr = len + 2;
      const unsigned k0 = ring.gk;
      auto slot_of = [&](int k) -> T * {
        const int q = q0 + k;
        return kind(q) == 2 ? smbuf(q) : ring.slot(k0 + k);
      };
      auto issue = [&](int k) {
        if (k < narr) {
          const int q = q0 + k;
          if (kind(q) == 0) ring.issue_full(k0 + k, src, boxmap, d, q, x0, y0, true);
          else ring.issue_halo(k0 + k, slot_of(k), src, d, q, x0, y0);
        } else {
          ring.issue_none();
        }
      };
      // output plane o (finished at arrival o+1): GLOBAL -> store; cached -> stays on chip
      auto store_out = [&](int o, T (&val)[G::R][G::V], const T (&old)[G::R][G::V]) {
        frame_select<T, G>(d, tt, o, val, old);
        const int kd = kind(o);
        if (kd == 0) {
          store_cells<T, G>(dst, d, tt, o, val);
        } else {
          publish_perimeter<T, G>(dst, d, o, x0, y0, val);
          if (kd == 2) slot_put<T, G>(smbuf(o), val);
        }
      };
      for (int k = 0; k < D; k++) issue(k);
      StreamState<T, G> st;
      st.zero();
      auto step_arrival = [&](int k, T (&outv)[G::R][G::V], T (&cq)[G::R][G::V]) {
        ring.wait(k0 + k);
        issue(k + D);
        arrival<T, S, G>(st, slot_of(k), c, outv, cq);
      };
      int k = 0;
      // phase A: arrivals zs-1 and zs (never cached); they finish no output of this unit
      for (; k < 2; k++) {
        T outv[G::R][G::V], cq[G::R][G::V];
        step_arrival(k, outv, cq);
        if (nreg > 0 && k == 1) slot_put<T, G>(ring.slot(k0 + 2), reg[0]);
        copy_cells<T, G>(st.cm1, cq);
      }
      if (NRP > 0 && nreg > 0) {
        // phase B: REG planes j = 0..NRP-1 (arrival k = 2 + j), statically indexed
#pragma unroll
        for (int j = 0; j < NRP; j++) {
          T outv[G::R][G::V], cq[G::R][G::V];
          step_arrival(2 + j, outv, cq);
          if (j == 0) {
            store_out(zs, outv, st.cm1);  // plane zs is GLOBAL
          } else {
            frame_select<T, G>(d, tt, zr0 + j - 1, outv, st.cm1);
            publish_perimeter<T, G>(dst, d, zr0 + j - 1, x0, y0, outv);
            copy_cells<T, G>(reg[j > 0 ? j - 1 : 0], outv);
          }
          if (j + 1 < NRP) slot_put<T, G>(ring.slot(k0 + 3 + j), reg[j + 1 < NRP ? j + 1 : 0]);
          copy_cells<T, G>(st.cm1, cq);
        }
        // phase C: the arrival after the last REG plane finishes REG plane NRP-1
        {
          k = 2 + NRP;
          T outv[G::R][G::V], cq[G::R][G::V];
          step_arrival(k, outv, cq);
          frame_select<T, G>(d, tt, zr0 + NRP - 1, outv, st.cm1);
          publish_perimeter<T, G>(dst, d, zr0 + NRP - 1, x0, y0, outv);
          copy_cells<T, G>(reg[NRP > 0 ? NRP - 1 : 0], outv);
          copy_cells<T, G>(st.cm1, cq);
          k++;
        }
      }
      // phase D: SMEM and GLOBAL arrivals
      for (; k < narr; k++) {
        T outv[G::R][G::V], cq[G::R][G::V];
        step_arrival(k, outv, cq);
        store_out(q0 + k - 1, outv, st.cm1);
        copy_cells<T, G>(st.cm1, cq);
      }
      ring.gk = k0 + narr;
      ring.drain();
    }
    // further (uncached) units of this CTA, if the tile count exceeds the grid
    for (int id = blockIdx.x + gridDim.x; id < nunits; id += gridDim.x) {
      const int tt2 = id % (u.tx * u.ty), zc = id / (u.tx * u.ty);
      const int ux0 = (tt2 % u.tx) * G::TX, uy0 = (tt2 / u.tx) * G::TY;
      const int uzs = zc * u.zc, uze = min(uzs + u.zc, d.nz);
      __syncthreads();
      stream_unit<T, S, G, TMA, false>(ring, src, boxmap, dst, d, ux0, uy0, uzs, uze, c, DistStep{}, true);
    }
    if (t + 1 < steps) grid_barrier(bar, (unsigned)((t + 1) * gridDim.x));
  }

  // ---- epilogue: cached planes to `out` (store half of 2·D_cache).  The last step's dst is out.
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NRP; j++)
    if (j < nreg) store_cells<T, G>(out, d, tt, zr0 + j, reg[j]);
  for (int q = zm0; q < zm0 + nsm; q++) {
    T v[G::R][G::V];
    slot_get<T, G>(smbuf(q), v);
    store_cells<T, G>(out, d, tt, q, v);
  }
}

// ------------------------------------------------------------------ host side
namespace {
template <typename T> void *kp3(int shape, bool tma) {
  if (shape == SHAPE_3D7) return tma ? (void *)perks3d_kernel<T, SHAPE_3D7, true> : (void *)perks3d_kernel<T, SHAPE_3D7, false>;
  if (shape == SHAPE_3D27) return tma ? (void *)perks3d_kernel<T, SHAPE_3D27, true> : (void *)perks3d_kernel<T, SHAPE_3D27, false>;
  return nullptr;
}
struct P3Geo {
  int TX, TY, NT, NRP, V, R, P, ROWS;
  size_t slot_bytes;
  int NS;
};
template <typename T> P3Geo p3geo() {
  using G = typename GP3Sel<T>::G;
  return P3Geo{G::TX, G::TY, G::NT, GP3Sel<T>::NRP, G::V, G::R, G::P, G::ROWS, G::SLOT_BYTES, G::NS};
}
}  // namespace

static void p3_units(const Problem &p, const P3Geo &g, int grid_max, P3Units &u) {
  u.tx = (int)((p.nx + g.TX - 1) / g.TX);
  u.ty = (int)((p.ny + g.TY - 1) / g.TY);
  const int tiles = u.tx * u.ty;
  // units = tiles x z-chunks with all chunks in lockstep z phase (neighbour halos hit L2); at most
  // one cached unit per CTA (units beyond the grid are streamed by the same CTAs, uncached)
  int nzc = std::max(1, grid_max / std::max(1, tiles));
  nzc = std::min<int>(nzc, (int)std::max<int64_t>(1, p.nz / 8));
  u.zc = (int)((p.nz + nzc - 1) / nzc);
  u.nzc = (int)((p.nz + u.zc - 1) / u.zc);
}

Plan plan_perks3d(const Problem &p) {
  Plan pl;
  pl.variant = PERKS_PERKS;
  if (p.ndim != 3 || (p.shape != SHAPE_3D7 && p.shape != SHAPE_3D27) || p.bc != PERKS_BC_FRAME) {
    pl.why = "perks3d: needs 3D 7pt/27pt FRAME";
    return pl;
  }
  const bool tma = use_tma3(p);
  const P3Geo g = p.dtype == PERKS_F32 ? p3geo<float>() : p3geo<double>();
  void *k = p.dtype == PERKS_F32 ? kp3<float>(p.shape, tma) : kp3<double>(p.shape, tma);
  P3Units u{};
  const int cps = PERKS_P3D_MINB;  // CTAs per SM
  p3_units(p, g, cps * p.num_sms, u);
  const int units = u.tx * u.ty * u.nzc;
  const int grid = std::min(units, cps * p.num_sms);
  // cache budget: whatever shared memory the ring leaves (one CTA per SM); REG planes if the chunk
  // has room after its first and last (never cached) planes
  const int eligible = std::max(0, u.zc - 2);
  const int forced_nsm = env_int("PERKS_P3D_NSM", -1);
  u.nreg = (eligible >= g.NRP && env_int("PERKS_P3D_NOREG", 0) == 0) ? g.NRP : 0;
  const size_t ring = (size_t)g.NS * g.slot_bytes + 128;
  const size_t per_cta = std::min<size_t>((size_t)p.max_smem_optin, (size_t)p.smem_per_sm / cps - 1024);
  int nsm = (int)((per_cta - ring) / g.slot_bytes);
  nsm = std::max(0, std::min(nsm, eligible - u.nreg));
  if (forced_nsm >= 0) nsm = std::min(nsm, forced_nsm);
  u.nsm = nsm;
  const size_t smem = ring + (size_t)nsm * g.slot_bytes;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    pl.why = "cudaFuncSetAttribute"; return pl;
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, g.NT, smem);
  if (occ < cps) { pl.why = "perks3d: not co-resident"; return pl; }
  pl.grid = grid;
  pl.block = g.NT;
  pl.ctas_per_sm = cps;
  pl.tile[0] = g.TX; pl.tile[1] = g.TY; pl.tile[2] = u.zc;
  pl.regs = fa.numRegs;
  pl.smem = (int)smem;
  pl.units = units;
  pl.zchunk = u.zc;
  pl.cfg = (tma ? (1 << 30) : 0) | (u.nreg << 16) | u.nsm;
  const int64_t plane_cells = (int64_t)g.TX * g.TY;  // per cached plane (tile, incl. padding)
  const int cached_units = std::min(units, grid);
  pl.cached_reg = (int64_t)cached_units * u.nreg * plane_cells;
  pl.cached_smem = (int64_t)cached_units * u.nsm * plane_cells;
  const double S = (double)p.elem();
  const double cached = std::min<double>((double)(pl.cached_reg + pl.cached_smem), (double)p.cells());
  pl.dram_bytes_step = 2.0 * S * ((double)p.cells() - cached);
  pl.halo_bytes_step = S * (double)cached_units * (u.nreg + u.nsm) * 2.0 * 2.0 * (g.TX + g.TY);
  pl.ws_bytes = align256((size_t)p.cells() * p.elem()) + 256;
  snprintf(pl.name, sizeof(pl.name), "perks3d_%s_%s_t%dx%d_z%d_r%d_s%d%s", p.shape == SHAPE_3D7 ? "7pt" : "27pt",
           p.dtype == PERKS_F32 ? "f32" : "f64", g.TX, g.TY, u.zc, u.nreg, u.nsm, tma ? "_tma" : "");
  pl.ok = true;
  return pl;
}

template <typename T, int S>
static cudaError_t launch_p3(const Problem &p, const Plan &pl, const T *in, T *out, void *ws,
                             int64_t steps, cudaStream_t s) {
  const P3Geo g = p3geo<T>();
  Coef<T, Shape<S>::N> c;
  for (int i = 0; i < Shape<S>::N; i++) c.w[i] = sizeof(T) == 4 ? (T)p.wf[i] : (T)p.wd[i];
  Dom3 d = make_dom3(p);
  P3Units u{};
  p3_units(p, g, PERKS_P3D_MINB * p.num_sms, u);
  const bool tma = (pl.cfg >> 30) & 1;
  u.nreg = (pl.cfg >> 16) & 0x3fff;
  u.nsm = pl.cfg & 0xffff;
  T *tmp = (T *)ws;
  unsigned *bar = (unsigned *)((char *)ws + align256((size_t)p.cells() * p.elem()));
  Maps3 maps;
  std::memset(&maps, 0, sizeof(maps));
  if (tma && !make_maps3(p, g.P, g.ROWS, in, out, tmp, &maps, nullptr)) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(bar, 0, 256, s);
  if (e != cudaSuccess) return e;
  void *k = kp3<T>(p.shape, tma);
  void *args[] = {(void *)&in, (void *)&out, (void *)&tmp, (void *)&maps, (void *)&d, (void *)&u,
                  (void *)&steps, (void *)&bar, (void *)&c};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(g.NT);
  cfg.dynamicSmemBytes = (size_t)pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, k, args);
}

cudaError_t run_perks3d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws,
                        int64_t steps, cudaStream_t s, const DistRun *dr) {
  if (dr) return cudaErrorNotSupported;
  if (p.dtype == PERKS_F32) {
    if (p.shape == SHAPE_3D7) return launch_p3<float, SHAPE_3D7>(p, pl, (const float *)in, (float *)out, ws, steps, s);
    return launch_p3<float, SHAPE_3D27>(p, pl, (const float *)in, (float *)out, ws, steps, s);
  }
  if (p.shape == SHAPE_3D7) return launch_p3<double, SHAPE_3D7>(p, pl, (const double *)in, (double *)out, ws, steps, s);
  return launch_p3<double, SHAPE_3D27>(p, pl, (const double *)in, (double *)out, ws, steps, s);
}

}  // namespace perks
