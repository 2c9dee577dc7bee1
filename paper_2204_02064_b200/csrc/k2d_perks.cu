// k2d_perks.cu — variant (c) PERKS for 2D stencils whose domain fits on chip.
//
// The time loop runs inside one cooperative launch (Fig. 3 right).  Each CTA (1 per SM)
// owns a TX x TY tile and keeps it resident across ALL steps ("cache inter-step data in
// registers and shared memory"): RR rows per thread in registers (reg_cache) and RS rows in
// shared memory (sm_cache) (Fig. 6 Source/Destination switch).  Only the tile's
// boundary cells leave the SM: each step a CTA publishes its four edges to a global exchange slot
// (the vertical edges stored contiguously, "we transpose the vertical edges of the halo region in
// global memory") and reads its neighbours' edges through L2 (halo cells are never cached,
// P:348-355).  Instead of a device-wide grid.sync each CTA waits only on the flags of the
// (up to 8) neighbours it reads — the paper's dependency is only between adjacent TBs.
// Exchange slots and smem edge buffers are double-buffered by step parity, so one flag per step
// suffices (no write-after-read hazard: a CTA overwrites parity p only after its neighbours have
// published the next step, which they do after reading parity p).
//
// Inside the CTA, thread (wx*32+lane, wy) owns V consecutive x cells and R = RR+RS consecutive
// rows.  x-neighbours come from warp shuffles (lanes 0/31 from shared-memory column buffers at
// warp edges); the rows above/below a thread's segment come from shared-memory row buffers.
// The compute body is the same FMA chain as the host-loop kernel (reading R5) so results are
// bit-identical to variants (a) and (b).
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "internal.h"
#include "shapes.cuh"

namespace perks {

template <typename T, int V_, int WX_, int WY_, int RR_, int RS_>
struct Geo2P {
  static constexpr int V = V_, WX = WX_, WY = WY_, RR = RR_, RS = RS_, R = RR_ + RS_;
  static constexpr int NT = 32 * WX * WY;
  static constexpr int TX = 32 * V * WX, TY = WY * R;
  static constexpr int ROWW = TX + 2;  // x = -1 .. TX
  // shared memory (elements): sm_cache | row buffers | column buffers
  static constexpr int CACHE = RS * NT * V;
  static constexpr int ROWBUF = 2 /*par*/ * 2 /*top,bot*/ * (WY + 1) * ROWW;
  static constexpr int COLBUF = 2 /*par*/ * 2 /*left,right*/ * (WX + 1) * TY;
  static constexpr size_t SMEM_BYTES = (size_t)(CACHE + ROWBUF + COLBUF) * sizeof(T);
  static constexpr int SLOT = 2 * (TX + TY);  // one parity of one tile's exchange slot
};

struct Tiles2 {
  int ntx, nty;
};

template <typename T, int S, class G>
__global__ void __launch_bounds__(G::NT, 1) perks2d_kernel(const T *__restrict__ in,
                                                           T *__restrict__ out, T *gslot,
                                                           unsigned *flags, int nx, int ny,
                                                           Tiles2 tl, int64_t steps,
                                                           Coef<T, Shape<S>::N> c) {
  constexpr int V = G::V, R = G::R, RR = G::RR, NT = G::NT, TX = G::TX, TY = G::TY;
  constexpr int WX = G::WX, WY = G::WY, ROWW = G::ROWW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *smc = reinterpret_cast<T *>(smem_raw);
  T *rowb = smc + G::CACHE;
  T *colb = rowb + G::ROWBUF;
  // row buffers: top[par][j][x+1], j = 0..WY (WY = halo below);  bot[par][j+1][x+1], j = -1..WY-1
  auto TOP = [&](int par, int j) -> T * { return rowb + ((par * 2 + 0) * (WY + 1) + j) * ROWW; };
  auto BOT = [&](int par, int jp1) -> T * { return rowb + ((par * 2 + 1) * (WY + 1) + jp1) * ROWW; };
  // column buffers: left[par][k][y], k = 0..WX (WX = halo right); right[par][k+1][y], k = -1..WX-1
  auto LEFT = [&](int par, int k) -> T * { return colb + ((par * 2 + 0) * (WX + 1) + k) * TY; };
  auto RIGHT = [&](int par, int kp1) -> T * { return colb + ((par * 2 + 1) * (WX + 1) + kp1) * TY; };

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wx = warp % WX, wy = warp / WX;
  const int tile = blockIdx.x;
  const int tx = tile % tl.ntx, ty = tile / tl.ntx;
  const int x0 = tx * TX, y0 = ty * TY;
  const int xr = (wx * 32 + lane) * V;  // x relative to tile
  const int yr0 = wy * R;               // first row relative to tile
  const int x = x0 + xr;
  // global exchange slot of tile t, parity par: [top TX | bot TX | left TY | right TY]
  auto GS = [&](int t, int par) -> T * { return gslot + ((size_t)t * 2 + par) * G::SLOT; };
  const bool has_up = ty > 0, has_dn = ty + 1 < tl.nty, has_lf = tx > 0, has_rt = tx + 1 < tl.ntx;

  for (int i = tid; i < G::ROWBUF + G::COLBUF; i += NT) rowb[i] = T(0);

  // ---- prologue: load the tile into the caches (P:519 the one-time 2·D_cache term, load half)
  T reg[RR > 0 ? RR : 1][V];
  auto get_row = [&](int r, T (&v)[V]) {
    if (r < RR) {
#pragma unroll
      for (int i = 0; i < V; i++) v[i] = reg[r < RR ? r : 0][i];
    } else {
      vload<T, V>(v, smc + ((size_t)(r - RR) * NT + tid) * V);
    }
  };
  auto put_row = [&](int r, const T (&v)[V]) {
    if (r < RR) {
#pragma unroll
      for (int i = 0; i < V; i++) reg[r < RR ? r : 0][i] = v[i];
    } else {
      vstore<T, V>(smc + ((size_t)(r - RR) * NT + tid) * V, v);
    }
  };
  // publish row r (new values) into parity np: smem edges for the neighbours inside the CTA and
  // the global exchange slot for the neighbouring tiles.
  auto publish_row = [&](int np, int r, const T (&v)[V]) {
    if (r == 0) {
#pragma unroll
      for (int i = 0; i < V; i++) TOP(np, wy)[xr + 1 + i] = v[i];
      if (wy == 0) {
#pragma unroll
        for (int i = 0; i < V; i++) st_cg(GS(tile, np) + xr + i, v[i]);
      }
    }
    if (r == R - 1) {
#pragma unroll
      for (int i = 0; i < V; i++) BOT(np, wy + 1)[xr + 1 + i] = v[i];
      if (wy == WY - 1) {
#pragma unroll
        for (int i = 0; i < V; i++) st_cg(GS(tile, np) + TX + xr + i, v[i]);
      }
    }
    if (lane == 0) {
      LEFT(np, wx)[yr0 + r] = v[0];
      if (wx == 0) st_cg(GS(tile, np) + 2 * TX + yr0 + r, v[0]);
    }
    if (lane == 31) {
      RIGHT(np, wx + 1)[yr0 + r] = v[V - 1];
      if (wx == WX - 1) st_cg(GS(tile, np) + 2 * TX + TY + yr0 + r, v[V - 1]);
    }
  };

  __syncthreads();  // zeroed buffers before anyone publishes
#pragma unroll
  for (int r = 0; r < R; r++) {
    const int y = y0 + yr0 + r;
    T v[V];
#pragma unroll
    for (int i = 0; i < V; i++) v[i] = (y < ny && x + i < nx) ? in[(size_t)y * nx + x + i] : T(0);
    put_row(r, v);
    publish_row(0, r, v);
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    st_release_gpu(flags + tile, 1u);  // x^0 published
  }

  // frame predicates (reading R1): interior cells only are updated
  // rows [ylo, yhi) of the thread's segment are interior (R1); r is compared per row
  const int ylo = max(0, 1 - (y0 + yr0)), yhi = min(R, ny - 1 - (y0 + yr0));
  bool xint[V];
#pragma unroll
  for (int i = 0; i < V; i++) xint[i] = (x + i) >= 1 && (x + i) <= nx - 2;

  for (int64_t t = 0; t < steps; t++) {
    const int par = (int)(t & 1), np = par ^ 1;
    // ---- wait for the neighbours' x^t edges (flag >= t+1)
    if (tid < 8) {
      // tid 0..3: up, down, left, right; 4..7: up-left, up-right, down-left, down-right
      const int ddx = tid < 2 ? 0 : (tid < 4 ? (tid == 2 ? -1 : 1) : ((tid & 1) ? 1 : -1));
      const int ddy = tid < 2 ? (tid == 0 ? -1 : 1) : (tid < 4 ? 0 : (tid < 6 ? -1 : 1));
      const int ntx = tx + ddx, nty = ty + ddy;
      const bool need = (tid < 4 || has_corners<S>()) && ntx >= 0 && ntx < tl.ntx && nty >= 0 &&
                        nty < tl.nty;
      if (need) {
        const unsigned *f = flags + nty * tl.ntx + ntx;
        while (ld_acquire_gpu(f) < (unsigned)(t + 1)) {
        }
      }
    }
    __syncthreads();
    // ---- halo fill from the neighbours' exchange slots (parity par) through L2
    {
      const int nrow = TX, ncol = TY;
      const int total = 2 * nrow + 2 * ncol;
      for (int i = tid; i < total; i += NT) {
        if (i < nrow) {  // row above the tile <- up neighbour's bottom edge
          BOT(par, 0)[i + 1] = has_up ? ld_cg(GS(tile - tl.ntx, par) + TX + i) : T(0);
        } else if (i < 2 * nrow) {  // row below <- down neighbour's top edge
          const int k = i - nrow;
          TOP(par, WY)[k + 1] = has_dn ? ld_cg(GS(tile + tl.ntx, par) + k) : T(0);
        } else if (i < 2 * nrow + ncol) {  // left column <- left neighbour's right edge
          const int k = i - 2 * nrow;
          RIGHT(par, 0)[k] = has_lf ? ld_cg(GS(tile - 1, par) + 2 * TX + TY + k) : T(0);
        } else {  // right column <- right neighbour's left edge
          const int k = i - 2 * nrow - ncol;
          LEFT(par, WX)[k] = has_rt ? ld_cg(GS(tile + 1, par) + 2 * TX + k) : T(0);
        }
      }
      if (has_corners<S>() && tid < 4 + 4 * (WY - 1)) {
        // corners of the row buffers at x = -1 and x = TX
        if (tid < 4) {
          const bool rt = tid & 1, below = tid >> 1;
          const int ntx = tx + (rt ? 1 : -1), nty = ty + (below ? 1 : -1);
          const bool ex = ntx >= 0 && ntx < tl.ntx && nty >= 0 && nty < tl.nty;
          const int nt = nty * tl.ntx + ntx;
          // up-left: bottom-right cell of that tile; down-left: top-right; etc.
          T val = T(0);
          if (ex) val = ld_cg(GS(nt, par) + (below ? 0 : TX) + (rt ? 0 : TX - 1));
          if (below) TOP(par, WY)[rt ? TX + 1 : 0] = val;
          else BOT(par, 0)[rt ? TX + 1 : 0] = val;
        } else {
          // internal thread-row boundaries j = 1..WY-1: x = -1 / TX cells of rows y0+j*R-1 (bot)
          // and y0+j*R (top) come from the left/right neighbours' edge columns
          const int k = tid - 4;
          const int j = 1 + (k >> 2);
          const bool rt = k & 1, topk = (k >> 1) & 1;
          const int yrow = topk ? j * R : j * R - 1;
          T val = T(0);
          if (rt ? has_rt : has_lf)
            val = ld_cg(GS(rt ? tile + 1 : tile - 1, par) + 2 * TX + (rt ? 0 : TY) + yrow);
          if (topk) TOP(par, j)[rt ? TX + 1 : 0] = val;
          else BOT(par, j)[rt ? TX + 1 : 0] = val;
        }
      }
    }
    __syncthreads();
    // ---- compute x^{t+1} for the thread's V x R cells (sliding window over rows)
    T prev[V + 2], cur[V + 2], nxt[V + 2];
    // own row (old values) + its x-neighbours: shuffles inside the warp, column buffers at edges
    auto widen = [&](T (&w)[V + 2], const T (&v)[V], int r) {
      const T l = __shfl_up_sync(0xffffffffu, v[V - 1], 1);
      const T rr = __shfl_down_sync(0xffffffffu, v[0], 1);
      w[0] = lane == 0 ? RIGHT(par, wx)[yr0 + r] : l;
      w[V + 1] = lane == 31 ? LEFT(par, wx + 1)[yr0 + r] : rr;
#pragma unroll
      for (int i = 0; i < V; i++) w[i + 1] = v[i];
    };
    auto halo_below = [&](T (&w)[V + 2]) {
      const T *b = TOP(par, wy + 1) + xr;
#pragma unroll
      for (int i = 0; i < V + 2; i++) w[i] = b[i];
    };
    // FMA chain (reading R5) + frame select + publish; rotates the window
    auto finish_row = [&](int r, T (&nv)[V]) {
#pragma unroll
      for (int i = 0; i < V; i++) {
        T acc;
#pragma unroll
        for (int p = 0; p < Shape<S>::N; p++) {
          const int dy = Shape<S>::dy(p), dx = Shape<S>::dx(p);
          const T val = dy < 0 ? prev[i + 1 + dx] : (dy > 0 ? nxt[i + 1 + dx] : cur[i + 1 + dx]);
          acc = (p == 0) ? mul_rn(c.w[0], val) : fma_rn(c.w[p], val, acc);
        }
        nv[i] = (r >= ylo && r < yhi && xint[i]) ? acc : cur[i + 1];
      }
      publish_row(np, r, nv);
#pragma unroll
      for (int i = 0; i < V + 2; i++) {
        prev[i] = cur[i];
        cur[i] = nxt[i];
      }
    };
    {
      const T *b = BOT(par, wy) + xr;  // row above the segment, x = xr-1 .. xr+V
#pragma unroll
      for (int i = 0; i < V + 2; i++) prev[i] = b[i];
      T v[V];
      if (RR > 0) {
#pragma unroll
        for (int i = 0; i < V; i++) v[i] = reg[0][i];
      } else {
        vload<T, V>(v, smc + (size_t)tid * V);
      }
      widen(cur, v, 0);
    }
    // rows held in registers: fully unrolled so reg[][] is statically indexed
#pragma unroll
    for (int r = 0; r < RR; r++) {
      if (r + 1 < RR) {
        T v[V];
#pragma unroll
        for (int i = 0; i < V; i++) v[i] = reg[r + 1 < RR ? r + 1 : 0][i];
        widen(nxt, v, r + 1);
      } else if (RR < R) {
        T v[V];
        vload<T, V>(v, smc + (size_t)tid * V);  // first shared-memory row
        widen(nxt, v, r + 1);
      } else {
        halo_below(nxt);
      }
      T nv[V];
      finish_row(r, nv);
#pragma unroll
      for (int i = 0; i < V; i++) reg[r][i] = nv[i];
    }
    // rows held in shared memory (sm_cache)
#pragma unroll 2
    for (int r = RR; r < R; r++) {
      if (r + 1 < R) {
        T v[V];
        vload<T, V>(v, smc + ((size_t)(r + 1 - RR) * NT + tid) * V);
        widen(nxt, v, r + 1);
      } else {
        halo_below(nxt);
      }
      T nv[V];
      finish_row(r, nv);
      vstore<T, V>(smc + ((size_t)(r - RR) * NT + tid) * V, nv);
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_gpu(flags + tile, (unsigned)(t + 2));  // x^{t+1} published
    }
  }

  // ---- epilogue: flush the cache to `out` (the store half of the 2·D_cache term)
#pragma unroll
  for (int r = 0; r < R; r++) {
    const int y = y0 + yr0 + r;
    T v[V];
    get_row(r, v);
    if (y < ny) {
#pragma unroll
      for (int i = 0; i < V; i++)
        if (x + i < nx) out[(size_t)y * nx + x + i] = v[i];
    }
  }
}

// ------------------------------------------------------------------ host side

namespace {
// Configurations (index = Plan::cfg).  f32 V=4, f64 V=2 (16-byte vectors per thread-row).
using P2F_A = Geo2P<float, 4, 2, 8, 8, 24>;    // 256 x 256 tile, 512 thr, 64 KiB regs + 192 KiB smem
using P2F_B = Geo2P<float, 4, 1, 8, 8, 8>;     // 128 x 128 tile, 256 thr
using P2F_C = Geo2P<float, 4, 1, 4, 8, 0>;     // 128 x  32 tile, 128 thr
using P2D_A = Geo2P<double, 2, 2, 8, 4, 12>;   // 128 x 128 tile, 512 thr
using P2D_B = Geo2P<double, 2, 2, 4, 8, 0>;    // 128 x  32 tile, 256 thr
using P2D_C = Geo2P<double, 2, 1, 2, 8, 0>;    //  64 x  16 tile,  64 thr
constexpr int NCFG = 3;

struct CfgInfo {
  void *k;
  int TX, TY, NT;
  size_t smem;
  int64_t reg_cells, smem_cells;
};

template <typename T, int S, class G> CfgInfo info() {
  return CfgInfo{(void *)perks2d_kernel<T, S, G>, G::TX, G::TY, G::NT, G::SMEM_BYTES,
                 (int64_t)G::RR * G::V * G::NT, (int64_t)G::RS * G::V * G::NT};
}
template <typename T, int S> CfgInfo info_t(int cfg);
template <> CfgInfo info_t<float, SHAPE_2D5>(int c) {
  return c == 0 ? info<float, SHAPE_2D5, P2F_A>() : c == 1 ? info<float, SHAPE_2D5, P2F_B>() : info<float, SHAPE_2D5, P2F_C>();
}
template <> CfgInfo info_t<float, SHAPE_2D9>(int c) {
  return c == 0 ? info<float, SHAPE_2D9, P2F_A>() : c == 1 ? info<float, SHAPE_2D9, P2F_B>() : info<float, SHAPE_2D9, P2F_C>();
}
template <> CfgInfo info_t<double, SHAPE_2D5>(int c) {
  return c == 0 ? info<double, SHAPE_2D5, P2D_A>() : c == 1 ? info<double, SHAPE_2D5, P2D_B>() : info<double, SHAPE_2D5, P2D_C>();
}
template <> CfgInfo info_t<double, SHAPE_2D9>(int c) {
  return c == 0 ? info<double, SHAPE_2D9, P2D_A>() : c == 1 ? info<double, SHAPE_2D9, P2D_B>() : info<double, SHAPE_2D9, P2D_C>();
}
CfgInfo cfg_info(const Problem &p, int cfg) {
  if (p.dtype == PERKS_F32) return p.shape == SHAPE_2D5 ? info_t<float, SHAPE_2D5>(cfg) : info_t<float, SHAPE_2D9>(cfg);
  return p.shape == SHAPE_2D5 ? info_t<double, SHAPE_2D5>(cfg) : info_t<double, SHAPE_2D9>(cfg);
}
}  // namespace

Plan plan_perks2d(const Problem &p) {
  Plan pl;
  pl.variant = PERKS_PERKS;
  if (p.ndim != 2 || (p.shape != SHAPE_2D5 && p.shape != SHAPE_2D9) || p.bc != PERKS_BC_FRAME) {
    pl.why = "perks2d: needs 2D 5pt/9pt FRAME";
    return pl;
  }
  if (p.nx > (1 << 30) || p.ny > (1 << 30)) { pl.why = "perks2d: extent too large"; return pl; }
  // Choose the smallest tile whose tile count fits one CTA per SM (all CTAs co-resident).
  int forced = env_int("PERKS_P2D_CFG", -1);
  int best = -1;
  for (int cfg = NCFG - 1; cfg >= 0; cfg--) {
    if (forced >= 0 && cfg != forced) continue;
    CfgInfo ci = cfg_info(p, cfg);
    const int64_t tiles = ((p.nx + ci.TX - 1) / ci.TX) * ((p.ny + ci.TY - 1) / ci.TY);
    if (tiles <= p.num_sms && ci.smem <= (size_t)p.max_smem_optin) { best = cfg; break; }
  }
  if (best < 0) { pl.why = "perks2d: domain does not fit on chip (tiles > SMs)"; return pl; }
  CfgInfo ci = cfg_info(p, best);
  if (cudaFuncSetAttribute(ci.k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ci.smem) != cudaSuccess) {
    pl.why = "cudaFuncSetAttribute"; return pl;
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, ci.k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ci.k, ci.NT, ci.smem);
  const int ntx = (int)((p.nx + ci.TX - 1) / ci.TX), nty = (int)((p.ny + ci.TY - 1) / ci.TY);
  pl.cfg = best;
  pl.grid = ntx * nty;
  if (occ < 1 || pl.grid > occ * p.num_sms) { pl.why = "perks2d: not co-resident"; return pl; }
  pl.block = ci.NT;
  pl.ctas_per_sm = 1;
  pl.tile[0] = ci.TX; pl.tile[1] = ci.TY; pl.tile[2] = 1;
  pl.regs = fa.numRegs;
  pl.smem = (int)ci.smem;
  pl.units = pl.grid;
  pl.cached_reg = ci.reg_cells * pl.grid;
  pl.cached_smem = ci.smem_cells * pl.grid;
  const double S = (double)p.elem();
  pl.dram_bytes_step = 0.0;  // domain fully resident: only the one-time 2·D_cache term
  pl.halo_bytes_step = S * 2.0 * pl.grid * 2.0 * (ci.TX + ci.TY);  // publish + read, L2
  const size_t slot_bytes = (size_t)pl.grid * 2 * 2 * (ci.TX + ci.TY) * p.elem();
  pl.ws_bytes = align256(slot_bytes) + align256((size_t)pl.grid * sizeof(unsigned));
  snprintf(pl.name, sizeof(pl.name), "perks2d_%s_%s_cfg%d_t%dx%d", p.shape == SHAPE_2D5 ? "5pt" : "9pt",
           p.dtype == PERKS_F32 ? "f32" : "f64", best, ci.TX, ci.TY);
  pl.ok = true;
  return pl;
}

template <typename T, int S>
static cudaError_t launch_p2d(const Problem &p, const Plan &pl, const T *in, T *out, void *ws,
                              int64_t steps, cudaStream_t s) {
  CfgInfo ci = cfg_info(p, pl.cfg);
  Coef<T, Shape<S>::N> c;
  for (int i = 0; i < Shape<S>::N; i++) c.w[i] = sizeof(T) == 4 ? (T)p.wf[i] : (T)p.wd[i];
  T *gslot = (T *)ws;
  const size_t slot_bytes = (size_t)pl.grid * 2 * 2 * (ci.TX + ci.TY) * p.elem();
  unsigned *flags = (unsigned *)((char *)ws + align256(slot_bytes));
  cudaError_t e = cudaMemsetAsync(flags, 0, (size_t)pl.grid * sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  Tiles2 tl{(int)((p.nx + ci.TX - 1) / ci.TX), (int)((p.ny + ci.TY - 1) / ci.TY)};
  int nx = (int)p.nx, ny = (int)p.ny;
  void *args[] = {(void *)&in, (void *)&out, (void *)&gslot, (void *)&flags, (void *)&nx,
                  (void *)&ny, (void *)&tl, (void *)&steps, (void *)&c};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(ci.NT);
  cfg.dynamicSmemBytes = ci.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, ci.k, args);
}

cudaError_t run_perks2d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws,
                        int64_t steps, cudaStream_t s) {
  if (p.dtype == PERKS_F32) {
    if (p.shape == SHAPE_2D5) return launch_p2d<float, SHAPE_2D5>(p, pl, (const float *)in, (float *)out, ws, steps, s);
    return launch_p2d<float, SHAPE_2D9>(p, pl, (const float *)in, (float *)out, ws, steps, s);
  }
  if (p.shape == SHAPE_2D5) return launch_p2d<double, SHAPE_2D5>(p, pl, (const double *)in, (double *)out, ws, steps, s);
  return launch_p2d<double, SHAPE_2D9>(p, pl, (const double *)in, (double *)out, ws, steps, s);
}

}  // namespace perks
