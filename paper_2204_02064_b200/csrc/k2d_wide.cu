// k2d_wide.cu — every variant for GENERAL 2D point sets: any radius r <= 6 (the rest of Table II,
// 2ds9pt (r=2), 2d13pt (3), 2d17pt (4), 2d21pt (5), 2ds25pt (6), 2d25pt (5x5 box), and
// any other list of <= 64 offsets in any order).  The point list is a kernel parameter; the FMA
// chain follows it (reading R5), so results are bit-identical to the oracle and across variants.
//
// One CTA computes a TX x TY output tile from a shared-memory copy of its input tile plus an r-wide
// halo ring; 256 threads sweep the tile x-fastest (conflict-free shared-memory reads).
//   (a) host loop:  one launch per step; each CTA loads tile + ring from the step's input buffer.
//   (b) persistent: one cooperative launch, CTAs loop over tiles, grid barrier per step.
//   (c) PERKS:      one CTA per tile for all steps (every tile co-resident); the tile stays in
//       shared memory (two buffers), only the r-wide border strips leave the SM: each step a
//       CTA publishes its four border strips as tagged words (value + step tag in one 8-byte store,
//       as the r=1 tile kernel, k2d_perks.cu) and fills its halo ring from its <= 8 neighbours'
//       strips (corners from the diagonal neighbours' row strips), waiting only on those tags (the
//       dependency of P:348) — no grid barrier.  Halo cells are never cached.
// The Table II presets run with compile-time point sets (WideSet: immediate shared-memory offsets,
// unrolled FMA chain); any other list runs the same kernels with a runtime loop.  The r=1 presets
// keep their specialised kernels.
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "internal.h"

namespace perks {

constexpr int KW_THREADS = 256;    // stream kernels (many CTAs per SM)
constexpr int KW_THREADS_P = 1024; // PERKS: one CTA per SM does all of its tile's work
constexpr int KW_MAXR = 6;

template <typename T> struct WideCoef {
  int n;
  int per;  // PERKS_BC_PERIODIC: indices wrap, every cell is updated (reading R1's alternative)
  int8_t dx[kMaxPoints2D], dy[kMaxPoints2D];
  T w[kMaxPoints2D];
};

// Compile-time point sets for the Table II presets (seeded_inputs.preset order, (dy,dx)
// lexicographic): PS 1..5 = stars of radius 2..6 (2ds9pt, 2d13pt, 2d17pt, 2d21pt, 2ds25pt),
// PS 6 = the 5x5 box (2d25pt).  PS 0 = any other list (runtime loop over WideCoef).  With a
// compile-time set every term is one shared-memory load at an immediate offset and one FMA.
constexpr int kNumWidePresets = 7;
template <int PS> struct WideSet;
template <> struct WideSet<0> { static constexpr int R = 0, N = 0; };
template <int PS> struct WideSet {
  static constexpr bool BOX = PS == 6;
  static constexpr int R = BOX ? 2 : PS + 1, N = BOX ? 25 : 4 * R + 1;
  static constexpr __host__ __device__ int dx(int p) {
    return BOX ? p % 5 - 2 : (p < R ? 0 : p < 3 * R + 1 ? p - 2 * R : 0);
  }
  static constexpr __host__ __device__ int dy(int p) {
    return BOX ? p / 5 - 2 : (p < R ? p - R : p < 3 * R + 1 ? 0 : p - 3 * R);
  }
};

// Tile geometry: the stream kernels use 128 x 32 tiles; PERKS 128 x 128 (fp32) / 128 x 64 (fp64)
// so two (TX+2r)(TY+2r) buffers fit in shared memory for r <= 6.
template <typename T> struct WideGeo {
  static constexpr int TXS = 128, TYS = 32;
  static constexpr int TXP = 128, TYP = sizeof(T) == 4 ? 128 : 64;
};

// Load the tile at (x0, y0) with its r-wide ring from src into s (pitch P = TX + 2r); cells
// outside the domain read as 0 (they only feed frame cells), or wrap around (PERIODIC).
template <typename T>
__device__ void load_tile(const T *__restrict__ src, int nx, int ny, int x0, int y0, int TX, int TY, int r,
                          T *s, bool per) {
  const int P = TX + 2 * r, H = TY + 2 * r;
  for (int i = threadIdx.x; i < P * H; i += blockDim.x) {
    const int ly = i / P, lx = i % P;
    int x = x0 - r + lx, y = y0 - r + ly;
    if (per) {
      x = x < 0 ? x + nx : (x >= nx ? x - nx : x);  // r < extent: one wrap suffices
      y = y < 0 ? y + ny : (y >= ny ? y - ny : y);
    }
    s[i] = (x >= 0 && x < nx && y >= 0 && y < ny) ? __ldcg(src + (size_t)y * nx + x) : T(0);
  }
}

// New value of cell (x, y) (tile-local (lx, ly)) from the tile copy s; frame cells (within r of a
// face, reading R1) keep their value.
template <typename T, int PS, int TX>
__device__ __forceinline__ T cell_update(const T *s, int P, int r, int lx, int ly, int x, int y, int nx, int ny,
                                         const WideCoef<T> &c) {
  if constexpr (PS == 0) {
    const T *ctr = s + (ly + r) * P + (lx + r);
    if (!c.per && (x < r || x >= nx - r || y < r || y >= ny - r)) return *ctr;
    T acc = mul_rn(c.w[0], ctr[c.dy[0] * P + c.dx[0]]);
    for (int p = 1; p < c.n; p++) acc = fma_rn(c.w[p], ctr[c.dy[p] * P + c.dx[p]], acc);
    return acc;
  } else {
    using WS = WideSet<PS>;
    constexpr int R = WS::R, PC = TX + 2 * R;  // compile-time radius and pitch
    const T *ctr = s + (ly + R) * PC + (lx + R);
    if (!c.per && (x < R || x >= nx - R || y < R || y >= ny - R)) return *ctr;
    T acc = mul_rn(c.w[0], ctr[WS::dy(0) * PC + WS::dx(0)]);
#pragma unroll
    for (int p = 1; p < WS::N; p++) acc = fma_rn(c.w[p], ctr[WS::dy(p) * PC + WS::dx(p)], acc);
    return acc;
  }
}

// Compute and store the tile (x0, y0) of one step from s into dst.
template <typename T, int PS, int TX, int TY>
__device__ void tile_step(const T *s, T *__restrict__ dst, int nx, int ny, int x0, int y0, int r,
                          const WideCoef<T> &c) {
  const int P = TX + 2 * r;
  for (int i = threadIdx.x; i < TX * TY; i += blockDim.x) {
    const int ly = i / TX, lx = i % TX;
    const int x = x0 + lx, y = y0 + ly;
    if (x < nx && y < ny) dst[(size_t)y * nx + x] = cell_update<T, PS, TX>(s, P, r, lx, ly, x, y, nx, ny, c);
  }
}

template <typename T, int PS>
__global__ void __launch_bounds__(KW_THREADS) wide_hostloop_kernel(const T *__restrict__ src, T *__restrict__ dst,
                                                                   int nx, int ny, int ntx, int r,
                                                                   const __grid_constant__ WideCoef<T> c) {
  extern __shared__ __align__(16) unsigned char kw_smem[];
  T *s = reinterpret_cast<T *>(kw_smem);
  constexpr int TX = WideGeo<T>::TXS, TY = WideGeo<T>::TYS;
  const int x0 = (blockIdx.x % ntx) * TX, y0 = (blockIdx.x / ntx) * TY;
  load_tile(src, nx, ny, x0, y0, TX, TY, r, s, c.per != 0);
  __syncthreads();
  tile_step<T, PS, TX, TY>(s, dst, nx, ny, x0, y0, r, c);
}

template <typename T, int PS>
__global__ void __launch_bounds__(KW_THREADS) wide_persistent_kernel(const T *__restrict__ in, T *out, T *tmp,
                                                                     int nx, int ny, int ntx, int ntiles, int r,
                                                                     int64_t steps, unsigned *bar,
                                                                     const __grid_constant__ WideCoef<T> c) {
  extern __shared__ __align__(16) unsigned char kw_smem[];
  T *s = reinterpret_cast<T *>(kw_smem);
  constexpr int TX = WideGeo<T>::TXS, TY = WideGeo<T>::TYS;
  for (int64_t t = 0; t < steps; t++) {
    const T *src = t == 0 ? in : ((((steps - t) & 1) == 0) ? out : tmp);
    T *dst = (((steps - 1 - t) & 1) == 0) ? out : tmp;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int x0 = (tile % ntx) * TX, y0 = (tile / ntx) * TY;
      load_tile(src, nx, ny, x0, y0, TX, TY, r, s, c.per != 0);
      __syncthreads();
      tile_step<T, PS, TX, TY>(s, dst, nx, ny, x0, y0, r, c);
      __syncthreads();
    }
    if (t + 1 < steps) grid_barrier(bar, (unsigned)(t + 1));
  }
}

// PERKS: exchange slot of tile k, parity p: [top r*TX | bottom r*TX | left TY*r | right TY*r]
// tagged values (LL<T>::WORDS words each).  Strip element (row j, column i) of the top strip is
// tile cell (i, j); of the bottom strip (i, TY-r+j); of the left strip (i, j) at index j*r + i; of
// the right strip (TX-r+i, j) at index j*r + i.
template <typename T, int PS>
__global__ void __launch_bounds__(KW_THREADS_P, 1) wide_perks_kernel(const T *__restrict__ in, T *__restrict__ out,
                                                                   LLWord *gslot, int nx, int ny, int ntx, int nty,
                                                                   int r, int64_t steps,
                                                                   const __grid_constant__ WideCoef<T> c) {
  extern __shared__ __align__(16) unsigned char kw_smem[];
  constexpr int TX = WideGeo<T>::TXP, TY = WideGeo<T>::TYP, W = LL<T>::WORDS;
  const int P = TX + 2 * r, H = TY + 2 * r;
  T *buf[2] = {reinterpret_cast<T *>(kw_smem), reinterpret_cast<T *>(kw_smem) + (size_t)P * H};
  const int tile = blockIdx.x, tx = tile % ntx, ty = tile / ntx;
  const int x0 = tx * TX, y0 = ty * TY;
  const int slot_words = (2 * r * TX + 2 * TY * r) * W;
  auto GS = [&](int k, int par) -> LLWord * { return gslot + ((size_t)k * 2 + par) * slot_words; };

  // publish the border strips of buffer s (tile-local interior at (+r, +r)) with `tag`
  auto publish = [&](const T *s, int par, unsigned tag) {
    LLWord *g = GS(tile, par);
    for (int i = threadIdx.x; i < r * TX; i += blockDim.x) {
      const int j = i / TX, xi = i % TX;
      LL<T>::put(g + (size_t)i * W, s[(r + j) * P + r + xi], tag);                          // top
      LL<T>::put(g + (size_t)(r * TX + i) * W, s[(r + TY - r + j) * P + r + xi], tag);      // bottom
    }
    for (int i = threadIdx.x; i < TY * r; i += blockDim.x) {
      const int j = i / r, xi = i % r;
      LL<T>::put(g + (size_t)(2 * r * TX + i) * W, s[(r + j) * P + r + xi], tag);            // left
      LL<T>::put(g + (size_t)(2 * r * TX + TY * r + i) * W, s[(r + j) * P + r + TX - r + xi], tag);  // right
    }
  };
  // wait for one tagged value (watchdog: a lost neighbour traps instead of hanging)
  auto get = [&](const LLWord *p, unsigned tag) -> T {
    T v;
    if (LL<T>::get(p, tag, v)) return v;
    const unsigned long long t0 = globaltimer_ns();
    unsigned n = 0;
    while (!LL<T>::get(p, tag, v))
      if ((++n & 1023u) == 0 && globaltimer_ns() - t0 > PERKS_WATCHDOG_NS) watchdog_fire("wide halo", tile, tag);
    return v;
  };
  // fill the halo ring of buffer s from the neighbours' strips of parity par (tag)
  auto fill_halo = [&](T *s, int par, unsigned tag) {
    const int ring = 2 * r * (TX + 2 * r) + 2 * TY * r;  // top+bottom rows (with corners), left+right
    for (int i = threadIdx.x; i < ring; i += blockDim.x) {
      int lx, ly;  // ring cell in buffer coordinates
      if (i < 2 * r * (TX + 2 * r)) {
        const int row = i / (TX + 2 * r), col = i % (TX + 2 * r);
        ly = row < r ? row : TY + row;  // rows 0..r-1 above, TY+r..TY+2r-1 below
        lx = col;
      } else {
        const int k = i - 2 * r * (TX + 2 * r), side = k / (TY * r), m = k % (TY * r);
        ly = r + m / r;
        lx = side == 0 ? m % r : TX + r + m % r;
      }
      const int gx = x0 - r + lx, gy = y0 - r + ly;  // global cell
      T v = T(0);
      if (gx >= 0 && gx < nx && gy >= 0 && gy < ny) {
        const int ntxi = (gx < x0) ? tx - 1 : (gx >= x0 + TX ? tx + 1 : tx);
        const int ntyi = (gy < y0) ? ty - 1 : (gy >= y0 + TY ? ty + 1 : ty);
        const int nk = ntyi * ntx + ntxi;
        const int cx = gx - ntxi * TX, cy = gy - ntyi * TY;  // cell in the neighbour's tile
        const LLWord *g = GS(nk, par);
        size_t idx;
        if (ntyi != ty) {  // from the neighbour's top / bottom row strip (corners included)
          idx = ntyi < ty ? (size_t)(r * TX) + (size_t)(cy - (TY - r)) * TX + cx : (size_t)cy * TX + cx;
        } else {           // from its left / right column strip
          idx = ntxi < tx ? (size_t)(2 * r * TX + TY * r) + (size_t)cy * r + (cx - (TX - r))
                          : (size_t)(2 * r * TX) + (size_t)cy * r + cx;
        }
        v = get(g + idx * W, tag);
      }
      s[ly * P + lx] = v;
    }
  };

  // ---- prologue: tile (and ring) from `in`; publish x^0's strips (tag 1, parity 0)
  load_tile(in, nx, ny, x0, y0, TX, TY, r, buf[0], false);  // (FRAME only)
  __syncthreads();
  publish(buf[0], 0, 1u);
  int cur = 0;
  for (int64_t t = 0; t < steps; t++) {
    const int par = (int)(t & 1);
    if (t > 0) fill_halo(buf[cur], par, (unsigned)(t + 1));  // step 0 has the ring from `in`
    __syncthreads();
    // x^{t+1} into the other buffer's interior
    T *sn = buf[cur ^ 1];
    for (int i = threadIdx.x; i < TX * TY; i += blockDim.x) {
      const int ly = i / TX, lx = i % TX;
      const int x = x0 + lx, y = y0 + ly;
      sn[(ly + r) * P + lx + r] = (x < nx && y < ny) ? cell_update<T, PS, TX>(buf[cur], P, r, lx, ly, x, y, nx, ny, c) : T(0);
    }
    __syncthreads();
    publish(sn, par ^ 1, (unsigned)(t + 2));
    cur ^= 1;
  }
  // ---- epilogue: the tile to `out`
  const T *s = buf[cur];
  for (int i = threadIdx.x; i < TX * TY; i += blockDim.x) {
    const int ly = i / TX, lx = i % TX;
    const int x = x0 + lx, y = y0 + ly;
    if (x < nx && y < ny) out[(size_t)y * nx + x] = s[(ly + r) * P + lx + r];
  }
}

// ------------------------------------------------------------------ host side
namespace {
int radius2d(const Problem &p) {
  int r = 0;
  for (int i = 0; i < p.npts; i++) r = std::max(r, std::max(std::abs(p.off[i][0]), std::abs(p.off[i][1])));
  return r;
}
template <typename T> WideCoef<T> make_coef(const Problem &p) {
  WideCoef<T> c{};
  c.per = p.bc == PERKS_BC_PERIODIC ? 1 : 0;
  c.n = p.npts;
  for (int i = 0; i < p.npts; i++) {
    c.dx[i] = (int8_t)p.off[i][0];
    c.dy[i] = (int8_t)p.off[i][1];
    c.w[i] = sizeof(T) == 4 ? (T)p.wf[i] : (T)p.wd[i];
  }
  return c;
}
template <typename T> size_t stream_smem(int r) {
  return (size_t)(WideGeo<T>::TXS + 2 * r) * (WideGeo<T>::TYS + 2 * r) * sizeof(T);
}
template <typename T> size_t perks_smem(int r) {
  return 2 * (size_t)(WideGeo<T>::TXP + 2 * r) * (WideGeo<T>::TYP + 2 * r) * sizeof(T);
}
// Which compile-time set (WideSet) the problem's point list is, 0 if none.
int wide_preset(const Problem &p) {
  for (int ps = 1; ps < kNumWidePresets; ps++) {
    const bool box = ps == 6;
    const int R = box ? 2 : ps + 1, N = box ? 25 : 4 * R + 1;
    if (p.npts != N) continue;
    bool ok = true;
    for (int q = 0; q < N && ok; q++) {
      const int dx = box ? q % 5 - 2 : (q < R ? 0 : q < 3 * R + 1 ? q - 2 * R : 0);
      const int dy = box ? q / 5 - 2 : (q < R ? q - R : q < 3 * R + 1 ? 0 : q - 3 * R);
      ok = p.off[q][0] == dx && p.off[q][1] == dy;
    }
    if (ok) return ps;
  }
  return 0;
}
template <typename T, int PS> void *wk_ps(perks_variant v) {
  return v == PERKS_HOSTLOOP ? (void *)wide_hostloop_kernel<T, PS>
         : v == PERKS_PERSISTENT ? (void *)wide_persistent_kernel<T, PS> : (void *)wide_perks_kernel<T, PS>;
}
template <typename T> void *wk(perks_variant v, int ps) {
  switch (ps) {
    case 1: return wk_ps<T, 1>(v);
    case 2: return wk_ps<T, 2>(v);
    case 3: return wk_ps<T, 3>(v);
    case 4: return wk_ps<T, 4>(v);
    case 5: return wk_ps<T, 5>(v);
    case 6: return wk_ps<T, 6>(v);
    default: return wk_ps<T, 0>(v);
  }
}
}  // namespace

Plan plan_wide2d(const Problem &p, perks_variant v) {
  Plan pl;
  pl.variant = v;
  const int r = radius2d(p);
  if (p.ndim != 2 || p.shape != SHAPE_G2D || r > KW_MAXR || p.npts > kMaxPoints2D) {
    pl.why = "wide2d: 2D point sets of radius <= 6";
    return pl;
  }
  if (p.bc == PERKS_BC_PERIODIC && v == PERKS_PERKS) {
    // PERIODIC: the resident-tile exchange assumes a bounded tile grid; PERKS runs the persistent
    // body with an empty cache split (as in 3D, §7)
    Plan q = plan_wide2d(p, PERKS_PERSISTENT);
    if (q.ok) {
      q.variant = PERKS_PERKS;
      q.persistent_body = true;
      q.cached_smem = 0;
      snprintf(q.name, sizeof(q.name), "perks2d_wide_r%d_%dpt_%s_per_c0", r, p.npts, p.dtype == PERKS_F32 ? "f32" : "f64");
    }
    return q;
  }
  const bool f32 = p.dtype == PERKS_F32;
  const int ps = wide_preset(p);
  void *k = f32 ? wk<float>(v, ps) : wk<double>(v, ps);
  const bool perks = v == PERKS_PERKS;
  const int TX = perks ? (f32 ? WideGeo<float>::TXP : WideGeo<double>::TXP) : (f32 ? WideGeo<float>::TXS : WideGeo<double>::TXS);
  const int TY = perks ? (f32 ? WideGeo<float>::TYP : WideGeo<double>::TYP) : (f32 ? WideGeo<float>::TYS : WideGeo<double>::TYS);
  const size_t smem = perks ? (f32 ? perks_smem<float>(r) : perks_smem<double>(r))
                            : (f32 ? stream_smem<float>(r) : stream_smem<double>(r));
  if (smem > (size_t)p.max_smem_optin) { pl.why = "wide2d: tile does not fit shared memory"; return pl; }
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    pl.why = "cudaFuncSetAttribute";
    return pl;
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, perks ? KW_THREADS_P : KW_THREADS, smem);
  if (occ < 1) { pl.why = "wide2d: not resident"; return pl; }
  const int ntx = (int)((p.nx + TX - 1) / TX), nty = (int)((p.ny + TY - 1) / TY);
  const int64_t tiles = (int64_t)ntx * nty;
  if (perks && tiles > (int64_t)occ * p.num_sms) { pl.why = "wide2d perks: domain does not fit on chip"; return pl; }
  pl.units = tiles;
  pl.grid = v == PERKS_PERSISTENT ? (int)std::min<int64_t>(tiles, (int64_t)occ * p.num_sms) : (int)tiles;
  pl.block = perks ? KW_THREADS_P : KW_THREADS;
  pl.ctas_per_sm = perks ? 1 : occ;
  pl.tile[0] = TX; pl.tile[1] = TY; pl.tile[2] = 1;
  pl.regs = fa.numRegs;
  pl.smem = (int)smem;
  pl.family = 4;  // (wide 2D)
  const double S = (double)p.elem();
  if (perks) {
    pl.cached_smem = std::min<int64_t>(tiles * TX * TY, p.cells());
    pl.dram_bytes_step = 0.0;
    pl.halo_bytes_step = S * 2.0 * tiles * 2.0 * r * (TX + TY);
    const size_t words = (size_t)tiles * 2 * (2 * r * TX + 2 * TY * r) * LL<float>::WORDS * (p.elem() == 8 ? 2 : 1);
    pl.ws_bytes = align256(words * sizeof(LLWord));
  } else {
    pl.dram_bytes_step = 2.0 * S * (double)p.cells();
    pl.halo_bytes_step = S * (double)tiles * 2.0 * r * (TX + TY + 2 * r);
    pl.ws_bytes = align256((size_t)p.cells() * p.elem()) + (v == PERKS_PERSISTENT ? 256 : 0);
  }
  pl.cfg = ps;  // compile-time point set (0: runtime list)
  snprintf(pl.name, sizeof(pl.name), "%s2d_wide_r%d_%dpt%s_%s_t%dx%d", perks ? "perks" : v == PERKS_PERSISTENT ? "persistent" : "hostloop",
           r, p.npts, ps ? "" : "_any", f32 ? "f32" : "f64", TX, TY);
  pl.ok = true;
  return pl;
}

namespace {
template <typename T>
cudaError_t run_wide_t(const Problem &p, const Plan &pl, const T *in, T *out, void *ws, int64_t steps, cudaStream_t s) {
  const WideCoef<T> c = make_coef<T>(p);
  const int r = radius2d(p);
  const perks_variant kv = pl.persistent_body ? PERKS_PERSISTENT : pl.variant;
  void *k = wk<T>(kv, pl.cfg);
  const int nx = (int)p.nx, ny = (int)p.ny;
  const int ntx = (nx + pl.tile[0] - 1) / pl.tile[0], nty = (ny + pl.tile[1] - 1) / pl.tile[1];
  if (pl.variant == PERKS_HOSTLOOP) {
    T *tmp = (T *)ws;
    for (int64_t t = 0; t < steps; t++) {
      const T *src = t == 0 ? in : ((((steps - t) & 1) == 0) ? out : tmp);
      T *dst = (((steps - 1 - t) & 1) == 0) ? out : tmp;
      void *args[] = {(void *)&src, (void *)&dst, (void *)&nx, (void *)&ny, (void *)&ntx, (void *)&r, (void *)&c};
      cudaError_t e = cudaLaunchKernel(k, dim3(pl.grid), dim3(KW_THREADS), args, pl.smem, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(pl.block);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (kv == PERKS_PERSISTENT) {
    T *tmp = (T *)ws;
    unsigned *bar = (unsigned *)((char *)ws + align256((size_t)p.cells() * p.elem()));
    cudaError_t e = reset_grid_barrier(bar, s);
    if (e != cudaSuccess) return e;
    const int ntiles = ntx * nty;
    void *args[] = {(void *)&in, (void *)&out, (void *)&tmp, (void *)&nx, (void *)&ny, (void *)&ntx,
                    (void *)&ntiles, (void *)&r, (void *)&steps, (void *)&bar, (void *)&c};
    return cudaLaunchKernelExC(&cfg, k, args);
  }
  cudaError_t e = cudaMemsetAsync(ws, 0, pl.ws_bytes, s);  // tags start at 0 (x^s carries s+1)
  if (e != cudaSuccess) return e;
  LLWord *gslot = (LLWord *)ws;
  void *args[] = {(void *)&in, (void *)&out, (void *)&gslot, (void *)&nx, (void *)&ny, (void *)&ntx,
                  (void *)&nty, (void *)&r, (void *)&steps, (void *)&c};
  return cudaLaunchKernelExC(&cfg, k, args);
}
}  // namespace

cudaError_t run_wide2d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws, int64_t steps,
                       cudaStream_t s) {
  if (p.dtype == PERKS_F32) return run_wide_t<float>(p, pl, (const float *)in, (float *)out, ws, steps, s);
  return run_wide_t<double>(p, pl, (const double *)in, (double *)out, ws, steps, s);
}

}  // namespace perks
