// k2d_tiled.cu — Tiled PERKS ([draft] P:416-441, model P:917-991) for 2D domains larger than the
// on-chip capacity.
//
// "We spatially tile the domain to sub-domain sizes we can entirely cache in shared memory and
// registers.  The tiles are loaded in a serial fashion such that at a given time the entire device
// is executing a single tile.  Each tile has a redundant halo region to enable the execution of
// consecutive time steps for the tile ... After all tiles are advanced to the maximum possible
// number of steps, ... we do another pass on the tiles".
//
// Here a device tile is a sub-domain the resident 2D PERKS kernels hold entirely on chip
// (perks2d tiles for 2d5pt/2d9pt, the general wide2d PERKS kernel for any other 2D point set).
// A pass advances every tile by Tb steps: the tile's valid region [x0,x1) x [y0,y1) is extended by
// a halo of H = r*Tb cells on every side that is not a global face, the extended tile is run with
// the unchanged PERKS kernel for Tb steps (its outer ring acts as a frozen frame: a cell at distance
// d from an interior edge is exact for d >= s after s steps, so the valid region is exact after
// Tb steps), and the valid region is copied to the pass's output buffer.  Passes ping-pong between
// the workspace and `out` so the last pass lands in `out` (reading R8).  The intra-tile temporal
// dependency is resolved by the kernel's own neighbour synchronisation, the inter-tile
// one by the pass structure.  Cost (P:976 model): the redundant halo work (E^2 / V^2 per step, E the
// extended and V the valid tile side) against one DRAM round trip of the tile per Tb steps instead
// of per step; the planner picks Tb minimising that estimate.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "internal.h"
#include "shapes.cuh"

namespace perks {

namespace {
int radius2d_any(const Problem &p) {
  if (p.shape == SHAPE_2D5 || p.shape == SHAPE_2D9) return 1;
  int r = 0;
  for (int i = 0; i < p.npts; i++) r = std::max(r, std::max(std::abs((int)p.off[i][0]), std::abs((int)p.off[i][1])));
  return r;
}
Problem sub_problem(const Problem &p, int64_t ny, int64_t nx) {
  Problem q = p;
  q.nx = nx;
  q.ny = ny;
  return q;
}
Plan sub_plan(const Problem &q) {
  return (q.shape == SHAPE_2D5 || q.shape == SHAPE_2D9) ? plan_perks2d(q) : plan_wide2d(q, PERKS_PERKS);
}
cudaError_t sub_run(const Problem &q, const Plan &pl, const void *in, void *out, void *ws, int64_t steps,
                    cudaStream_t s) {
  return (q.shape == SHAPE_2D5 || q.shape == SHAPE_2D9) ? run_perks2d(q, pl, in, out, ws, steps, s)
                                                        : run_wide2d(q, pl, in, out, ws, steps, s);
}
// Tiling of one axis of extent n into k valid segments with a halo h: segment i = [a, b),
// extended [max(0, a - h), min(n, b + h)).
struct Axis {
  int64_t n, h;
  int k;
  int64_t v;  // valid segment length (the last one may be shorter)
  int64_t a(int i) const { return std::min(n, (int64_t)i * v); }
  int64_t b(int i) const { return std::min(n, (int64_t)(i + 1) * v); }
  int64_t ea(int i) const { return std::max<int64_t>(0, a(i) - h); }
  int64_t eb(int i) const { return std::min(n, b(i) + h); }
  int64_t emax() const {
    int64_t m = 0;
    for (int i = 0; i < k; i++) m = std::max(m, eb(i) - ea(i));
    return m;
  }
};
Axis make_axis(int64_t n, int64_t h, int k) {
  Axis ax{n, h, k, (n + k - 1) / k};
  return ax;
}
}  // namespace

// Plan: the largest square extended tile the resident kernel accepts (capacity E), then the pass
// length Tb and tile counts minimising (redundant on-chip work) x (1 + DRAM round trip / Tb).
Plan plan_tiled2d(const Problem &p, int64_t steps_hint) {
  Plan pl;
  pl.variant = PERKS_PERKS;
  if (p.ndim != 2 || p.bc != PERKS_BC_FRAME || p.nranks > 1 ||
      !(p.shape == SHAPE_2D5 || p.shape == SHAPE_2D9 || p.shape == SHAPE_G2D)) {
    pl.why = "tiled2d: 2D FRAME single GPU";
    return pl;
  }
  const int r = radius2d_any(p);
  // capacity: largest E (multiple of 64) with a resident plan for an E x E tile
  int64_t lo = 0;
  for (int64_t e = 64; e <= 16384; e += 64) {
    if (sub_plan(sub_problem(p, e, e)).ok) lo = e;
    else if (lo > 0) break;
  }
  if (lo < 8 * r + 64) { pl.why = "tiled2d: no resident tile size"; return pl; }
  const int64_t E = lo;
  (void)steps_hint;
  const int forced = env_int("PERKS_TILED_TB", 0);
  // Cost per time step of a tiling (seconds, estimated): every pass runs each extended tile for
  // Tb steps on the resident kernel, whose step time is set by the cells of ONE CTA tile (the
  // CTAs run in parallel: profiles/r01_c2_tile_scaling.txt), plus one DRAM round trip of the
  // extended tile per pass (copy in + kernel load + kernel store + copy out of the valid part).
  // resident step time of one CTA tile of c cells ~ a + b*c (fit to profiles/r01_sweep2d.txt:
  // 2d9pt fp32 256x256 6.47, 256x192 5.31, 256x128 4.01, 128x64 2.25 us; 2d5pt fp64 128x128 3.17 us)
  const double a_chip = p.dtype == PERKS_F64 ? 1.2e-6 : 1.5e-6, b_chip = p.dtype == PERKS_F64 ? 0.10e-9 : 0.077e-9;
  const double B_gm = 6.5e12;
  double best = 1e300;
  int best_tb = 0, bkx = 0, bky = 0;
  std::vector<int> tbs = {4, 8, 12, 16, 24, 32, 48, 64, 96, 128};
  if (forced > 0) tbs = {forced};
  for (int tb : tbs) {
    const int64_t h = (int64_t)r * tb;
    if (E - 2 * h < 16) continue;
    auto kmin = [&](int64_t n) {
      for (int k = 1; k <= 4096; k++)
        if (make_axis(n, h, k).emax() <= E) return k;
      return 0;
    };
    const int kx0 = kmin(p.nx), ky0 = kmin(p.ny);
    if (kx0 == 0 || ky0 == 0) continue;
    for (int kx = kx0; kx <= kx0 + 3; kx++) {
      for (int ky = ky0; ky <= ky0 + 3; ky++) {
        const Axis ax = make_axis(p.nx, h, kx), ay = make_axis(p.ny, h, ky);
        if (ax.v <= h || ay.v <= h) continue;
        double t_pass = 0;
        bool ok = true;
        for (int j = 0; j < ky && ok; j++)
          for (int i = 0; i < kx && ok; i++) {
            const int64_t ex = ax.eb(i) - ax.ea(i), ey = ay.eb(j) - ay.ea(j);
            const Plan sp = sub_plan(sub_problem(p, ey, ex));
            if (!sp.ok) { ok = false; break; }
            const double cta = (double)std::min<int64_t>(sp.tile[0], ex) * (double)std::min<int64_t>(sp.tile[1], ey);
            t_pass += tb * (a_chip + b_chip * cta) + 4.0 * (double)ex * ey * p.elem() / B_gm;
          }
        if (!ok) continue;
        const double cost = t_pass / tb;
        if (cost < best) { best = cost; best_tb = tb; bkx = kx; bky = ky; }
      }
    }
  }
  if (best_tb == 0) { pl.why = "tiled2d: no tiling"; return pl; }
  const int64_t h = (int64_t)r * best_tb;
  const Axis ax = make_axis(p.nx, h, bkx), ay = make_axis(p.ny, h, bky);
  const Plan big = sub_plan(sub_problem(p, ay.emax(), ax.emax()));
  if (!big.ok) { pl.why = "tiled2d: extended tile not resident"; return pl; }
  pl.grid = big.grid;
  pl.block = big.block;
  pl.ctas_per_sm = big.ctas_per_sm;
  pl.regs = big.regs;
  pl.smem = big.smem;
  pl.tile[0] = (int)ax.v; pl.tile[1] = (int)ay.v; pl.tile[2] = 1;
  pl.zchunk = best_tb;    // steps per pass
  pl.units = (int64_t)bkx * bky;
  pl.cfg = bkx;           // tiles along x (y: units / cfg)
  pl.family = 5;          // (2D tiled PERKS)
  const double S = (double)p.elem();
  // cached: the whole valid domain is resident for Tb steps at a time; DRAM per step: each pass
  // copies the extended tiles in and the valid tiles out, and the kernel loads / stores its tile
  double ext_area = 0;
  for (int j = 0; j < bky; j++)
    for (int i = 0; i < bkx; i++) ext_area += (double)(ax.eb(i) - ax.ea(i)) * (double)(ay.eb(j) - ay.ea(j));
  pl.cached_smem = std::min<int64_t>(big.cached_smem, p.cells());
  pl.cached_reg = std::min<int64_t>(big.cached_reg, p.cells() - pl.cached_smem);
  pl.cached_tmem = std::min<int64_t>(big.cached_tmem, p.cells() - pl.cached_smem - pl.cached_reg);
  pl.dram_bytes_step = S * (3.0 * ext_area + (double)p.cells()) / best_tb;
  pl.halo_bytes_step = big.halo_bytes_step * (double)pl.units;
  const size_t stage = align256((size_t)ax.emax() * ay.emax() * p.elem());
  pl.ws_bytes = align256((size_t)p.cells() * p.elem()) + 2 * stage + align256(big.ws_bytes);
  snprintf(pl.name, sizeof(pl.name), "perks2d_tiled_%dx%d_tb%d_%s", bkx, bky, best_tb, big.name);
  pl.ok = true;
  return pl;
}

cudaError_t run_tiled2d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws, int64_t steps,
                        cudaStream_t s) {
  const int r = radius2d_any(p);
  const int tb = pl.zchunk, kx = pl.cfg, ky = (int)(pl.units / pl.cfg);
  const int64_t h = (int64_t)r * tb;
  const Axis ax = make_axis(p.nx, h, kx), ay = make_axis(p.ny, h, ky);
  const size_t S = p.elem();
  char *w = (char *)ws;
  char *A = w;
  const size_t stage = align256((size_t)ax.emax() * ay.emax() * S);
  char *sin = A + align256((size_t)p.cells() * S);
  char *sout = sin + stage;
  void *sws = sout + stage;
  const int64_t passes = (steps + tb - 1) / tb;
  const char *cur = (const char *)in;
  for (int64_t ps = 0; ps < passes; ps++) {
    const int64_t tp = std::min<int64_t>(tb, steps - ps * tb);
    char *nxt = ((passes - 1 - ps) % 2 == 0) ? (char *)out : A;
    for (int j = 0; j < ky; j++) {
      for (int i = 0; i < kx; i++) {
        const int64_t ex0 = ax.ea(i), ex1 = ax.eb(i), ey0 = ay.ea(j), ey1 = ay.eb(j);
        const int64_t x0 = ax.a(i), x1 = ax.b(i), y0 = ay.a(j), y1 = ay.b(j);
        const int64_t enx = ex1 - ex0, eny = ey1 - ey0;
        const Problem q = sub_problem(p, eny, enx);
        const Plan qp = sub_plan(q);
        if (!qp.ok) return cudaErrorInvalidConfiguration;
        cudaError_t e = cudaMemcpy2DAsync(sin, (size_t)enx * S, cur + ((size_t)ey0 * p.nx + ex0) * S, (size_t)p.nx * S,
                                          (size_t)enx * S, (size_t)eny, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return e;
        if ((e = sub_run(q, qp, sin, sout, sws, tp, s)) != cudaSuccess) return e;
        e = cudaMemcpy2DAsync(nxt + ((size_t)y0 * p.nx + x0) * S, (size_t)p.nx * S,
                              sout + ((size_t)(y0 - ey0) * enx + (x0 - ex0)) * S, (size_t)enx * S,
                              (size_t)(x1 - x0) * S, (size_t)(y1 - y0), cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return e;
      }
    }
    cur = nxt;
  }
  return cudaSuccess;
}

}  // namespace perks
