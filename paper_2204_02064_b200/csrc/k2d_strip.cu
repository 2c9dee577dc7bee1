// k2d_strip.cu — variant (c) PERKS for 2D fp32 domains 1025..3072 cells wide: each CTA (one per SM)
// owns a FULL-WIDTH strip of SR rows for all T steps.
//
// Why strips on B200 (vs the square tiles of k2d_perks.cu): with full-width strips a CTA has only
// two halo neighbours (the strips above and below) and no halo columns, so the per-step exchange is
// two rows.  The strip computes its two EDGE rows first and publishes them at once, then sweeps
// the interior rows (registers + shared memory, the Fig. 6 reg/sm cache) while the
// neighbours' edges travel through L2 — the halo for step t+1 was published at the START of the
// neighbours' step t, so the per-step exchange latency is hidden behind the interior sweep instead
// of sitting between steps (the overlap the paper suggests for boundary vs. interior; the
// dependency is only between adjacent TBs, so no grid barrier is used).
//
// Thread (lane, warp w) owns 4 consecutive columns x = (32 w + lane) * 4 .. +3 and every row of the
// strip: rows 0..RR-1 in registers, rows RR..SR-1 in shared memory (one float4 per thread per row,
// [row][thread] so LDS.128/STS.128 are conflict free).  x-neighbours: warp shuffles inside a warp,
// a per-warp shared-memory column buffer (double-buffered by step parity) at warp boundaries.
// Inter-strip exchange: tagged LL words (value + step tag in one 8-byte store, common.cuh) in a
// per-strip, per-parity slot [top row | bottom row].
//
// The compute body is the canonical FMA chain (reading R5): results are bit-identical to the other
// variants and the oracle.
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "internal.h"
#include "shapes.cuh"

namespace perks {

constexpr int KS_V = 4;   // columns per thread (one float4)
constexpr int KS_RR = 4;  // rows per thread held in registers

// shared memory: smc[(r - RR) * NT + tid] (float4) | edge[par][w][side][SR] (side 0: first column of
// warp w, side 1: last column)
template <int S, int NWX>
__global__ void __launch_bounds__(32 * NWX, 1) perks2d_strip_kernel(const float *__restrict__ in,
                                                                  float *__restrict__ out,
                                                                  LLWord *gslot, int nx, int ny, int SR,
                                                                  int64_t steps,
                                                                  Coef<float, Shape<S>::N> c) {
  constexpr int NT = 32 * NWX, V = KS_V, RR = KS_RR;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int strip = blockIdx.x, nstrips = gridDim.x;
  const int y0 = strip * SR;
  const int R = min(SR, ny - y0);  // rows of this strip (the last strip may be shorter)
  float4 *smc = reinterpret_cast<float4 *>(smem_raw);
  float *edge = reinterpret_cast<float *>(smem_raw + (size_t)max(SR - RR, 0) * NT * sizeof(float4));
  auto EDGE = [&](int par, int ww, int side, int r) -> float & {
    return edge[(((size_t)par * NWX + ww) * 2 + side) * SR + r];
  };
  const int x = (w * 32 + lane) * V;
  // exchange slot of strip s, parity p: [top row nx | bottom row nx] tagged words
  auto GS = [&](int s, int p) -> LLWord * { return gslot + ((size_t)s * 2 + p) * 2 * (size_t)nx; };

  // ---- prologue: the strip into registers / shared memory (load half of 2·D_cache)
  float reg[RR][V];
  auto gload = [&](int y, float (&v)[V]) {
#pragma unroll
    for (int i = 0; i < V; i++) v[i] = (y >= 0 && y < ny && x + i < nx) ? in[(size_t)y * nx + x + i] : 0.f;
  };
#pragma unroll
  for (int r = 0; r < RR; r++) gload(y0 + r, reg[r]);
  for (int r = RR; r < R; r++) {
    float v[V];
    gload(y0 + r, v);
    smc[(size_t)(r - RR) * NT + tid] = make_float4(v[0], v[1], v[2], v[3]);
  }
  // halo rows of x^0 come straight from `in`, with the x-1 / x+V corner cells
  float htop[V + 2], hbot[V + 2];
  auto gload_halo = [&](int y, float (&h)[V + 2]) {
#pragma unroll
    for (int i = 0; i < V + 2; i++) {
      const int xx = x - 1 + i;
      h[i] = (y >= 0 && y < ny && xx >= 0 && xx < nx) ? in[(size_t)y * nx + xx] : 0.f;
    }
  };
  gload_halo(y0 - 1, htop);
  gload_halo(y0 + R, hbot);

  // row storage access (r is a runtime row index; registers need static indices)
  auto row_get = [&](int r, float (&v)[V]) {
    if (r < RR) {
#pragma unroll
      for (int j = 0; j < RR; j++)
        if (j == r) {
#pragma unroll
          for (int i = 0; i < V; i++) v[i] = reg[j][i];
        }
    } else {
      const float4 q = smc[(size_t)(r - RR) * NT + tid];
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    }
  };
  auto row_put = [&](int r, const float (&v)[V]) {
    if (r < RR) {
#pragma unroll
      for (int j = 0; j < RR; j++)
        if (j == r) {
#pragma unroll
          for (int i = 0; i < V; i++) reg[j][i] = v[i];
        }
    } else {
      smc[(size_t)(r - RR) * NT + tid] = make_float4(v[0], v[1], v[2], v[3]);
    }
  };
  auto put_edges = [&](int par, int r, const float (&v)[V]) {
    if (lane == 0) EDGE(par, w, 0, r) = v[0];
    if (lane == 31) EDGE(par, w, 1, r) = v[V - 1];
  };
  // initial column buffers (parity 0) from x^0
  for (int r = 0; r < R; r++) {
    float v[V];
    row_get(r, v);
    put_edges(0, r, v);
  }
  __syncthreads();

  // frame predicates (reading R1)
  unsigned colint = 0;
#pragma unroll
  for (int i = 0; i < V; i++) colint |= (x + i >= 1 && x + i <= nx - 2) ? (1u << i) : 0u;
  auto row_interior = [&](int r) { const int y = y0 + r; return y >= 1 && y <= ny - 2; };

  for (int64_t t = 0; t < steps; t++) {
    const int par = (int)(t & 1), np = par ^ 1;
    // neighbourhood of row r (old values): w[0] = x-1, w[1..V] = own, w[V+1] = x+V
    auto widen = [&](int r, const float (&v)[V], float (&wv)[V + 2]) {
      const float l = __shfl_up_sync(0xffffffffu, v[V - 1], 1);
      const float rr = __shfl_down_sync(0xffffffffu, v[0], 1);
      wv[0] = lane == 0 ? (w > 0 ? EDGE(par, w - 1, 1, r) : 0.f) : l;
      wv[V + 1] = lane == 31 ? (w < NWX - 1 ? EDGE(par, w + 1, 0, r) : 0.f) : rr;
#pragma unroll
      for (int i = 0; i < V; i++) wv[i + 1] = v[i];
    };
    auto update = [&](int r, const float (&a)[V + 2], const float (&b)[V + 2], const float (&d)[V + 2],
                      float (&nv)[V]) {
      const bool rin = row_interior(r);
#pragma unroll
      for (int i = 0; i < V; i++) {
        float acc;
#pragma unroll
        for (int p = 0; p < Shape<S>::N; p++) {
          const int dy = Shape<S>::dy(p), dx = Shape<S>::dx(p);
          const float val = dy < 0 ? a[i + 1 + dx] : (dy > 0 ? d[i + 1 + dx] : b[i + 1 + dx]);
          acc = (p == 0) ? mul_rn(c.w[0], val) : fma_rn(c.w[p], val, acc);
        }
        nv[i] = (rin && ((colint >> i) & 1u)) ? acc : b[i + 1];
      }
    };
    const unsigned tag_out = (unsigned)(t + 2);  // x^{t+1}
    // ---- 1. edge rows first, published at once (the neighbours' halo for step t+1)
    float new0[V], newL[V];
    {
      float v0[V], v1[V], a[V + 2], b[V + 2], d[V + 2];
      row_get(0, v0);
      widen(0, v0, b);
      if (R > 1) {
        row_get(1, v1);
        widen(1, v1, d);
      } else {
#pragma unroll
        for (int i = 0; i < V + 2; i++) d[i] = hbot[i];
      }
#pragma unroll
      for (int i = 0; i < V + 2; i++) a[i] = htop[i];
      update(0, a, b, d, new0);
      if (R > 1) {
        float vm[V], vl[V];
        row_get(R - 2, vm);
        row_get(R - 1, vl);
        widen(R - 2, vm, a);
        widen(R - 1, vl, b);
#pragma unroll
        for (int i = 0; i < V + 2; i++) d[i] = hbot[i];
        update(R - 1, a, b, d, newL);
      } else {
#pragma unroll
        for (int i = 0; i < V; i++) newL[i] = new0[i];
      }
    }
    {
      LLWord *g = GS(strip, np);
#pragma unroll
      for (int i = 0; i < V; i++) {
        if (x + i < nx) {
          LL<float>::put(g + x + i, new0[i], tag_out);            // top row -> strip above
          LL<float>::put(g + nx + x + i, newL[i], tag_out);       // bottom row -> strip below
        }
      }
    }
    put_edges(np, 0, new0);
    put_edges(np, R - 1, newL);
    // ---- 2. interior rows 1 .. R-2 (old values in a sliding window; register rows statically
    //         indexed, shared-memory rows in a plain loop)
    if (R > 2) {
      float a[V + 2], b[V + 2], d[V + 2];
      {
        float v[V];
#pragma unroll
        for (int i = 0; i < V; i++) v[i] = opaque_copy(reg[0][i]);
        widen(0, v, a);
#pragma unroll
        for (int i = 0; i < V; i++) v[i] = opaque_copy(reg[1][i]);
        widen(1, v, b);
      }
#pragma unroll
      for (int r = 1; r < RR; r++) {  // rows held in registers (r + 1 <= RR)
        if (r < R - 1) {
          float nx_[V];
          if (r + 1 < RR) {
#pragma unroll
            for (int i = 0; i < V; i++) nx_[i] = opaque_copy(reg[r + 1 < RR ? r + 1 : 0][i]);
          } else {
            const float4 q = smc[tid];
            nx_[0] = q.x; nx_[1] = q.y; nx_[2] = q.z; nx_[3] = q.w;
          }
          widen(r + 1, nx_, d);
          float nv[V];
          update(r, a, b, d, nv);
#pragma unroll
          for (int i = 0; i < V; i++) reg[r][i] = nv[i];
          put_edges(np, r, nv);
#pragma unroll
          for (int i = 0; i < V + 2; i++) {
            a[i] = b[i];
            b[i] = d[i];
          }
        }
      }
#pragma unroll 2
      for (int r = RR; r < R - 1; r++) {  // rows held in shared memory
        const float4 q = smc[(size_t)(r + 1 - RR) * NT + tid];
        const float nx_[V] = {q.x, q.y, q.z, q.w};
        widen(r + 1, nx_, d);
        float nv[V];
        update(r, a, b, d, nv);
        smc[(size_t)(r - RR) * NT + tid] = make_float4(nv[0], nv[1], nv[2], nv[3]);
        put_edges(np, r, nv);
#pragma unroll
        for (int i = 0; i < V + 2; i++) {
          a[i] = b[i];
          b[i] = d[i];
        }
      }
    }
    row_put(0, new0);
    if (R > 1) row_put(R - 1, newL);
    // ---- 3. halo rows of x^{t+1} from the neighbour strips (published at the START of their
    //         step, so normally already in L2): issue all 12 loads, re-poll only stale words
    if (t + 1 < steps) {
      const bool up = strip > 0, dn = strip + 1 < nstrips;
      const LLWord *gt = GS(up ? strip - 1 : 0, np) + nx;  // upper strip's bottom row
      const LLWord *gb = GS(dn ? strip + 1 : 0, np);       // lower strip's top row
      unsigned pending = 0;
#pragma unroll
      for (int i = 0; i < V + 2; i++) {
        const int xx = x - 1 + i;
        const bool in_x = xx >= 0 && xx < nx;
        htop[i] = 0.f;
        hbot[i] = 0.f;
        if (up && in_x && !LL<float>::get(gt + xx, tag_out, htop[i])) pending |= 1u << i;
        if (dn && in_x && !LL<float>::get(gb + xx, tag_out, hbot[i])) pending |= 1u << (8 + i);
      }
      const unsigned long long t0 = pending ? globaltimer_ns() : 0ull;
      while (pending) {
#pragma unroll
        for (int i = 0; i < V + 2; i++) {
          const int xx = x - 1 + i;
          if (((pending >> i) & 1u) && LL<float>::get(gt + xx, tag_out, htop[i])) pending &= ~(1u << i);
          if (((pending >> (8 + i)) & 1u) && LL<float>::get(gb + xx, tag_out, hbot[i])) pending &= ~(1u << (8 + i));
        }
        if (pending && globaltimer_ns() - t0 > PERKS_WATCHDOG_NS) watchdog_fire("perks2d strip halo", pending, tag_out);
      }
    }
    __syncthreads();  // column buffers of parity np complete before the next step reads them
  }

  // ---- epilogue: the strip to `out` (store half of 2·D_cache)
  for (int r = 0; r < R; r++) {
    float v[V];
    row_get(r, v);
#pragma unroll
    for (int i = 0; i < V; i++)
      if (x + i < nx) out[(size_t)(y0 + r) * nx + x + i] = v[i];
  }
}

// ------------------------------------------------------------------ host side
namespace {
template <int S> void *ks_ptr(int nwx) {
  if (nwx == 16) return (void *)perks2d_strip_kernel<S, 16>;
  return (void *)perks2d_strip_kernel<S, 24>;  // (32 warps would cap registers at 64: spills)
}
void *ks_kernel(const Problem &p, int nwx) {
  return p.shape == SHAPE_2D5 ? ks_ptr<SHAPE_2D5>(nwx) : ks_ptr<SHAPE_2D9>(nwx);
}
}  // namespace

Plan plan_perks2d_strip(const Problem &p) {
  Plan pl;
  pl.variant = PERKS_PERKS;
  if (p.ndim != 2 || (p.shape != SHAPE_2D5 && p.shape != SHAPE_2D9) || p.bc != PERKS_BC_FRAME ||
      p.dtype != PERKS_F32) {
    pl.why = "perks2d_strip: needs 2D 5pt/9pt fp32 FRAME";
    return pl;
  }
  if (env_int("PERKS_NO_STRIP", 0)) { pl.why = "disabled"; return pl; }
  const int64_t wcols = 32 * KS_V;  // columns per warp
  int nwx = -1;
  for (int c : {16, 24})
    if (p.nx > (c - 8) * wcols && p.nx <= c * wcols) { nwx = c; break; }
  if (nwx < 0) { pl.why = "perks2d_strip: nx outside (1024, 3072]"; return pl; }
  const int nstrips_max = p.num_sms;
  const int SR = (int)((p.ny + nstrips_max - 1) / nstrips_max);
  const int nstrips = (int)((p.ny + SR - 1) / SR);
  if (SR < 3) { pl.why = "perks2d_strip: too few rows per strip"; return pl; }
  const int NT = 32 * nwx;
  const size_t smem = (size_t)std::max(SR - KS_RR, 0) * NT * 16 + (size_t)2 * nwx * 2 * SR * sizeof(float);
  if (smem > (size_t)p.max_smem_optin) { pl.why = "perks2d_strip: strip does not fit on chip"; return pl; }
  void *k = ks_kernel(p, nwx);
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    pl.why = "cudaFuncSetAttribute"; return pl;
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem);
  if (occ < 1 || nstrips > occ * p.num_sms) { pl.why = "perks2d_strip: not co-resident"; return pl; }
  pl.cfg = (nwx << 16) | SR;
  pl.grid = nstrips;
  pl.block = NT;
  pl.ctas_per_sm = 1;
  pl.tile[0] = (int)p.nx; pl.tile[1] = SR; pl.tile[2] = 1;
  pl.regs = fa.numRegs;
  pl.smem = (int)smem;
  pl.units = nstrips;
  pl.cached_reg = (int64_t)nstrips * KS_RR * NT * KS_V;
  pl.cached_smem = std::max<int64_t>(0, p.cells() - pl.cached_reg);
  pl.dram_bytes_step = 0.0;  // resident: only the one-time 2·D_cache term
  pl.halo_bytes_step = 8.0 * 2.0 * 2.0 * (double)nstrips * (double)p.nx;  // LL words: publish + read
  pl.ws_bytes = align256((size_t)nstrips * 2 * 2 * p.nx * sizeof(LLWord));
  snprintf(pl.name, sizeof(pl.name), "perks2d_strip_%s_f32_w%d_r%d", p.shape == SHAPE_2D5 ? "5pt" : "9pt", nwx, SR);
  pl.ok = true;
  return pl;
}

cudaError_t run_perks2d_strip(const Problem &p, const Plan &pl, const void *in, void *out, void *ws,
                              int64_t steps, cudaStream_t s) {
  const int nwx = pl.cfg >> 16, SR = pl.cfg & 0xffff;
  LLWord *gslot = (LLWord *)ws;
  cudaError_t e = cudaMemsetAsync(gslot, 0, pl.ws_bytes, s);  // tags restart at 1 every run
  if (e != cudaSuccess) return e;
  int nx = (int)p.nx, ny = (int)p.ny, sr = SR;
  void *k = ks_kernel(p, nwx);
  const float *fin = (const float *)in;
  float *fout = (float *)out;
  void *args9[] = {(void *)&fin, (void *)&fout, (void *)&gslot, (void *)&nx, (void *)&ny, (void *)&sr,
                   (void *)&steps, nullptr};
  Coef<float, Shape<SHAPE_2D5>::N> c5;
  Coef<float, Shape<SHAPE_2D9>::N> c9;
  if (p.shape == SHAPE_2D5) {
    for (int i = 0; i < Shape<SHAPE_2D5>::N; i++) c5.w[i] = p.wf[i];
    args9[7] = (void *)&c5;
  } else {
    for (int i = 0; i < Shape<SHAPE_2D9>::N; i++) c9.w[i] = p.wf[i];
    args9[7] = (void *)&c9;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(pl.block);
  cfg.dynamicSmemBytes = (size_t)pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all strips co-resident (neighbours spin on tags)
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, k, args9);
}

}  // namespace perks
