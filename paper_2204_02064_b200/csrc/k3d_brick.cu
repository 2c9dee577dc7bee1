// k3d_brick.cu — PERKS (c) for 3D domains that fit on chip: the resident-brick kernel.
//
// "Planes that already have the data cached from the previous time step do not load from global
// memory": here EVERY plane is cached.  The domain is cut into bricks (an xy tile of
// TX x TY cells times NZ planes), one brick per CTA and one CTA per SM (one cooperative launch,
// the time loop inside).  A brick stays in shared memory for all T steps (the paper's
// register/shared-memory cache): one slot per plane, each slot holding the plane's
// tile plus a one-cell halo ring, and two extra slots for the planes just below and above the
// brick.  Per time step:
//
//   1. halo refresh — the ring cells of every plane and the two z-halo planes are the surface
//      cells of the <= 26 neighbouring bricks at step t.  Neighbours publish them as tagged words
//      (value and step tag in one 8-byte store, common.cuh LL<T>; no flag, no fence, no grid
//      barrier: a brick waits only for the words it reads, the dependency of P:348).  Each thread
//      issues all its loads first, then re-polls only words whose tag has not arrived.
//   2. sweep — the planes are swept in z with the plane-streaming body of the uncached kernels
//      (stream3d.cuh arrival(): each resident plane's neighbourhood is read from shared memory
//      once and applied to outputs q+1 / q / q-1 in list order, reading R5), one CTA barrier per
//      plane.  Output plane q-1 is final when plane q has been read; it replaces the old plane q-1
//      in its slot (no warp reads that slot again this step), and its surface cells (tile edges,
//      and the whole plane for the brick's first/last plane) are published for step t+1.
//
// DRAM traffic is only the one-time load and store of the domain (A_gm = 2·D_cache); the
// per-step traffic is the brick surface through L2 (A_gm(H(D_cache))).
// Parity of the exchange words: step t publishes x^{t+1} into parity (t+1)&1 with tag t+1 (tags
// restart at 1 every run: the exchange region is zeroed before the launch).  Write-after-read is
// impossible: a brick can publish x^{t+2} into parity t&1 only after it gathered x^{t+1} from all
// its neighbours, each of which published x^{t+1} only after finishing its own gather of x^t.
#include <algorithm>
#include <cstdio>

#include "internal.h"
#include "stream3d.cuh"

namespace perks {

// Brick geometries: one thread owns V x R cells of every plane, 8 warps: tiles of TX x TY cells.
#ifndef PERKS_BRICK_R
#define PERKS_BRICK_R 2
#endif
#ifndef PERKS_BRICK_V
#define PERKS_BRICK_V 2
#endif
template <typename T> struct GBrick { using G = Geo3D<T, PERKS_BRICK_V, PERKS_BRICK_R, 8, 2>; };
constexpr int kBrickThreads = 256;
constexpr int kMaxSegs = 26;
#ifndef PERKS_BRICK_GMAX
#define PERKS_BRICK_GMAX 16
#endif
constexpr int kGatherMax = PERKS_BRICK_GMAX;  // halo words one thread holds in flight per pass

struct BrickGeo {
  int ntx, nty, nbz;  // bricks along x, y, z
  int NZ;             // planes per brick (the last z brick may have fewer)
  long long bw;       // exchange cells per brick (per parity)
};

// Exchange block of one brick (cells; x LLG<T>::WORDS words): the surface of the brick.
//   W/E columns [NZ][TY], low/high rows [NZ][TX], low/high z faces [TY][TX].
template <class G> struct Sec {
  int NZ;
  PERKS_DEVINL int wcol(int z, int y) const { return z * G::TY + y; }
  PERKS_DEVINL int ecol(int z, int y) const { return (NZ + z) * G::TY + y; }
  PERKS_DEVINL int ylo(int z, int x) const { return 2 * NZ * G::TY + z * G::TX + x; }
  PERKS_DEVINL int yhi(int z, int x) const { return 2 * NZ * G::TY + (NZ + z) * G::TX + x; }
  PERKS_DEVINL int zlo(int y, int x) const { return 2 * NZ * (G::TY + G::TX) + y * G::TX + x; }
  PERKS_DEVINL int zhi(int y, int x) const { return 2 * NZ * (G::TY + G::TX) + (G::TY + y) * G::TX + x; }
};
template <class G> long long brick_cells(int NZ) { return 2LL * NZ * (G::TY + G::TX) + 2LL * G::TY * G::TX; }

// One halo segment: a 2D block of exchange cells (loop kz < nz, ki < ni) copied into slots.
struct Seg {
  long long src;  // exchange cell index of (0, 0) within the parity buffer
  int ssz, ssi;   // source strides (cells)
  int dst;        // shared-memory element offset of (0, 0) from the first slot
  int dsz, dsi;   // destination strides (elements)
  int nz, ni;
  int end;        // prefix count of elements up to and including this segment
};

struct BrickPos {
  int tx, ty, bz;      // brick coordinates
  int x0, y0, zb;      // origin
  int txc, tyc, nzc;   // extents clipped to the domain
};
template <class G>
PERKS_DEVINL BrickPos brick_pos(const BrickGeo &bg, const Dom3 &d, int b) {
  BrickPos q;
  q.tx = b % bg.ntx;
  q.ty = (b / bg.ntx) % bg.nty;
  q.bz = b / (bg.ntx * bg.nty);
  q.x0 = q.tx * G::TX;
  q.y0 = q.ty * G::TY;
  q.zb = q.bz * bg.NZ;
  q.txc = min(G::TX, d.nx - q.x0);
  q.tyc = min(G::TY, d.ny - q.y0);
  q.nzc = min(bg.NZ, d.nz - q.zb);
  return q;
}

// Build the CTA's halo segment table (thread 0).  Slot k holds plane zb - 1 + k.
template <class G, bool CORNERS>
PERKS_DEVINL int build_segs(const BrickGeo &bg, const Dom3 &d, const BrickPos &me, Seg *segs) {
  const Sec<G> sec{bg.NZ};
  int n = 0, cnt = 0;
  auto nb = [&](int dx, int dy, int dz, BrickPos &o) -> bool {
    const int tx = me.tx + dx, ty = me.ty + dy, bz = me.bz + dz;
    if (tx < 0 || tx >= bg.ntx || ty < 0 || ty >= bg.nty || bz < 0 || bz >= bg.nbz) return false;
    o = brick_pos<G>(bg, d, (bz * bg.nty + ty) * bg.ntx + tx);
    return true;
  };
  auto base = [&](const BrickPos &o) { return (long long)((o.bz * bg.nty + o.ty) * bg.ntx + o.tx) * bg.bw; };
  auto add = [&](long long src, int ssz, int ssi, int dst, int dsz, int dsi, int nz, int ni) {
    if (nz <= 0 || ni <= 0) return;
    cnt += nz * ni;
    segs[n++] = Seg{src, ssz, ssi, dst, dsz, dsi, nz, ni, cnt};
  };
  const int P = G::P, SL = G::SLOT, C0 = G::PAD;  // C0: column of the tile's first cell
  BrickPos o;
  // ---- in-plane rings of the brick's own planes (slots 1..nzc), from the same z layer
  if (nb(0, -1, 0, o)) add(base(o) + sec.yhi(0, 0), G::TX, 1, SL + C0, SL, 1, me.nzc, me.txc);
  if (nb(0, 1, 0, o)) add(base(o) + sec.ylo(0, 0), G::TX, 1, SL + (me.tyc + 1) * P + C0, SL, 1, me.nzc, me.txc);
  if (nb(-1, 0, 0, o)) add(base(o) + sec.ecol(0, 0), G::TY, 1, SL + P + C0 - 1, SL, P, me.nzc, me.tyc);
  if (nb(1, 0, 0, o)) add(base(o) + sec.wcol(0, 0), G::TY, 1, SL + P + C0 + me.txc, SL, P, me.nzc, me.tyc);
  if (CORNERS) {
    if (nb(-1, -1, 0, o)) add(base(o) + sec.yhi(0, o.txc - 1), G::TX, 1, SL + C0 - 1, SL, 1, me.nzc, 1);
    if (nb(1, -1, 0, o)) add(base(o) + sec.yhi(0, 0), G::TX, 1, SL + C0 + me.txc, SL, 1, me.nzc, 1);
    if (nb(-1, 1, 0, o)) add(base(o) + sec.ylo(0, o.txc - 1), G::TX, 1, SL + (me.tyc + 1) * P + C0 - 1, SL, 1, me.nzc, 1);
    if (nb(1, 1, 0, o)) add(base(o) + sec.ylo(0, 0), G::TX, 1, SL + (me.tyc + 1) * P + C0 + me.txc, SL, 1, me.nzc, 1);
  }
  // ---- z-halo planes: slot 0 (plane zb-1) from the high faces of the layer below, slot nzc+1
  // (plane zb+nzc) from the low faces of the layer above; each with its ring (star shapes: the
  // z-halo plane's ring is never read, only its interior)
  for (int side = 0; side < 2; side++) {
    const int dz = side == 0 ? -1 : 1;
    const int s0 = side == 0 ? 0 : (me.nzc + 1) * SL;
    auto face = [&](const BrickPos &q, int y, int x) {
      return base(q) + (side == 0 ? sec.zhi(y, x) : sec.zlo(y, x));
    };
    if (nb(0, 0, dz, o)) add(face(o, 0, 0), G::TX, 1, s0 + P + C0, P, 1, me.tyc, me.txc);
    if (!CORNERS) continue;
    if (nb(0, -1, dz, o)) add(face(o, o.tyc - 1, 0), 0, 1, s0 + C0, 0, 1, 1, me.txc);
    if (nb(0, 1, dz, o)) add(face(o, 0, 0), 0, 1, s0 + (me.tyc + 1) * P + C0, 0, 1, 1, me.txc);
    if (nb(-1, 0, dz, o)) add(face(o, 0, o.txc - 1), G::TX, 1, s0 + P + C0 - 1, P, 1, me.tyc, 1);
    if (nb(1, 0, dz, o)) add(face(o, 0, 0), G::TX, 1, s0 + P + C0 + me.txc, P, 1, me.tyc, 1);
    if (nb(-1, -1, dz, o)) add(face(o, o.tyc - 1, o.txc - 1), 0, 1, s0 + C0 - 1, 0, 1, 1, 1);
    if (nb(1, -1, dz, o)) add(face(o, o.tyc - 1, 0), 0, 1, s0 + C0 + me.txc, 0, 1, 1, 1);
    if (nb(-1, 1, dz, o)) add(face(o, 0, o.txc - 1), 0, 1, s0 + (me.tyc + 1) * P + C0 - 1, 0, 1, 1, 1);
    if (nb(1, 1, dz, o)) add(face(o, 0, 0), 0, 1, s0 + (me.tyc + 1) * P + C0 + me.txc, 0, 1, 1, 1);
  }
  return n;
}

// Halo refresh: every thread takes elements tid, tid + NT, ... of the segment list, issues up to
// kGatherMax tagged loads, then re-polls the words whose tag has not arrived (watchdog), and
// writes the values into the slots.
template <typename T>
__device__ __noinline__ void gather(const Seg *segs, int nseg, const LLWord *ll, unsigned tag, T *slots) {
  constexpr int W = LLG<T>::WORDS;
  const int total = nseg > 0 ? segs[nseg - 1].end : 0;
  // element e of the list -> (segment, kz, ki); e grows with k, so the segment index only moves
  // forward (nothing but the values is kept in registers between the passes below)
  auto locate = [&](int e, int &si, long long &src, int &dst) {
    while (segs[si].end <= e) si++;
    const Seg &sg = segs[si];
    const int rel = e - (sg.end - sg.nz * sg.ni);
    const int kz = rel / sg.ni, ki = rel - kz * sg.ni;
    src = sg.src + (long long)kz * sg.ssz + (long long)ki * sg.ssi;
    dst = sg.dst + kz * sg.dsz + ki * sg.dsi;
  };
  int si = 0;
  for (int e0 = (int)threadIdx.x; e0 < total; e0 += kBrickThreads * kGatherMax) {
    T val[kGatherMax];
    unsigned pend = 0;
    const int si0 = si;
#pragma unroll
    for (int k = 0; k < kGatherMax; k++) {
      const int e = e0 + k * kBrickThreads;
      if (e < total) {
        long long src;
        int dst;
        locate(e, si, src, dst);
        if (!LLG<T>::get(ll + src * W, tag, val[k])) pend |= 1u << k;
      }
    }
    if (pend) {
      const unsigned long long t0 = globaltimer_ns();
      while (pend) {
        int s2 = si0;
#pragma unroll
        for (int k = 0; k < kGatherMax; k++) {
          if ((pend >> k) & 1u) {
            long long src;
            int dst;
            locate(e0 + k * kBrickThreads, s2, src, dst);
            if (LLG<T>::get(ll + src * W, tag, val[k])) pend &= ~(1u << k);
          }
        }
        if (pend && globaltimer_ns() - t0 > PERKS_WATCHDOG_NS) watchdog_fire("perks3d brick halo", pend, tag);
      }
    }
    int s3 = si0;
#pragma unroll
    for (int k = 0; k < kGatherMax; k++) {
      const int e = e0 + k * kBrickThreads;
      if (e < total) {
        long long src;
        int dst;
        locate(e, s3, src, dst);
        slots[dst] = val[k];
      }
    }
  }
}

template <typename T, int S>
__global__ void __launch_bounds__(kBrickThreads, 1)
    perks3d_brick_kernel(const T *__restrict__ in, T *__restrict__ out, LLWord *__restrict__ xch, Dom3 d,
                         BrickGeo bg, int64_t steps, Coef<T, Shape<S>::N> c, int dbg) {
  using G = typename GBrick<T>::G;
  constexpr int W = LLG<T>::WORDS;
  constexpr bool CORNERS = has_corners<S>();  // shapes with diagonal terms read ring corners / z-halo rings
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T *slots = reinterpret_cast<T *>(smem_raw);
  __shared__ Seg segs[kMaxSegs];
  __shared__ int nseg_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const BrickPos me = brick_pos<G>(bg, d, (int)blockIdx.x);
  const Sec<G> sec{bg.NZ};
  const size_t nslot = (size_t)(me.nzc + 2) * G::SLOT;
  if (tid == 0) nseg_s = build_segs<G, CORNERS>(bg, d, me, segs);

  // ---- prologue: the brick and its halo box from `in` (zero outside the domain), the one-time
  // load half of A_gm's 2·D_cache term
  for (size_t i = tid; i < nslot; i += kBrickThreads) slots[i] = T(0);
  __syncthreads();
  {
    const int bx = me.txc + 2, by = me.tyc + 2, bzn = me.nzc + 2;
    const int tot = bx * by * bzn;
    for (int e = tid; e < tot; e += kBrickThreads) {
      const int i = e % bx, j = (e / bx) % by, k = e / (bx * by);
      const int x = me.x0 - 1 + i, y = me.y0 - 1 + j, z = me.zb - 1 + k;
      if (x < 0 || x >= d.nx || y < 0 || y >= d.ny || z < 0 || z >= d.nz) continue;
      slots[(size_t)k * G::SLOT + j * G::P + G::PAD - 1 + i] = in[((size_t)z * d.ny + y) * d.nx + x];
    }
  }
  __syncthreads();
  const int nseg = nseg_s;

  // ---- per-thread surface predicates (which exchange sections this thread's cells belong to)
  ThreadTile<G> tt;
  tt.init(d, me.x0, me.y0);
  const int xl0 = lane * G::V, yl0 = warp * G::R;
  const size_t xbase = (size_t)blockIdx.x * (size_t)bg.bw;
  auto publish = [&](LLWord *buf, unsigned tag, int o, const T (&v)[G::R][G::V]) {
    const bool zl = o == 0, zh = o == me.nzc - 1;
#pragma unroll
    for (int r = 0; r < G::R; r++) {
      const int yl = yl0 + r;
      if (yl >= me.tyc) continue;
#pragma unroll
      for (int i = 0; i < G::V; i++) {
        const int xl = xl0 + i;
        if (xl >= me.txc) continue;
        if (xl == 0) LLG<T>::put(buf + (xbase + sec.wcol(o, yl)) * W, v[r][i], tag);
        if (xl == me.txc - 1) LLG<T>::put(buf + (xbase + sec.ecol(o, yl)) * W, v[r][i], tag);
        if (yl == 0) LLG<T>::put(buf + (xbase + sec.ylo(o, xl)) * W, v[r][i], tag);
        if (yl == me.tyc - 1) LLG<T>::put(buf + (xbase + sec.yhi(o, xl)) * W, v[r][i], tag);
        if (zl) LLG<T>::put(buf + (xbase + sec.zlo(yl, xl)) * W, v[r][i], tag);
        if (zh) LLG<T>::put(buf + (xbase + sec.zhi(yl, xl)) * W, v[r][i], tag);
      }
    }
  };
  // a thread with no surface cell in the brick's inner planes skips the publish call there
  const bool edge_thread = xl0 == 0 || xl0 + G::V - 1 >= me.txc - 1 || yl0 == 0 || yl0 + G::R - 1 >= me.tyc - 1;
  const size_t par_words = (size_t)gridDim.x * (size_t)bg.bw * W;

  for (int64_t t = 0; t < steps; t++) {
    if (t > 0 && !(dbg & 1)) {  // 1. halo refresh: x^t surfaces of the neighbours (parity t&1, tag t)
      gather<T>(segs, nseg, xch + (size_t)(t & 1) * par_words, (unsigned)t, slots);
      __syncthreads();
    }
    // 2. sweep: arrivals of planes zb-1 .. zb+nzc (slots 0 .. nzc+1)
    const bool pub = t + 1 < steps && !(dbg & 2);
    LLWord *pbuf = xch + (size_t)((t + 1) & 1) * par_words;
    const unsigned ptag = (unsigned)(t + 1);
    StreamState<T, G> st;
    st.zero();
    for (int k = 0; k <= me.nzc + 1; k++) {
      if (k > 0) __syncthreads();  // every warp is done reading slot k-1 (arrival k-1)
      T o_[G::R][G::V], cq[G::R][G::V];
      arrival<T, S, G>(st, slots + (size_t)k * G::SLOT, c, o_, cq);
      if (k >= 2) {
        const int o = k - 2;  // brick-local plane of the finished output
        frame_select<T, G>(d, tt, me.zb + o, o_, st.cm1);
        if (pub && (edge_thread || o == 0 || o == me.nzc - 1)) publish(pbuf, ptag, o, o_);
        write_own<T, G>(slots + (size_t)(k - 1) * G::SLOT, o_);
      }
#pragma unroll
      for (int r = 0; r < G::R; r++)
#pragma unroll
        for (int i = 0; i < G::V; i++) st.cm1[r][i] = cq[r][i];
    }
    __syncthreads();
  }

  // ---- epilogue: the brick to `out` (the store half of 2·D_cache)
  {
    const int tot = me.txc * me.tyc * me.nzc;
    for (int e = tid; e < tot; e += kBrickThreads) {
      const int i = e % me.txc, j = (e / me.txc) % me.tyc, k = e / (me.txc * me.tyc);
      out[((size_t)(me.zb + k) * d.ny + (me.y0 + j)) * d.nx + me.x0 + i] =
          slots[(size_t)(k + 1) * G::SLOT + (j + 1) * G::P + G::PAD + i];
    }
  }
}

// ------------------------------------------------------------------ host side
namespace {
template <typename T> int brick_slot_bytes() { return (int)GBrick<T>::G::SLOT_BYTES; }
template <typename T> int brick_tx() { return GBrick<T>::G::TX; }
template <typename T> int brick_ty() { return GBrick<T>::G::TY; }
template <typename T> long long brick_bw(int NZ) { return brick_cells<typename GBrick<T>::G>(NZ); }
template <typename T> void *brick_kernel(int shape) {
  return shape == SHAPE_3D7    ? (void *)perks3d_brick_kernel<T, SHAPE_3D7>
         : shape == SHAPE_3D19 ? (void *)perks3d_brick_kernel<T, SHAPE_3D19>
                               : (void *)perks3d_brick_kernel<T, SHAPE_3D27>;
}
}  // namespace

// Plan: one brick per SM; the planner takes as many z layers as the SMs allow (smaller bricks,
// more parallel sweeps) and requires the brick (NZ + 2 slots) to fit in shared memory.
Plan plan_brick3d(const Problem &p) {
  Plan pl;
  pl.variant = PERKS_PERKS;
  if (p.ndim != 3 || (p.shape != SHAPE_3D7 && p.shape != SHAPE_3D27 && p.shape != SHAPE_3D19) ||
      p.bc != PERKS_BC_FRAME || p.nranks > 1) {
    pl.why = "brick3d: 3D 7/19/27pt FRAME, single GPU";
    return pl;
  }
  const bool f32 = p.dtype == PERKS_F32;
  const int TX = f32 ? brick_tx<float>() : brick_tx<double>();
  const int TY = f32 ? brick_ty<float>() : brick_ty<double>();
  const int slot = f32 ? brick_slot_bytes<float>() : brick_slot_bytes<double>();
  const int ntx = (int)((p.nx + TX - 1) / TX), nty = (int)((p.ny + TY - 1) / TY);
  const int tiles = ntx * nty;
  const int sms = env_int("PERKS_NUM_SMS", p.num_sms);
  if (tiles > sms) { pl.why = "brick3d: xy plane needs more tiles than SMs"; return pl; }
  int nbz = std::max(1, std::min<int>(sms / tiles, (int)p.nz));
  int NZ = (int)((p.nz + nbz - 1) / nbz);
  nbz = (int)((p.nz + NZ - 1) / NZ);
  const size_t smem = (size_t)(NZ + 2) * slot;
  if (smem > (size_t)p.max_smem_optin - 1024) { pl.why = "brick3d: brick does not fit in shared memory"; return pl; }
  void *k = f32 ? brick_kernel<float>(p.shape) : brick_kernel<double>(p.shape);
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    pl.why = "brick3d: cudaFuncSetAttribute";
    return pl;
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kBrickThreads, smem);
  if (occ < 1) { pl.why = "brick3d: not resident"; return pl; }
  pl.grid = tiles * nbz;
  pl.block = kBrickThreads;
  pl.ctas_per_sm = 1;
  pl.tile[0] = TX; pl.tile[1] = TY; pl.tile[2] = NZ;
  pl.zchunk = NZ;
  pl.regs = fa.numRegs;
  pl.smem = (int)smem;
  pl.units = pl.grid;
  pl.family = 6;  // (3D resident bricks)
  pl.cfg = nbz;
  const double S = (double)p.elem();
  pl.cached_smem = p.cells();
  pl.dram_bytes_step = 0.0;  // one-time 2·S·cells only (prologue + epilogue)
  const long long bw = f32 ? brick_bw<float>(NZ) : brick_bw<double>(NZ);
  const int W = f32 ? 1 : 2;
  pl.halo_bytes_step = 2.0 * (double)pl.grid * (double)bw * W * 8.0;  // publish + gather (tagged words)
  pl.ws_bytes = align256((size_t)2 * pl.grid * bw * W * sizeof(LLWord));
  snprintf(pl.name, sizeof(pl.name), "perks3d_brick_%s_%s_%dx%dx%d_%db",
           p.shape == SHAPE_3D7 ? "7pt" : p.shape == SHAPE_3D19 ? "19pt" : "27pt", f32 ? "f32" : "f64", TX, TY, NZ,
           pl.grid);
  pl.ok = true;
  return pl;
}

namespace {
template <typename T, int S>
cudaError_t launch_brick(const Problem &p, const Plan &pl, const T *in, T *out, void *ws, int64_t steps,
                         cudaStream_t s) {
  Coef<T, Shape<S>::N> c;
  for (int i = 0; i < Shape<S>::N; i++) c.w[i] = sizeof(T) == 4 ? (T)p.wf[i] : (T)p.wd[i];
  Dom3 d{(int)p.nx, (int)p.ny, (int)p.nz, 1, (int)p.nz - 2};
  BrickGeo bg;
  bg.ntx = (int)((p.nx + pl.tile[0] - 1) / pl.tile[0]);
  bg.nty = (int)((p.ny + pl.tile[1] - 1) / pl.tile[1]);
  bg.nbz = pl.cfg;
  bg.NZ = pl.tile[2];
  bg.bw = brick_bw<T>(bg.NZ);
  LLWord *xch = (LLWord *)ws;
  cudaError_t e = cudaMemsetAsync(xch, 0, pl.ws_bytes, s);  // tags restart at 1 every run
  if (e != cudaSuccess) return e;
  void *k = (void *)perks3d_brick_kernel<T, S>;
  int dbg = env_int("PERKS_BRICK_DEBUG", 0);  // timing experiments only: 1 skip the halo refresh, 2 skip publishing
  void *args[] = {(void *)&in, (void *)&out, (void *)&xch, (void *)&d, (void *)&bg, (void *)&steps, (void *)&c, (void *)&dbg};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(pl.block);
  cfg.dynamicSmemBytes = (size_t)pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // co-residency: bricks wait on their neighbours
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, k, args);
}
}  // namespace

cudaError_t run_brick3d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws, int64_t steps,
                        cudaStream_t s) {
  if (p.dtype == PERKS_F32)
    return p.shape == SHAPE_3D7    ? launch_brick<float, SHAPE_3D7>(p, pl, (const float *)in, (float *)out, ws, steps, s)
           : p.shape == SHAPE_3D19 ? launch_brick<float, SHAPE_3D19>(p, pl, (const float *)in, (float *)out, ws, steps, s)
                                   : launch_brick<float, SHAPE_3D27>(p, pl, (const float *)in, (float *)out, ws, steps, s);
  return p.shape == SHAPE_3D7    ? launch_brick<double, SHAPE_3D7>(p, pl, (const double *)in, (double *)out, ws, steps, s)
         : p.shape == SHAPE_3D19 ? launch_brick<double, SHAPE_3D19>(p, pl, (const double *)in, (double *)out, ws, steps, s)
                                 : launch_brick<double, SHAPE_3D27>(p, pl, (const double *)in, (double *)out, ws, steps, s);
}

}  // namespace perks
