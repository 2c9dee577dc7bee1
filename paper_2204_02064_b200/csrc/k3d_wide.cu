// k3d_wide.cu — host-loop (a), persistent (b) and PERKS (c) for GENERAL 3D point sets: any list of
// <= 64 offsets of radius <= 3, in any order (Table II 3d13pt, the radius-2 star, runs
// with a compile-time point set).  The FMA chain follows the list order (reading R5), so results
// are bit-identical to the oracle and across variants.
//
// One CTA owns a 32 x 16 (x, y) column of outputs and a chunk of KW3_ZC planes in z (one thread per
// (x, y)); it streams the input planes z0-r .. z0+ZC-1+r through a ring of 2r+1+LA shared-memory planes
// ((32+2r) x (16+2r), cp.async, zero outside the domain): planes z+r+1 .. z+r+LA are in flight
// while output plane z is computed from the 2r+1 resident planes.  Every input plane is read once per chunk
// ((16+2r)/16 x (32+2r)/32 x (ZC+2r)/ZC re-reads, served by the 126 MB L2).  (b) loops the units
// with a grid barrier per step (zig-zag order: odd steps run the units in reverse, so a step starts
// where the previous one ended, in L2 — [draft] P:395-404); (c) runs it with an empty on-chip cache
// split, the 3D policy of k3d_stream.cu measured there.  An earlier block kernel
// (32x8x8 output block + shell per CTA, no streaming) ran 3d13pt fp64 256^3 at 182.3 / 200.8 us/step
// (host loop / persistent); a double-buffered variant of it was slower still (231.9).
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "internal.h"
#include "stream3d.cuh"

namespace perks {

// TMA descriptors (k3d_stream.cu)
bool tma_available();
bool encode_map3(CUtensorMap *m, const Problem &p, const void *base, int bx, int by);

constexpr int KW3_TX = 32, KW3_TY = 16, KW3_THREADS = KW3_TX * KW3_TY, KW3_ZC = 32, KW3_MAXR = 3;
// planes in flight ahead of the one being waited for (one-plane lookahead ran 3d13pt fp64 256^3 at
// 176.5 us/step: each CTA waited out an L2/HBM round trip per plane)
#ifndef PERKS_W3_LA
#define PERKS_W3_LA 4
#endif
constexpr int KW3_LA = PERKS_W3_LA;

template <typename T> struct WideCoef3 {
  int n;
  int per;  // PERKS_BC_PERIODIC: indices wrap, every cell is updated (reading R1's alternative)
  int8_t dx[kMaxPoints2D], dy[kMaxPoints2D], dz[kMaxPoints2D];
  T w[kMaxPoints2D];
};

// Compile-time point sets: PS 1 = 3d13pt (the radius-2 star: centre + two points per half-axis),
// (dz,dy,dx) lexicographic.  PS 0 = any other list.
template <int PS> struct WideSet3;
template <> struct WideSet3<1> {
  static constexpr int R = 2, N = 13;
  // (dz, dy, dx) of point p, lexicographic
  static constexpr __host__ __device__ int dz(int p) { return p < 2 ? p - 2 : p < 11 ? 0 : p - 10; }
  static constexpr __host__ __device__ int dy(int p) { return p < 2 || p >= 11 ? 0 : p < 4 ? p - 4 : p < 9 ? 0 : p - 8; }
  static constexpr __host__ __device__ int dx(int p) { return p >= 4 && p < 9 ? p - 6 : 0; }
};

// Do all out-of-plane points of the set lie on the thread's own z column (dx = dy = 0)?  Then the
// column values of planes z-R .. z+R live in registers (2.5D blocking) and only plane z's in-plane
// neighbours are read from shared memory (3d13pt: 9 shared-memory loads per cell instead of 13).
template <int PS> constexpr bool column_only_dz() {
  for (int p = 0; p < WideSet3<PS>::N; p++)
    if (WideSet3<PS>::dz(p) != 0 && (WideSet3<PS>::dx(p) != 0 || WideSet3<PS>::dy(p) != 0)) return false;
  return true;
}

struct Blocks3 {
  int bx, by, bz;
};

// This thread's share of a plane window: up to KW3_CPT elements (smem index, x-y offset in the
// field, inside the x-y domain?), the same for every plane of the unit (no per-plane division).
constexpr int KW3_CPT = 2;  // (32+2r)(16+2r) <= 2 * 512 for r <= 3
struct PlaneCopy {
  int sidx[KW3_CPT];
  int gxy[KW3_CPT];  // -1: outside the x-y domain or beyond the window
};
PERKS_DEVINL PlaneCopy plane_copy(int nx, int ny, int x0, int y0, int r, bool per) {
  const int PX = KW3_TX + 2 * r, PXY = PX * (KW3_TY + 2 * r);
  PlaneCopy pc;
#pragma unroll
  for (int k = 0; k < KW3_CPT; k++) {
    const int i = threadIdx.x + k * KW3_THREADS;
    const int ly = i / PX, lx = i - ly * PX;
    int x = x0 - r + lx, y = y0 - r + ly;
    if (per) {  // r < extent: one wrap suffices
      x = x < 0 ? x + nx : (x >= nx ? x - nx : x);
      y = y < 0 ? y + ny : (y >= ny ? y - ny : y);
    }
    pc.sidx[k] = i;
    pc.gxy[k] = (i < PXY && x >= 0 && x < nx && y >= 0 && y < ny) ? y * nx + x : (i < PXY ? -1 : -2);
  }
  return pc;
}
// Issue the cp.async copies of input plane z into s (one commit group); zero outside the domain
// (FRAME), or plane z mod nz (PERIODIC).
template <typename T>
PERKS_DEVINL void load_plane3(const T *__restrict__ src, T *s, const PlaneCopy &pc, int nx, int ny, int nz, int z,
                              bool per) {
  if (per) z = z < 0 ? z + nz : (z >= nz ? z - nz : z);
  const bool zok = z >= 0 && z < nz;
  const T *pz = src + (size_t)(zok ? z : 0) * nx * ny;
#pragma unroll
  for (int k = 0; k < KW3_CPT; k++) {
    if (pc.gxy[k] == -2) continue;
    const bool ok = zok && pc.gxy[k] >= 0;
    cp_async<(int)sizeof(T)>(s + pc.sidx[k], ok ? pz + pc.gxy[k] : src, ok);
  }
  cp_async_commit();
}

// One unit (32 x 16 columns x ZC planes) of one step: src -> dst.  One CTA barrier per plane: after
// it every warp has finished the previous plane, so the slot of plane z-r-1 can be refilled.
template <typename T, int PS>
__device__ void unit3(const T *__restrict__ src, T *__restrict__ dst, int nx, int ny, int nz, int ux, int uy, int z0,
                      int z1, int r, const WideCoef3<T> &c, T *ring) {
  const int PX = KW3_TX + 2 * r, PXY = PX * (KW3_TY + 2 * r), NP = 2 * r + 1 + KW3_LA;
  const int x0 = ux * KW3_TX, y0 = uy * KW3_TY;
  const int lx = threadIdx.x % KW3_TX, ly = threadIdx.x / KW3_TX;
  const int x = x0 + lx, y = y0 + ly;
  const bool own = x < nx && y < ny;
  const bool inner_xy = x >= r && x < nx - r && y >= r && y < ny - r;
  const int cell = (ly + r) * PX + (lx + r);  // this thread's centre within a plane
  const bool per = c.per != 0;
  const PlaneCopy pc = plane_copy(nx, ny, x0, y0, r, per);
  // every warp has finished reading the previous unit's planes before the prefill overwrites their
  // slots (persistent kernels run several units per CTA back to back; this barrier used to follow
  // the prefill, a rare race: one failure of the C3-size PERIODIC persistent Fourier test in ~30)
  __syncthreads();
  // ring slot of input plane zz: (zz - (z0 - r)) mod NP; planes z0-r .. z0+r+LA-1 first (one
  // commit group each; planes past the chunk's last need are empty groups)
  for (int q = 0; q < 2 * r + KW3_LA; q++) {
    if (z0 - r + q < z1 + r) load_plane3(src, ring + q * PXY, pc, nx, ny, nz, z0 - r + q, per);
    else cp_async_commit();
  }
  int base = 0;     // slot of plane z - r
  constexpr bool COL = PS != 0 && column_only_dz<PS != 0 ? PS : 1>();
  constexpr int CR = PS != 0 ? WideSet3<PS != 0 ? PS : 1>::R : 0;
  T col[2 * CR + 1];  // COL: own-column values of planes z-R .. z+R
  for (int z = z0; z < z1; z++) {
    cp_async_wait<KW3_LA - 1>();  // plane z + r has landed
    __syncthreads();
    if constexpr (COL) {
      constexpr int QXY = (KW3_TX + 2 * CR) * (KW3_TY + 2 * CR), QP = 2 * CR + 1 + KW3_LA;
      if (z == z0) {
#pragma unroll
        for (int k = 0; k < 2 * CR; k++) col[k] = ring[(base + k) * QXY + cell];  // base = 0 here
      }
      int sl = base + 2 * CR;
      if (sl >= QP) sl -= QP;
      col[2 * CR] = ring[sl * QXY + cell];
    }
    {
      int sn = base + 2 * r + KW3_LA;  // plane z + r + LA -> the slot of plane z - r - 1
      if (sn >= NP) sn -= NP;
      if (z + r + KW3_LA < z1 + r) load_plane3(src, ring + sn * PXY, pc, nx, ny, nz, z + r + KW3_LA, per);
      else cp_async_commit();
    }
    if (own) {
      const bool inner = per || (inner_xy && z >= r && z < nz - r);
      int sc = base + r;
      if (sc >= NP) sc -= NP;
      T v;
      if (!inner) {
        v = ring[sc * PXY + cell];  // frame (reading R1)
      } else if constexpr (COL) {
        using WS = WideSet3<PS>;
        constexpr int R = WS::R, QX = KW3_TX + 2 * R, QXY = QX * (KW3_TY + 2 * R);
        const T *pz = ring + sc * QXY + cell;
        auto at = [&](int p) -> T {
          if (WS::dz(p) != 0 || (WS::dx(p) == 0 && WS::dy(p) == 0)) return col[WS::dz(p) + R];
          return pz[WS::dy(p) * QX + WS::dx(p)];
        };
        v = mul_rn(c.w[0], at(0));
#pragma unroll
        for (int p = 1; p < WS::N; p++) v = fma_rn(c.w[p], at(p), v);
      } else if constexpr (PS == 0) {
        auto at = [&](int p) {
          int sl = base + r + c.dz[p];
          if (sl >= NP) sl -= NP;
          return ring[sl * PXY + cell + c.dy[p] * PX + c.dx[p]];
        };
        v = mul_rn(c.w[0], at(0));
        for (int p = 1; p < c.n; p++) v = fma_rn(c.w[p], at(p), v);
      } else {
        using WS = WideSet3<PS>;
        constexpr int R = WS::R, QX = KW3_TX + 2 * R, QXY = QX * (KW3_TY + 2 * R), QP = 2 * R + 1 + KW3_LA;
        const T *pl[2 * R + 1];
#pragma unroll
        for (int k = 0; k <= 2 * R; k++) {
          int sl = base + k;
          if (sl >= QP) sl -= QP;
          pl[k] = ring + sl * QXY + cell;
        }
        v = mul_rn(c.w[0], pl[WS::dz(0) + R][WS::dy(0) * QX + WS::dx(0)]);
#pragma unroll
        for (int p = 1; p < WS::N; p++) v = fma_rn(c.w[p], pl[WS::dz(p) + R][WS::dy(p) * QX + WS::dx(p)], v);
      }
      dst[((size_t)z * ny + y) * nx + x] = v;
    }
    if constexpr (COL) {
#pragma unroll
      for (int k = 0; k < 2 * CR; k++) col[k] = col[k + 1];
    }
    if (++base == NP) base = 0;
  }
  cp_async_wait<0>();
}

template <typename T, int PS>
__global__ void __launch_bounds__(KW3_THREADS) wide3_hostloop_kernel(const T *__restrict__ src, T *__restrict__ dst,
                                                                     int nx, int ny, int nz, Blocks3 b, int zc, int r,
                                                                     const __grid_constant__ WideCoef3<T> c) {
  extern __shared__ __align__(16) unsigned char kw3_smem[];
  const int id = blockIdx.x, z0 = (id / (b.bx * b.by)) * zc;
  unit3<T, PS>(src, dst, nx, ny, nz, id % b.bx, (id / b.bx) % b.by, z0, min(z0 + zc, nz), r, c,
               reinterpret_cast<T *>(kw3_smem));
}

template <typename T, int PS>
__global__ void __launch_bounds__(KW3_THREADS) wide3_persistent_kernel(const T *__restrict__ in, T *out, T *tmp,
                                                                       int nx, int ny, int nz, Blocks3 b, int zc, int r,
                                                                       int64_t steps, unsigned *bar,
                                                                       const __grid_constant__ WideCoef3<T> c) {
  extern __shared__ __align__(16) unsigned char kw3_smem[];
  const int nb = b.bx * b.by * b.bz;
  for (int64_t t = 0; t < steps; t++) {
    const T *src = t == 0 ? in : ((((steps - t) & 1) == 0) ? out : tmp);
    T *dst = (((steps - 1 - t) & 1) == 0) ? out : tmp;
    // units strided over the grid (concurrent CTAs share halos in L2); odd steps in reverse order
    for (int i = blockIdx.x; i < nb; i += gridDim.x) {
      const int id = (t & 1) ? nb - 1 - i : i;
      const int z0 = (id / (b.bx * b.by)) * zc;
      unit3<T, PS>(src, dst, nx, ny, nz, id % b.bx, (id / b.bx) % b.by, z0, min(z0 + zc, nz), r, c,
                   reinterpret_cast<T *>(kw3_smem));
    }
    if (t + 1 < steps) grid_barrier(bar, (unsigned)(t + 1));
  }
}

// ------------------------------------------------------------------ TMA column kernel (3d13pt)
// The Table II 3d13pt preset (PS 1: every out-of-plane point on the cell's own z column) on a
// B200-style pipeline instead of per-element cp.async: one thread issues ONE tensor-box copy per
// input plane (the (TX+2r) x (TY+2r) window, out-of-domain cells zero-filled by the TMA unit) into
// a ring of NSL shared-memory slots, completing on the slot's mbarrier; a thread owns V cells in x
// (16 bytes) x RY rows, keeps its cells' values of planes o-r .. o+r in registers (the z terms)
// and reads only the in-plane neighbours of output plane o from the slot.  Per output plane and
// cell: 9 in-plane values shared across the thread's V x RY cells (row segments loaded once)
// instead of 13 scalar loads, no address arithmetic for the loads, one CTA barrier per plane.
// Same chain order (reading R5) as every other kernel: bit-identical results.
#ifndef PERKS_W3T_MINB
#define PERKS_W3T_MINB 2
#endif
constexpr int KT3_NW = 8, KT3_RY = 2, KT3_NT = 32 * KT3_NW, KT3_TY = KT3_NW * KT3_RY, KT3_LA = 3;
template <typename T> struct KT3 {
  static constexpr int V = 16 / (int)sizeof(T), TX = 32 * V;
  static constexpr int R = WideSet3<1>::R;
  // the box starts PX = R rounded up to 16 bytes left of the tile: the tensor copy's innermost
  // start must be 16-byte aligned (an fp32 box starting 8 bytes off faults as an illegal
  // instruction on B200)
  static constexpr int PX = (R * (int)sizeof(T) + 15) / 16 * 16 / (int)sizeof(T);
  static constexpr int BX = TX + 2 * PX;  // box width (a 16-byte multiple)
  static constexpr int BY = KT3_TY + 2 * R;
  static constexpr int SLOT = (BX * BY * (int)sizeof(T) + 127) / 128 * 128 / (int)sizeof(T);
  static constexpr int NSL = R + 1 + KT3_LA;  // plane o's window + planes up to o+r+LA in flight
  static constexpr size_t SMEM = (size_t)NSL * SLOT * sizeof(T) + 128;  // + mbarriers
};

struct WideMaps3 {
  CUtensorMap m[3];  // in, out, tmp: box {BX, BY, 1}
};

// The units a CTA runs in one step, as one stream of plane arrivals: unit j (id(j)) = tile
// (x0, y0), output planes [z0, z1); its arrivals are input planes z0-R .. z1+R-1.  Plane q's own
// cells enter the column window when it lands; output o = q - R is computed while plane q is
// resident (its in-plane window is the slot of arrival k - R).  The TMA producer (thread 0) runs
// NSL arrivals ahead of the consumers ACROSS unit boundaries, so a CTA's next unit is already
// loading while it finishes the current one (no ring drain/refill per unit).  `k` = running
// arrival counter over the whole launch (slot = k % NSL, mbarrier parity = (k / NSL) & 1).
struct Unit3t {
  int x0, y0, z0, z1;
};
template <typename T, class Units>
__device__ void stream3t(const CUtensorMap *map, T *__restrict__ dst, int nx, int ny, int nz, const Units &units,
                         int nu, const WideCoef3<T> &c, T *ring, uint64_t *bars, unsigned &k) {
  using K = KT3<T>;
  using WS = WideSet3<1>;
  constexpr int R = K::R, V = K::V, NSL = K::NSL;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int xl = lane * V, yl = w * KT3_RY;  // tile-local first cell
  if (nu <= 0) return;
  // producer cursor (thread 0 only): unit jp, next plane qp
  int jp = 0, qp = 0;
  Unit3t up = units(0);
  qp = up.z0 - R;
  auto issue_one = [&](unsigned kk) {  // issue the producer cursor's arrival as arrival kk
    if (jp >= nu) return;
    if (qp >= 0 && qp < nz) {
      mbar_arrive_tx(bars + kk % NSL, (unsigned)(K::BX * K::BY * sizeof(T)));
      tma_load_3d(ring + (size_t)(kk % NSL) * K::SLOT, map, up.x0 - K::PX, up.y0 - R, qp, bars + kk % NSL);
    } else {
      mbar_arrive(bars + kk % NSL);  // outside the domain: complete the phase without data
    }
    if (++qp == up.z1 + R && ++jp < nu) {
      up = units(jp);
      qp = up.z0 - R;
    }
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < NSL; i++) issue_one(k + i);
  T col[2 * R + 1][KT3_RY][V];  // own cells of planes o-R .. o+R (index 2R = newest)
  unsigned kstart = k;           // first arrival of the current unit
  for (int j = 0; j < nu; j++) {
    const Unit3t u = units(j);
    const int q0 = u.z0 - R, q1 = u.z1 + R;
#pragma unroll
    for (int a = 0; a < 2 * R + 1; a++)
#pragma unroll
      for (int ry = 0; ry < KT3_RY; ry++)
#pragma unroll
        for (int v = 0; v < V; v++) col[a][ry][v] = T(0);
    for (int q = q0; q < q1; q++, k++) {
      const unsigned sl = k % NSL;
      mbar_wait(bars + sl, (k / NSL) & 1);
      const T *pq = ring + (size_t)sl * K::SLOT;
#pragma unroll
      for (int a = 0; a < 2 * R; a++)
#pragma unroll
        for (int ry = 0; ry < KT3_RY; ry++)
#pragma unroll
          for (int v = 0; v < V; v++) col[a][ry][v] = col[a + 1][ry][v];
      const bool qin = q >= 0 && q < nz;
#pragma unroll
      for (int ry = 0; ry < KT3_RY; ry++) {
        T own[V];
        const T *src = pq + (size_t)(yl + ry + R) * K::BX + xl + K::PX;
        if constexpr ((K::PX * sizeof(T)) % 16 == 0) vload<T, V>(own, src);
        else
#pragma unroll
          for (int v = 0; v < V; v++) own[v] = src[v];
#pragma unroll
        for (int v = 0; v < V; v++) col[2 * R][ry][v] = qin ? own[v] : T(0);
      }
      const int o = q - R;
      if (o >= u.z0) {  // output plane o: in-plane window = the slot of arrival k - R
        const T *po = ring + (size_t)((k - R) % NSL) * K::SLOT;
        const bool zin = o >= R && o < nz - R;
#pragma unroll
        for (int ry = 0; ry < KT3_RY; ry++) {
          const int y = u.y0 + yl + ry;
          // row segments: centre row x-R .. x+V+R-1, rows y+dy (dy != 0) at x .. x+V-1
          T seg[2 * R + 1][V + 2 * R];
#pragma unroll
          for (int dy = -R; dy <= R; dy++) {
            const T *row = po + (size_t)(yl + ry + R + dy) * K::BX + xl + K::PX - R;
            if (dy == 0) {
#pragma unroll
              for (int i = 0; i < V + 2 * R; i++) seg[dy + R][i] = row[i];
            } else {
#pragma unroll
              for (int i = 0; i < V; i++) seg[dy + R][i + R] = row[i + R];
            }
          }
          T out[V];
#pragma unroll
          for (int v = 0; v < V; v++) {
            const int x = u.x0 + xl + v;
            auto at = [&](int p) -> T {
              if (WS::dz(p) != 0 || (WS::dx(p) == 0 && WS::dy(p) == 0)) return col[WS::dz(p) + R][ry][v];
              return seg[WS::dy(p) + R][v + R + WS::dx(p)];
            };
            T a = mul_rn(c.w[0], at(0));
#pragma unroll
            for (int p = 1; p < WS::N; p++) a = fma_rn(c.w[p], at(p), a);
            const bool inner = zin && x >= R && x < nx - R && y >= R && y < ny - R;
            out[v] = inner ? a : col[R][ry][v];  // frame (reading R1): the input value
          }
          if (y < ny) {
            T *d = dst + ((size_t)o * ny + y) * nx + u.x0 + xl;
            if (u.x0 + xl + V <= nx) vstore<T, V>(d, out);
            else
#pragma unroll
              for (int v = 0; v < V; v++)
                if (u.x0 + xl + v < nx) d[v] = out[v];
          }
        }
      }
      // every warp is done with the slot of arrival k - R after this barrier (the window of output
      // o, or a plane no output of its unit reads): the producer refills it with the next arrival
      __syncthreads();
      if (threadIdx.x == 0 && k >= kstart + R) issue_one(k - R + NSL);
    }
  }
  (void)kstart;
}

template <typename T>
PERKS_DEVINL void kt3_init(T *&ring, uint64_t *&bars) {
  extern __shared__ __align__(128) unsigned char kt3_smem[];
  ring = reinterpret_cast<T *>(kt3_smem);
  bars = reinterpret_cast<uint64_t *>(kt3_smem + (size_t)KT3<T>::NSL * KT3<T>::SLOT * sizeof(T));
  if (threadIdx.x == 0) {
    for (int i = 0; i < KT3<T>::NSL; i++) mbar_init(bars + i, 1);
    mbar_fence_init();
  }
  __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(KT3_NT, PERKS_W3T_MINB) wide3t_hostloop_kernel(const __grid_constant__ WideMaps3 maps, int src_idx,
                                                                T *__restrict__ dst, int nx, int ny, int nz, Blocks3 b,
                                                                int zc, const __grid_constant__ WideCoef3<T> c) {
  T *ring;
  uint64_t *bars;
  kt3_init<T>(ring, bars);
  const int id = blockIdx.x, z0 = (id / (b.bx * b.by)) * zc;
  const Unit3t u1{(id % b.bx) * KT3<T>::TX, ((id / b.bx) % b.by) * KT3_TY, z0, min(z0 + zc, nz)};
  unsigned k = 0;
  stream3t<T>(&maps.m[src_idx], dst, nx, ny, nz, [&](int) { return u1; }, 1, c, ring, bars, k);
}

template <typename T>
__global__ void __launch_bounds__(KT3_NT, PERKS_W3T_MINB) wide3t_persistent_kernel(const __grid_constant__ WideMaps3 maps, T *out,
                                                                  T *tmp, int nx, int ny, int nz, Blocks3 b, int zc,
                                                                  int64_t steps, unsigned *bar,
                                                                  const __grid_constant__ WideCoef3<T> c) {
  T *ring;
  uint64_t *bars;
  kt3_init<T>(ring, bars);
  const int nb = b.bx * b.by * b.bz;
  unsigned k = 0;
  for (int64_t t = 0; t < steps; t++) {
    const int si = t == 0 ? 0 : ((((steps - t) & 1) == 0) ? 1 : 2);
    T *dst = (((steps - 1 - t) & 1) == 0) ? out : tmp;
    // this CTA's units blockIdx.x, +gridDim.x, ...; odd steps in reverse order (zig-zag)
    const int nu = blockIdx.x < nb ? (nb - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    auto unit = [&](int j) -> Unit3t {
      const int i = (int)blockIdx.x + j * (int)gridDim.x;
      const int id = (t & 1) ? nb - 1 - i : i;
      const int z0 = (id / (b.bx * b.by)) * zc;
      return Unit3t{(id % b.bx) * KT3<T>::TX, ((id / b.bx) % b.by) * KT3_TY, z0, min(z0 + zc, nz)};
    };
    stream3t<T>(&maps.m[si], dst, nx, ny, nz, unit, nu, c, ring, bars, k);
    if (t + 1 < steps) {
      grid_barrier(bar, (unsigned)(t + 1));
      // the step's outputs were written through the generic proxy; the next step reads them with TMA
      asm volatile("fence.proxy.async.global;\n" ::: "memory");
    }
  }
}

// ------------------------------------------------------------------ host side
namespace {
int radius3d(const Problem &p) {
  int r = 0;
  for (int i = 0; i < p.npts; i++)
    r = std::max(r, std::max(std::abs(p.off[i][0]), std::max(std::abs(p.off[i][1]), std::abs(p.off3z[i]))));
  return r;
}
int wide3_preset(const Problem &p) {
  if (p.npts != WideSet3<1>::N) return 0;
  for (int q = 0; q < WideSet3<1>::N; q++)
    if (p.off[q][0] != WideSet3<1>::dx(q) || p.off[q][1] != WideSet3<1>::dy(q) || p.off3z[q] != WideSet3<1>::dz(q))
      return 0;
  return 1;
}
template <typename T> WideCoef3<T> make_coef3(const Problem &p) {
  WideCoef3<T> c{};
  c.n = p.npts;
  c.per = p.bc == PERKS_BC_PERIODIC ? 1 : 0;
  for (int i = 0; i < p.npts; i++) {
    c.dx[i] = (int8_t)p.off[i][0];
    c.dy[i] = (int8_t)p.off[i][1];
    c.dz[i] = (int8_t)p.off3z[i];
    c.w[i] = sizeof(T) == 4 ? (T)p.wf[i] : (T)p.wd[i];
  }
  return c;
}
template <typename T> void *wk3t(bool hostloop) {
  return hostloop ? (void *)wide3t_hostloop_kernel<T> : (void *)wide3t_persistent_kernel<T>;
}
template <typename T> void *wk3(bool hostloop, int ps) {
  if (hostloop) return ps == 1 ? (void *)wide3_hostloop_kernel<T, 1> : (void *)wide3_hostloop_kernel<T, 0>;
  return ps == 1 ? (void *)wide3_persistent_kernel<T, 1> : (void *)wide3_persistent_kernel<T, 0>;
}
size_t smem3(int r, size_t S) {  // the ring: 2r+1+LA planes of (32+2r) x (16+2r)
  return (size_t)(2 * r + 1 + KW3_LA) * (KW3_TX + 2 * r) * (KW3_TY + 2 * r) * S;
}
}  // namespace

Plan plan_wide3d(const Problem &p, perks_variant v) {
  Plan pl;
  pl.variant = v;
  const int r = radius3d(p);
  if (p.ndim != 3 || p.shape != SHAPE_G3D || r > KW3_MAXR) {
    pl.why = "wide3d: 3D point sets of radius <= 3";
    return pl;
  }
  const bool f32 = p.dtype == PERKS_F32, hostloop = v == PERKS_HOSTLOOP;
  const int ps = wide3_preset(p);
  // the TMA column kernel for the 3d13pt preset (16-byte aligned rows for the tensor map)
  const bool tk = ps == 1 && p.bc == PERKS_BC_FRAME && (p.nx * (int64_t)p.elem()) % 16 == 0 && p.nx >= 8 && tma_available() &&
                  env_int("PERKS_W3_TMA", 1) != 0;
  void *k = tk ? (f32 ? wk3t<float>(hostloop) : wk3t<double>(hostloop))
               : (f32 ? wk3<float>(hostloop, ps) : wk3<double>(hostloop, ps));
  const size_t smem = tk ? (f32 ? KT3<float>::SMEM : KT3<double>::SMEM) : smem3(r, p.elem());
  const int threads = tk ? KT3_NT : KW3_THREADS;
  const int TXu = tk ? (f32 ? KT3<float>::TX : KT3<double>::TX) : KW3_TX, TYu = tk ? KT3_TY : KW3_TY;
  if (smem > (size_t)p.max_smem_optin) { pl.why = "wide3d: block does not fit shared memory"; return pl; }
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    pl.why = "cudaFuncSetAttribute";
    return pl;
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) { pl.why = "cudaFuncGetAttributes"; return pl; }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, smem);
  if (occ < 1) { pl.why = "wide3d: not resident"; return pl; }
  const int bx = (int)((p.nx + TXu - 1) / TXu), by = (int)((p.ny + TYu - 1) / TYu);
  // z-chunk length: balance the units over the resident CTAs (whole waves) against the 2r-plane
  // re-read per chunk
  const int64_t G = (int64_t)occ * p.num_sms;
  int zc = KW3_ZC;
  double best = -1;
  for (int z = 16; z <= 64; z++) {
    const int64_t u = (int64_t)bx * by * ((p.nz + z - 1) / z);
    const double eff = (double)u / (double)(((u + G - 1) / G) * G) * (double)z / (double)(z + 2 * r);
    if (eff > best + 1e-9) { best = eff; zc = z; }
  }
  const int bz = (int)((p.nz + zc - 1) / zc);
  const int64_t blocks = (int64_t)bx * by * bz;
  pl.units = blocks;
  // persistent: every resident CTA, each with an equal share of the planes
  pl.grid = hostloop ? (int)blocks : (int)std::min<int64_t>(blocks, G);
  pl.block = threads;
  pl.ctas_per_sm = occ;
  pl.tile[0] = TXu; pl.tile[1] = TYu; pl.tile[2] = zc;
  pl.regs = fa.numRegs;
  pl.smem = (int)smem;
  pl.cfg = tk ? 2 : ps;
  pl.family = 5;  // (wide 3D)
  const double S = (double)p.elem();
  pl.dram_bytes_step = 2.0 * S * (double)p.cells();
  pl.halo_bytes_step = S * (double)blocks *  // window re-reads per unit (L2)
                       ((double)(TXu + 2 * r) * (TYu + 2 * r) * (zc + 2 * r) - (double)TXu * TYu * zc);
  pl.ws_bytes = align256((size_t)p.cells() * p.elem()) + (hostloop ? 0 : 256);
  snprintf(pl.name, sizeof(pl.name), "%s3d_wide_r%d_%dpt%s_%s%s%s%s", v == PERKS_PERKS ? "perks" : hostloop ? "hostloop" : "persistent",
           r, p.npts, ps ? "" : "_any", f32 ? "f32" : "f64", tk ? "_tma" : "",
           p.bc == PERKS_BC_PERIODIC ? "_per" : "", v == PERKS_PERKS ? "_c0" : "");
  pl.ok = true;
  return pl;
}

namespace {
template <typename T>
cudaError_t run_wide3_t(const Problem &p, const Plan &pl, const T *in, T *out, void *ws, int64_t steps,
                        cudaStream_t s) {
  const WideCoef3<T> c = make_coef3<T>(p);
  int r = radius3d(p);
  int nx = (int)p.nx, ny = (int)p.ny, nz = (int)p.nz;
  int zc = pl.tile[2];
  Blocks3 b{(nx + pl.tile[0] - 1) / pl.tile[0], (ny + pl.tile[1] - 1) / pl.tile[1], (nz + zc - 1) / zc};
  T *tmp = (T *)ws;
  if (pl.cfg == 2) {  // TMA column kernel
    WideMaps3 maps;
    const void *bs[3] = {in, out, tmp};
    for (int i = 0; i < 3; i++)
      if (!encode_map3(&maps.m[i], p, bs[i], KT3<T>::BX, KT3<T>::BY)) return cudaErrorInvalidValue;
    void *k = wk3t<T>(pl.variant == PERKS_HOSTLOOP);
    if (pl.variant == PERKS_HOSTLOOP) {
      for (int64_t t = 0; t < steps; t++) {
        int si = t == 0 ? 0 : ((((steps - t) & 1) == 0) ? 1 : 2);
        T *dst = (((steps - 1 - t) & 1) == 0) ? out : tmp;
        void *args[] = {(void *)&maps, (void *)&si, (void *)&dst, (void *)&nx, (void *)&ny, (void *)&nz, (void *)&b,
                        (void *)&zc, (void *)&c};
        cudaError_t e = cudaLaunchKernel(k, dim3(pl.grid), dim3(KT3_NT), args, pl.smem, s);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    }
    unsigned *bar = (unsigned *)((char *)ws + align256((size_t)p.cells() * p.elem()));
    cudaError_t e = reset_grid_barrier(bar, s);
    if (e != cudaSuccess) return e;
    void *args[] = {(void *)&maps, (void *)&out, (void *)&tmp, (void *)&nx, (void *)&ny, (void *)&nz, (void *)&b,
                    (void *)&zc, (void *)&steps, (void *)&bar, (void *)&c};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.grid);
    cfg.blockDim = dim3(KT3_NT);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, k, args);
  }
  void *k = wk3<T>(pl.variant == PERKS_HOSTLOOP, pl.cfg);
  if (pl.variant == PERKS_HOSTLOOP) {
    for (int64_t t = 0; t < steps; t++) {
      const T *src = t == 0 ? in : ((((steps - t) & 1) == 0) ? out : tmp);
      T *dst = (((steps - 1 - t) & 1) == 0) ? out : tmp;
      void *args[] = {(void *)&src, (void *)&dst, (void *)&nx, (void *)&ny, (void *)&nz, (void *)&b, (void *)&zc,
                      (void *)&r, (void *)&c};
      cudaError_t e = cudaLaunchKernel(k, dim3(pl.grid), dim3(KW3_THREADS), args, pl.smem, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  unsigned *bar = (unsigned *)((char *)ws + align256((size_t)p.cells() * p.elem()));
  cudaError_t e = reset_grid_barrier(bar, s);
  if (e != cudaSuccess) return e;
  void *args[] = {(void *)&in, (void *)&out, (void *)&tmp, (void *)&nx, (void *)&ny, (void *)&nz, (void *)&b,
                  (void *)&zc, (void *)&r, (void *)&steps, (void *)&bar, (void *)&c};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(KW3_THREADS);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, k, args);
}
}  // namespace

cudaError_t run_wide3d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws, int64_t steps,
                       cudaStream_t s) {
  if (p.dtype == PERKS_F32) return run_wide3_t<float>(p, pl, (const float *)in, (float *)out, ws, steps, s);
  return run_wide3_t<double>(p, pl, (const double *)in, (double *)out, ws, steps, s);
}

}  // namespace perks
