// stream3d.cuh — the 3D plane-streaming compute body shared by the host-loop (a), persistent (b)
// and PERKS (c) variants.  "2D planes are loaded one after the other in shared memory, and each
// thread computes the cells in a vertical direction".
//
// A CTA owns an xy tile of TX x TY cells (TX = 32*V: one warp spans x; TY = NWARP*R) and a z range.
// Planes arrive in increasing z into a ring of NS shared-memory slots (cp.async, NS-1 planes in
// flight).  Each slot holds the tile plus a one-cell halo ring; rows are padded so the interior
// starts 16-byte aligned.  Thread (lane, warp) owns V x R cells of every plane.  When plane q is
// resident, the chain terms of outputs q+1 / q / q-1 that read plane q are applied in list order
// (stages A/B/C of shapes.cuh), so each plane is read from shared memory once per thread.
#pragma once
#include "common.cuh"
#include "shapes.cuh"

namespace perks {

template <typename T, int V_, int R_, int NWARP_, int NS_>
struct Geo3D {
  static constexpr int V = V_, R = R_, NWARP = NWARP_, NS = NS_;
  static constexpr int NT = 32 * NWARP;
  static constexpr int TX = 32 * V, TY = NWARP * R;
  static constexpr int PAD = 16 / (int)sizeof(T);  // interior starts 16-B aligned
  static constexpr int P = TX + 2 * PAD;             // row pitch (elements)
  static constexpr int ROWS = TY + 2;
  static constexpr int SLOT = ROWS * P;              // elements per slot
  static constexpr size_t SLOT_BYTES = (size_t)SLOT * sizeof(T);
  static_assert(V * (int)sizeof(T) == 16, "one 16-byte vector per thread per row");
  static_assert(NT >= 2 * ROWS, "halo-column loaders");
};

struct Dom3 {
  int nx, ny, nz;
};

// Issue cp.async copies of plane q of `src` (tile origin x0,y0) into `slot`.  Cells outside the
// domain are zero-filled (they only feed frame cells, whose results are discarded).
// If `halo_only`, only the one-cell ring around the tile is fetched (PERKS cached planes).
template <typename T, class G>
PERKS_DEVINL void issue_plane(T *slot, const T *__restrict__ src, const Dom3 &d, int q, int x0,
                              int y0, bool halo_only) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool zin = q >= 0 && q < d.nz;
  const size_t pl = (size_t)d.nx * d.ny;
  const T *base = src + (zin ? (size_t)q * pl : 0);
  const int x = x0 + lane * G::V;
  const bool xin = x < d.nx;
  // own rows (tile interior)
  // one row segment of V cells: a 16-byte copy when rows are vector aligned (nx % V == 0),
  // else V element copies with per-element bounds (ragged nx)
  const bool vec = (d.nx % G::V) == 0;
  auto seg = [&](int j, bool rowok) {
    const int y = y0 - 1 + j;
    T *s = slot + j * G::P + G::PAD + lane * G::V;
    if (vec) {
      const bool ok = rowok && xin;
      cp_async<16>(s, ok ? base + (size_t)y * d.nx + x : src, ok);
    } else {
#pragma unroll
      for (int i = 0; i < G::V; i++) {
        const bool ok = rowok && x + i < d.nx;
        cp_async<(int)sizeof(T)>(s + i, ok ? base + (size_t)y * d.nx + x + i : src, ok);
      }
    }
  };
  if (!halo_only) {
#pragma unroll
    for (int r = 0; r < G::R; r++) {
      const int j = warp * G::R + r + 1;  // slot row
      seg(j, zin && (y0 - 1 + j) < d.ny);
    }
  }
  // halo rows y0-1 (warp 0) and y0+TY (last warp)
  if (warp == 0 || warp == G::NWARP - 1) {
    const int j = warp == 0 ? 0 : G::ROWS - 1;
    const int y = y0 - 1 + j;
    seg(j, zin && y >= 0 && y < d.ny);
  }
  // halo columns x0-1 and x0+TX for all ROWS rows (corners included)
  if (tid < 2 * G::ROWS) {
    const int j = tid >> 1;
    const bool right = tid & 1;
    const int y = y0 - 1 + j;
    const int xx = right ? x0 + G::TX : x0 - 1;
    const bool ok = zin && y >= 0 && y < d.ny && xx >= 0 && xx < d.nx;
    const T *g = ok ? base + (size_t)y * d.nx + xx : src;
    cp_async<(int)sizeof(T)>(slot + j * G::P + (right ? G::PAD + G::TX : G::PAD - 1), g, ok);
  }
}

// Neighbourhood of the thread's V x R cells in one resident plane:
// nb[j][i] = cell (x - 1 + i, y - 1 + j) for j in [0, R+2), i in [0, V+2).
template <typename T, class G>
PERKS_DEVINL void read_nb(const T *slot, T (&nb)[G::R + 2][G::V + 2]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int j = 0; j < G::R + 2; j++) {
    const T *row = slot + (warp * G::R + j) * G::P;
    T v[G::V];
    vload<T, G::V>(v, row + G::PAD + lane * G::V);
    const T l = __shfl_up_sync(0xffffffffu, v[G::V - 1], 1);
    const T r = __shfl_down_sync(0xffffffffu, v[0], 1);
    nb[j][0] = lane == 0 ? row[G::PAD - 1] : l;
    nb[j][G::V + 1] = lane == 31 ? row[G::PAD + G::TX] : r;
#pragma unroll
    for (int i = 0; i < G::V; i++) nb[j][i + 1] = v[i];
  }
}

// Apply chain terms [PB, PE) of shape S for all V x R cells.  Terms with dz == DZ_NB read the
// resident plane (nb); other terms read the retained centre values `cen` (checked at compile time
// by stage_end in shapes.cuh).
template <typename T, int S, class G, int PB, int PE, int DZ_NB>
PERKS_DEVINL void apply_terms(T (&acc)[G::R][G::V], const T (&nb)[G::R + 2][G::V + 2],
                              const T (&cen)[G::R][G::V], const Coef<T, Shape<S>::N> &c) {
#pragma unroll
  for (int p = PB; p < PE; p++) {
#pragma unroll
    for (int r = 0; r < G::R; r++) {
#pragma unroll
      for (int i = 0; i < G::V; i++) {
        const T val = (Shape<S>::dz(p) == DZ_NB)
                          ? nb[r + 1 + Shape<S>::dy(p)][i + 1 + Shape<S>::dx(p)]
                          : cen[r][i];
        acc[r][i] = (p == 0) ? mul_rn(c.w[0], val) : fma_rn(c.w[p], val, acc[r][i]);
      }
    }
  }
}

// Per-thread streaming state across arrivals.
template <typename T, class G>
struct StreamState {
  T accA[G::R][G::V];  // output q+1 (chain prefix with dz=-1)
  T accB[G::R][G::V];  // output q
  T accC[G::R][G::V];  // output q-1
  T cm1[G::R][G::V];   // centre of the previous plane (q-1)
};

// Process the arrival of plane q (resident in `slot`): finish output q-1 (returned in `out`,
// frame cells replaced by their old value), advance outputs q and q+1, rotate the state.
// `center_out` receives the centre values of plane q (the thread's own cells).
template <typename T, int S, class G>
PERKS_DEVINL void arrival(StreamState<T, G> &st, const T *slot, const Coef<T, Shape<S>::N> &c,
                          T (&out)[G::R][G::V], T (&center_q)[G::R][G::V]) {
  constexpr int e0 = stage_end<S>(0), e1 = stage_end<S>(1), e2 = stage_end<S>(2);
  T nb[G::R + 2][G::V + 2];
  read_nb<T, G>(slot, nb);
#pragma unroll
  for (int r = 0; r < G::R; r++)
#pragma unroll
    for (int i = 0; i < G::V; i++) center_q[r][i] = nb[r + 1][i + 1];
  // stage C: output q-1 reads plane q (dz=+1) or its own retained centre (dz=0)
  apply_terms<T, S, G, e1, e2, 1>(st.accC, nb, st.cm1, c);
#pragma unroll
  for (int r = 0; r < G::R; r++)
#pragma unroll
    for (int i = 0; i < G::V; i++) out[r][i] = st.accC[r][i];
  // stage B: output q reads plane q (dz=0) or retained centre of q-1 (dz=-1)
  apply_terms<T, S, G, e0, e1, 0>(st.accB, nb, st.cm1, c);
  // stage A: output q+1 reads plane q (dz=-1)
  apply_terms<T, S, G, 0, e0, -1>(st.accA, nb, st.cm1, c);
#pragma unroll
  for (int r = 0; r < G::R; r++)
#pragma unroll
    for (int i = 0; i < G::V; i++) {
      st.accC[r][i] = st.accB[r][i];
      st.accB[r][i] = st.accA[r][i];
    }
}

// Frame select + store of output plane o.  `old` = the plane's step-k values (centre).
template <typename T, class G>
PERKS_DEVINL void store_plane(T *__restrict__ dst, const Dom3 &d, int o, int x0, int y0,
                              const T (&val)[G::R][G::V], const T (&old)[G::R][G::V]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x = x0 + lane * G::V;
  if (x >= d.nx) return;
  const bool zint = o >= 1 && o <= d.nz - 2;
  T *base = dst + (size_t)o * d.nx * d.ny;
#pragma unroll
  for (int r = 0; r < G::R; r++) {
    const int y = y0 + warp * G::R + r;
    if (y >= d.ny) break;
    const bool yint = zint && y >= 1 && y <= d.ny - 2;
    T v[G::V];
#pragma unroll
    for (int i = 0; i < G::V; i++) {
      const bool inter = yint && (x + i) >= 1 && (x + i) <= d.nx - 2;
      v[i] = inter ? val[r][i] : old[r][i];
    }
    if ((d.nx % G::V) == 0) {
      vstore<T, G::V>(base + (size_t)y * d.nx + x, v);
    } else {
#pragma unroll
      for (int i = 0; i < G::V; i++)
        if (x + i < d.nx) base[(size_t)y * d.nx + x + i] = v[i];
    }
  }
}

// Stream one unit (tile x0,y0; planes [zs, ze)) of one time step from src to dst.
// All slots must be free on entry (caller synchronises); leaves no copies in flight that target
// slots still being read.
template <typename T, int S, class G>
PERKS_DEVINL void stream_unit(T *smem, const T *__restrict__ src, T *__restrict__ dst,
                              const Dom3 &d, int x0, int y0, int zs, int ze,
                              const Coef<T, Shape<S>::N> &c) {
  constexpr int D = G::NS - 1;
  const int q0 = zs - 1, qn = ze;  // arrivals q0..qn inclusive
  const int narr = qn - q0 + 1;
#pragma unroll
  for (int k = 0; k < D; k++) {
    if (k < narr) issue_plane<T, G>(smem + (size_t)(k % G::NS) * G::SLOT, src, d, q0 + k, x0, y0, false);
    cp_async_commit();
  }
  StreamState<T, G> st;
#pragma unroll
  for (int r = 0; r < G::R; r++)
#pragma unroll
    for (int i = 0; i < G::V; i++) st.accA[r][i] = st.accB[r][i] = st.accC[r][i] = st.cm1[r][i] = T(0);
  for (int k = 0; k < narr; k++) {
    const int q = q0 + k;
    cp_async_wait<D - 1>();
    __syncthreads();
    if (k + D < narr)
      issue_plane<T, G>(smem + (size_t)((k + D) % G::NS) * G::SLOT, src, d, q + D, x0, y0, false);
    cp_async_commit();
    T out[G::R][G::V], cq[G::R][G::V];
    arrival<T, S, G>(st, smem + (size_t)(k % G::NS) * G::SLOT, c, out, cq);
    if (q - 1 >= zs) store_plane<T, G>(dst, d, q - 1, x0, y0, out, st.cm1);
#pragma unroll
    for (int r = 0; r < G::R; r++)
#pragma unroll
      for (int i = 0; i < G::V; i++) st.cm1[r][i] = cq[r][i];
  }
  cp_async_wait<0>();
}

}  // namespace perks
