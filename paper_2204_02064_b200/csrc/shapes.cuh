// shapes.cuh — compile-time point sets of the hot-path stencils (Table II) in the
// canonical accumulation order (reading R5), and the plane-streaming schedule used by
// the 3D (and row-streaming 2D) kernels.
//
//   SHAPE_2D5  2d5pt  star r=1: W,E,S,C,N          (Eq. iterativeStencil; Fig. 6 order)
//   SHAPE_2D9  2d9pt  box  r=1: (dy,dx) lexicographic ascending
//   SHAPE_3D7  3d7pt  star r=1: W,E,S,C,N,B,F
//   SHAPE_3D27 3d27pt box  r=1: (dz,dy,dx) lexicographic ascending
//   SHAPE_3D19 poisson 19pt r=1 (Table II "poisson(1,38)"): the 3x3x3 cube without its 8 corners,
//              (dz,dy,dx) lexicographic ascending (reading R3b)
//
// The host matches a descriptor's (offset list, order) against these tables exactly; any other
// list is PERKS_ERR_UNSUPPORTED (the kernels follow the list order, so bit-exactness holds).
#pragma once
#include "common.cuh"

namespace perks {

enum ShapeId : int { SHAPE_2D5 = 0, SHAPE_2D9 = 1, SHAPE_3D7 = 2, SHAPE_3D27 = 3, SHAPE_3D19 = 4, SHAPE_COUNT = 5 };

template <int S> struct Shape;

template <> struct Shape<SHAPE_2D5> {
  static constexpr int N = 5, NDIM = 2;
  static constexpr __host__ __device__ int dx(int p) { return p == 0 ? -1 : p == 1 ? 1 : 0; }
  static constexpr __host__ __device__ int dy(int p) { return p == 2 ? -1 : p == 4 ? 1 : 0; }
  static constexpr __host__ __device__ int dz(int) { return 0; }
};
template <> struct Shape<SHAPE_2D9> {
  static constexpr int N = 9, NDIM = 2;
  static constexpr __host__ __device__ int dx(int p) { return p % 3 - 1; }
  static constexpr __host__ __device__ int dy(int p) { return p / 3 - 1; }
  static constexpr __host__ __device__ int dz(int) { return 0; }
};
template <> struct Shape<SHAPE_3D7> {
  static constexpr int N = 7, NDIM = 3;
  static constexpr __host__ __device__ int dx(int p) { return p == 0 ? -1 : p == 1 ? 1 : 0; }
  static constexpr __host__ __device__ int dy(int p) { return p == 2 ? -1 : p == 4 ? 1 : 0; }
  static constexpr __host__ __device__ int dz(int p) { return p == 5 ? -1 : p == 6 ? 1 : 0; }
};
template <> struct Shape<SHAPE_3D27> {
  static constexpr int N = 27, NDIM = 3;
  static constexpr __host__ __device__ int dx(int p) { return p % 3 - 1; }
  static constexpr __host__ __device__ int dy(int p) { return (p / 3) % 3 - 1; }
  static constexpr __host__ __device__ int dz(int p) { return p / 9 - 1; }
};

// 3d19pt: the p-th non-corner point of the 3x3x3 cube in (dz,dy,dx) lexicographic order, as cube
// index c = (dz+1)*9 + (dy+1)*3 + (dx+1) (a literal table: folds at every unrolled use).
template <> struct Shape<SHAPE_3D19> {
  static constexpr int N = 19, NDIM = 3;
  static constexpr __host__ __device__ int cube(int p) {
    constexpr int c[19] = {1, 3, 4, 5, 7, 9, 10, 11, 12, 13, 14, 15, 16, 17, 19, 21, 22, 23, 25};
    return c[p];
  }
  static constexpr __host__ __device__ int dx(int p) { return cube(p) % 3 - 1; }
  static constexpr __host__ __device__ int dy(int p) { return (cube(p) / 3) % 3 - 1; }
  static constexpr __host__ __device__ int dz(int p) { return cube(p) / 9 - 1; }
};

// Does the in-plane part of the shape touch corners (|dx| and |dy| both nonzero)?
template <int S> constexpr bool has_corners() {
  for (int p = 0; p < Shape<S>::N; p++)
    if (Shape<S>::dx(p) != 0 && Shape<S>::dy(p) != 0) return true;
  return false;
}

// Coefficients, passed by value as a kernel parameter (constant bank operands of FFMA/DFMA).
template <typename T, int N> struct Coef {
  T w[N];
};

// ------------------------------------------------------------------ plane-streaming stages
// Planes arrive in increasing z.  When plane q is resident, output o in {q+1, q, q-1} consumes
// its next chain terms in list order:
//   stage A (o = q+1): the maximal prefix of terms with dz = -1                  (start chain)
//   stage B (o = q)  : then terms with dz == 0, or dz == -1 at the centre (retained register)
//   stage C (o = q-1): then terms with dz == +1, or dz == 0 at the centre (retained register)
// so the accumulation order is exactly the list order.  stage_end<S>(k) gives the first term
// index after stage k (0:A 1:B 2:C).
template <int S> constexpr int stage_end(int k) {
  constexpr int N = Shape<S>::N;
  int p = 0;
  while (p < N && Shape<S>::dz(p) == -1) p++;
  if (k == 0) return p;
  while (p < N && (Shape<S>::dz(p) == 0 ||
                   (Shape<S>::dz(p) == -1 && Shape<S>::dx(p) == 0 && Shape<S>::dy(p) == 0)))
    p++;
  if (k == 1) return p;
  while (p < N && (Shape<S>::dz(p) == 1 ||
                   (Shape<S>::dz(p) == 0 && Shape<S>::dx(p) == 0 && Shape<S>::dy(p) == 0)))
    p++;
  return p;
}
template <int S> constexpr bool streamable() { return stage_end<S>(2) == Shape<S>::N; }
// Which retained planes a stage needs (dz = -1 centre in stage B; dz = 0 centre in stage C).
template <int S> constexpr bool needs_prev_center() {
  for (int p = stage_end<S>(0); p < stage_end<S>(1); p++)
    if (Shape<S>::dz(p) == -1) return true;
  return false;
}
template <int S> constexpr bool needs_cur_center_late() {
  for (int p = stage_end<S>(1); p < stage_end<S>(2); p++)
    if (Shape<S>::dz(p) == 0) return true;
  return false;
}

static_assert(streamable<SHAPE_2D5>(), "2d5pt order not streamable");
static_assert(streamable<SHAPE_2D9>(), "2d9pt order not streamable");
static_assert(streamable<SHAPE_3D7>(), "3d7pt order not streamable");
static_assert(streamable<SHAPE_3D27>(), "3d27pt order not streamable");
static_assert(streamable<SHAPE_3D19>(), "3d19pt order not streamable");

}  // namespace perks
