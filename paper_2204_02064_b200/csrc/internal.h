// internal.h — host-side structures shared by the C-ABI layer (api.cu) and the kernel
// launchers (k2d_stream.cu, k3d_stream.cu, k2d_perks.cu, k3d_perks.cu).  Not installed.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/perks/perks_stencil.h"

namespace perks {

// General point sets run on the k2d_wide.cu (2D: radius <= 6) and k3d_wide.cu (3D: radius <= 3)
// kernels (any order, <= 64 points).
constexpr int SHAPE_G2D = 100;
constexpr int SHAPE_G3D = 101;
constexpr int kMaxPoints2D = 64;

struct Problem {
  int ndim;
  int64_t nx, ny, nz;
  int shape;          // ShapeId
  perks_dtype dtype;
  perks_bc bc;
  int npts;
  double wd[kMaxPoints2D];  // weights rounded to f64 (identity)
  float wf[kMaxPoints2D];   // weights rounded once to f32 (reading R6)
  int16_t off[kMaxPoints2D][2];  // (dx, dy) of each point (SHAPE_G2D / G3D)
  int16_t off3z[kMaxPoints2D];   // dz of each point (SHAPE_G3D)
  int device;
  int rank = 0, nranks = 1;  // multi-GPU slab decomposition along z
  int num_sms;
  int max_smem_optin;
  int smem_per_sm;
  int64_t l2_bytes = 0;
  size_t elem() const { return dtype == PERKS_F64 ? 8 : 4; }
  int64_t cells() const { return nx * ny * nz; }
};

// One launchable plan for a variant.
struct Plan {
  perks_variant variant = PERKS_AUTO;
  bool ok = false;
  const char *why = "";       // reason when !ok
  int grid = 0, block = 0, ctas_per_sm = 0;
  int tile[3] = {0, 0, 0};
  int regs = 0, smem = 0;
  int64_t units = 0;          // work units per step
  int zchunk = 0;             // planes per unit (3D)
  int cfg = 0;                // index of the kernel configuration
  int family = 0;             // kernel family within a variant (2D PERKS: 0 tiles, 1 cluster, 3 strips; 3D PERKS: 2)
  bool cache_kernel = false;  // 3D PERKS: the kernel with the on-chip plane cache tiers
  int nc = 0;                 // 3D PERKS: shared-memory plane slots per CTA
  int ntm = 0, tcols = 0;     // 3D PERKS: TMEM planes per CTA, TMEM columns allocated per CTA
  int wsg = 0;                // 3D persistent: warp-specialised geometry (k3d_stream.cu)
  bool persistent_body = false;  // a PERKS plan that runs the persistent kernel (empty cache split)
  int64_t cached_reg = 0, cached_smem = 0, cached_tmem = 0;
  double dram_bytes_step = 0, halo_bytes_step = 0;
  size_t ws_bytes = 0;
  char name[64] = {0};
};

inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// Host view of one rank's exchange state for one run (multi-GPU slabs; device side: dist.cuh).
struct DistRun {
  void *ghost = nullptr;                      // local ghost planes G[4][ny][nx]
  unsigned long long *ctr = nullptr;          // local arrival counters [2]
  void *lo_ghost = nullptr, *hi_ghost = nullptr;  // neighbours' G (mapped into this process)
  unsigned long long *lo_ctr = nullptr, *hi_ctr = nullptr;  // neighbours' counters [2]
  unsigned long long xbase = 0;               // exchange index of this run's input (plane units)
  unsigned long long tbx = 0;                 // two-steps-per-pass exchanges done so far (k3d_tb.cu)
  int has_lo = 0, has_hi = 0;
  int noncoop = 0;                            // launch persistent kernels non-cooperatively
                                              // (several slabs resident on ONE device)
};

// ---- launchers (return cudaSuccess or the failing CUDA error) ----
// 2D row-strip streaming kernels: host-loop (a) and persistent (b).
Plan plan_stream2d(const Problem &p, perks_variant v);
cudaError_t run_stream2d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws,
                         int64_t steps, cudaStream_t s);
// 3D plane streaming kernels: host-loop (a), persistent (b) and PERKS (c).
Plan plan_stream3d(const Problem &p, perks_variant v);
cudaError_t run_stream3d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws,
                         int64_t steps, cudaStream_t s, const DistRun *dr = nullptr);
// Host loop (a) on a group of same-device slab handles: step kernels interleaved in step order.
cudaError_t run_stream3d_hostloop_group(const Problem *const *ps, const Plan *const *pls,
                                        const void *const *in, void *const *out, void *const *ws,
                                        const DistRun *drs, int n, int64_t steps, cudaStream_t s);
// Multi-GPU: the exchange of the run's input faces (exchange xbase) before the first step.
cudaError_t launch_dist_prologue(const Problem &p, const void *in, const DistRun &dr, cudaStream_t s);
// PERKS (c), 2D, domain resident on chip.
Plan plan_perks2d(const Problem &p);
cudaError_t run_perks2d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws,
                        int64_t steps, cudaStream_t s);
// PERKS (c), 2D small domains: the whole domain in one thread-block cluster's registers.
Plan plan_perks2d_cluster(const Problem &p);
cudaError_t run_perks2d_cluster(const Problem &p, const Plan &pl, const void *in, void *out,
                                int64_t steps, cudaStream_t s);
// Tiled PERKS, 2D domains beyond the on-chip capacity ([draft] P:416-441): device-sized tiles with a
// redundant halo advanced Tb steps per pass by the resident kernels (k2d_tiled.cu).
Plan plan_tiled2d(const Problem &p, int64_t steps_hint);
cudaError_t run_tiled2d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws, int64_t steps,
                        cudaStream_t s);
// PERKS (c), 2D fp32 domains 1025..3072 wide: full-width strips, edge rows first.
Plan plan_perks2d_strip(const Problem &p);
cudaError_t run_perks2d_strip(const Problem &p, const Plan &pl, const void *in, void *out, void *ws,
                              int64_t steps, cudaStream_t s);
// PERKS (c), 3D: the persistent kernel with a shared-memory plane cache (k3d_stream.cu).
// PERKS (c), 3D domains that fit on chip: resident bricks, tagged surface exchange (k3d_brick.cu).
Plan plan_brick3d(const Problem &p);
cudaError_t run_brick3d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws, int64_t steps,
                        cudaStream_t s);

// PERKS (c), 3D domains beyond the on-chip capacity: two time steps per pass, level t+1 of the planes
// in flight kept in shared memory (k3d_tb.cu).
Plan plan_tb3d(const Problem &p);
cudaError_t run_tb3d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws, int64_t steps,
                     cudaStream_t s, const DistRun *dr = nullptr);

// Any variant for general 2D point sets of radius <= 6 (k2d_wide.cu).
Plan plan_wide2d(const Problem &p, perks_variant v);
cudaError_t run_wide2d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws, int64_t steps,
                       cudaStream_t s);

// Any variant for general 3D point sets of radius <= 3 (k3d_wide.cu; PERKS = the persistent body).
Plan plan_wide3d(const Problem &p, perks_variant v);
cudaError_t run_wide3d(const Problem &p, const Plan &pl, const void *in, void *out, void *ws, int64_t steps,
                       cudaStream_t s);

// Reset a grid-barrier block (common.cuh grid_barrier): ctr[0] = ctr[1] = base, base = 0 unless
// PERKS_TEST_BAR_BASE sets it (tests start the counter just below 2^32 to exercise the wrap).
cudaError_t reset_grid_barrier(unsigned *bar, cudaStream_t s);

// Map a failing CUDA call to a perks_status, recording it for perks_last_cuda_error (api.cu).
perks_status cuda_status(cudaError_t e);

// Environment override helper (sweeps only): returns def if unset.
int env_int(const char *name, int def);

}  // namespace perks
