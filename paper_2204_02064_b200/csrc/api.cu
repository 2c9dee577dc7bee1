// api.cu — the C-ABI boundary (include/perks/perks_stencil.h): descriptor validation, shape
// matching, planning, workspace sizing, dispatch to the kernel families and error mapping.
// No C++ exception crosses the ABI; every CUDA failure maps to PERKS_ERR_CUDA with the CUDA
// error kept in a thread-local (perks_last_cuda_error).
#include <cuda_runtime.h>

#include <unistd.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "internal.h"
#include "shapes.cuh"

namespace perks {
int env_int(const char *name, int def) {
  const char *v = std::getenv(name);
  if (!v || !*v) return def;
  return std::atoi(v);
}

namespace {
__global__ void reset_bar_kernel(unsigned *bar, unsigned base) {
  if (threadIdx.x < 64) bar[threadIdx.x] = threadIdx.x < 2 ? base : 0u;
}
}  // namespace
cudaError_t reset_grid_barrier(unsigned *bar, cudaStream_t s) {
  const char *v = std::getenv("PERKS_TEST_BAR_BASE");
  const unsigned base = (v && *v) ? (unsigned)std::strtoul(v, nullptr, 0) : 0u;
  if (base == 0) return cudaMemsetAsync(bar, 0, 256, s);  // (no kernel launch in the normal case)
  reset_bar_kernel<<<1, 64, 0, s>>>(bar, base);
  return cudaGetLastError();
}
}  // namespace perks

using namespace perks;

static thread_local int g_last_cuda = 0;

// Multi-GPU slab state of a handle (device side in dist.cuh).
struct DistState {
  bool on = false, connected = false;
  void *alloc = nullptr;          // ghost planes G[4][ny][nx] + counters [2] (one cudaMalloc)
  size_t ghost_bytes = 0, alloc_bytes = 0;
  void *lo_base = nullptr, *hi_base = nullptr;  // neighbours' allocations mapped here
  bool lo_ipc = false, hi_ipc = false;          // opened with cudaIpcOpenMemHandle
  unsigned long long xbase = 0;   // exchanges done so far, in plane units (a one-step-per-pass run
                                  // of T steps does T + 1; a two-steps-per-pass run 2 + 2 * passes)
  unsigned long long tbx = 0;     // two-steps-per-pass exchanges so far (their ghost parity)
};

// Connection blob (PERKS_DIST_BLOB_BYTES): what a neighbour needs to map our ghost planes.
struct DistBlob {
  uint32_t magic, version;
  int32_t pid, device, rank, nranks;
  int64_t nx, ny;
  int32_t dtype, pad;
  uint64_t dev_ptr, ghost_bytes;
  cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(DistBlob) <= PERKS_DIST_BLOB_BYTES, "blob size");
constexpr uint32_t kBlobMagic = 0x504b5344u;  // "PKSD"

struct perks_stencil_s {
  Problem p;
  DistState dist;
  std::mutex mu;
  Plan plans[4];
  bool planned[4] = {false, false, false, false};
  // run_host scratch (device), grown on demand
  void *h_in = nullptr, *h_out = nullptr, *h_ws = nullptr;
  size_t h_ws_bytes = 0;
  cudaStream_t h_stream = nullptr;
  std::vector<cudaStream_t> g_streams;  // run_group: this handle's private launch stream
};

namespace {

struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

perks_status cuda_fail(cudaError_t e) {
  g_last_cuda = (int)e;
  if (e == cudaErrorCooperativeLaunchTooLarge) return PERKS_ERR_NOT_CORESIDENT;
  if (e == cudaErrorMemoryAllocation) return PERKS_ERR_OOM;
  return PERKS_ERR_CUDA;
}

}  // namespace
perks_status perks::cuda_status(cudaError_t e) { return cuda_fail(e); }
namespace {

template <int S> bool match_shape(const int32_t *off, int n) {
  if (n != Shape<S>::N) return false;
  for (int p = 0; p < n; p++)
    if (off[3 * p] != Shape<S>::dx(p) || off[3 * p + 1] != Shape<S>::dy(p) ||
        off[3 * p + 2] != Shape<S>::dz(p))
      return false;
  return true;
}

int find_shape(int ndim, const int32_t *off, int n) {
  if (ndim == 2) {
    if (match_shape<SHAPE_2D5>(off, n)) return SHAPE_2D5;
    if (match_shape<SHAPE_2D9>(off, n)) return SHAPE_2D9;
  } else {
    if (match_shape<SHAPE_3D7>(off, n)) return SHAPE_3D7;
    if (match_shape<SHAPE_3D27>(off, n)) return SHAPE_3D27;
    if (match_shape<SHAPE_3D19>(off, n)) return SHAPE_3D19;
  }
  return -1;
}

bool dist_perks_ok(perks_stencil_s *h);

const Plan &get_plan(perks_stencil_s *h, perks_variant v) {
  std::lock_guard<std::mutex> lk(h->mu);
  const int i = (int)v;
  if (!h->planned[i]) {
    const Problem &p = h->p;
    Plan pl;
    if (p.shape == SHAPE_G2D) {
      pl = plan_wide2d(p, v);
      // beyond the on-chip capacity: Tiled PERKS over the wide2d resident kernel (k2d_tiled.cu)
      if (!pl.ok && v == PERKS_PERKS && env_int("PERKS_TILED", 1)) pl = plan_tiled2d(p, 1000);
    }
    else if (p.shape == SHAPE_G3D)
      pl = plan_wide3d(p, v);
    else if (v == PERKS_HOSTLOOP || v == PERKS_PERSISTENT)
      pl = p.ndim == 2 ? plan_stream2d(p, v) : plan_stream3d(p, v);
    else if (v == PERKS_PERKS && p.ndim == 2) {
      pl = plan_perks2d_cluster(p);  // small domains: one cluster, registers only
      if (pl.ok) {
        pl.family = 1;
      } else {
        // full-width strips (fp32, 1025..3072 wide) are opt-in: measured slower than square tiles
        // on C2 (profiles/r01_c2_strip_first.txt), kept as a tested alternative
        if (env_int("PERKS_STRIP", 0)) pl = plan_perks2d_strip(p);
        if (pl.ok && env_int("PERKS_STRIP", 0)) pl.family = 3;
        else pl = plan_perks2d(p);   // square tiles
        // beyond the on-chip capacity: Tiled PERKS (device-sized tiles with a redundant halo,
        // Tb steps per pass, k2d_tiled.cu); PERKS_TILED=0 disables it
        if (!pl.ok && env_int("PERKS_TILED", 1)) pl = plan_tiled2d(p, 1000);
      }
    } else if (v == PERKS_PERKS) {
      // resident bricks (k3d_brick.cu) are opt-in (PERKS_P3D_BRICK=1): measured slower than the
      // plane-streaming persistent kernel on every 3D domain that fits them, because such domains
      // also fit B200's L2 (profiles/r02_brick3d.txt); default: the streaming kernel (k3d_stream.cu)
      if (env_int("PERKS_P3D_BRICK", 0) && p.nranks == 1) pl = plan_brick3d(p);
      // two time steps per pass (k3d_tb.cu): the default for the 7-point star (PERKS_P3D_TB=-1;
      // not when the opt-in plane-cache tiers are requested), PERKS_P3D_TB=1 for every r = 1
      // shape, 0 off
      const int tb = env_int("PERKS_P3D_TB", -1);
      const bool tb_auto = tb < 0 && p.shape == SHAPE_3D7 && env_int("PERKS_P3D_CACHE", 0) == 0;
      // multi-GPU slabs: the two-deep ghost exchange per pass (k3d_tb.cu), PERKS_TB_DIST=0 keeps the
      // one-step slab kernel
      const bool tb_slabs = p.nranks == 1 || env_int("PERKS_TB_DIST", 1) != 0;
      if (!pl.ok && tb_slabs && (tb == 1 || tb_auto)) pl = plan_tb3d(p);
      if (!pl.ok) pl = plan_stream3d(p, PERKS_PERKS);
    }
    h->plans[i] = pl;
    h->planned[i] = true;
  }
  return h->plans[i];
}

perks_variant resolve(perks_stencil_s *h, perks_variant v) {
  if (v != PERKS_AUTO) return v;
  if (h->dist.on && !dist_perks_ok(h)) return PERKS_PERSISTENT;
  const Plan &pp = get_plan(h, PERKS_PERKS);
  // Tiled PERKS over the general (radius >= 2) kernels: its r*Tb halo makes it slower than the
  // host loop (profiles/r02_tiled2d.txt); AUTO takes the host loop there (explicit PERKS still tiles)
  if (pp.ok && pp.family == 5 && h->p.shape == SHAPE_G2D) return PERKS_HOSTLOOP;
  if (pp.ok) return PERKS_PERKS;
  return PERKS_PERSISTENT;
}

bool dist_perks_ok(perks_stencil_s *h) {
  const Plan &pl = get_plan(h, PERKS_PERKS);
  return pl.ok && (pl.family == 2 || pl.family == 7);
}
// Exchange bookkeeping after a slab run of `steps` with plan `pl` (plane units, see DistState).
void dist_advance(DistState &ds, const Plan &pl, int64_t steps) {
  if (pl.family == 7) {
    const unsigned long long passes = (unsigned long long)((steps + 1) / 2);
    ds.xbase += 2ull + 2ull * passes;
    ds.tbx += 1ull + passes;
  } else {
    ds.xbase += (unsigned long long)steps + 1;  // prologue exchange + one per step
  }
}

DistRun dist_run(perks_stencil_s *h) {
  DistRun r;
  const DistState &ds = h->dist;
  const Problem &p = h->p;
  r.ghost = ds.alloc;
  r.ctr = (unsigned long long *)((char *)ds.alloc + ds.ghost_bytes);
  r.lo_ghost = ds.lo_base;
  r.hi_ghost = ds.hi_base;
  r.lo_ctr = ds.lo_base ? (unsigned long long *)((char *)ds.lo_base + ds.ghost_bytes) : nullptr;
  r.hi_ctr = ds.hi_base ? (unsigned long long *)((char *)ds.hi_base + ds.ghost_bytes) : nullptr;
  r.has_lo = p.rank > 0;
  r.has_hi = p.rank < p.nranks - 1;
  r.xbase = ds.xbase;
  r.tbx = ds.tbx;
  return r;
}

bool valid_variant(perks_variant v) {
  return v == PERKS_AUTO || v == PERKS_HOSTLOOP || v == PERKS_PERSISTENT || v == PERKS_PERKS;
}

}  // namespace

extern "C" {

const char *perks_version(void) { return "perks-b200 0.1 (sm_100a)"; }

int perks_last_cuda_error(void) { return g_last_cuda; }

const char *perks_status_string(perks_status s) {
  switch (s) {
    case PERKS_OK: return "PERKS_OK";
    case PERKS_ERR_INVALID_ARGUMENT: return "PERKS_ERR_INVALID_ARGUMENT";
    case PERKS_ERR_INVALID_DOMAIN: return "PERKS_ERR_INVALID_DOMAIN";
    case PERKS_ERR_UNSUPPORTED: return "PERKS_ERR_UNSUPPORTED";
    case PERKS_ERR_ALIAS: return "PERKS_ERR_ALIAS";
    case PERKS_ERR_WORKSPACE: return "PERKS_ERR_WORKSPACE";
    case PERKS_ERR_NOT_CORESIDENT: return "PERKS_ERR_NOT_CORESIDENT";
    case PERKS_ERR_CUDA: return "PERKS_ERR_CUDA";
    case PERKS_ERR_COMM: return "PERKS_ERR_COMM";
    case PERKS_ERR_OOM: return "PERKS_ERR_OOM";
  }
  return "PERKS_ERR_UNKNOWN";
}

static perks_status create_impl(const perks_stencil_desc *d, int device, int rank, int nranks,
                                perks_stencil_t *out) {
  if (!d || !out) return PERKS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (d->ndim != 2 && d->ndim != 3) return PERKS_ERR_INVALID_ARGUMENT;
  if (d->npoints < 1 || d->npoints > kMaxPoints2D || !d->offsets || !d->weights)
    return PERKS_ERR_INVALID_ARGUMENT;
  if (d->dtype != PERKS_F32 && d->dtype != PERKS_F64) return PERKS_ERR_INVALID_ARGUMENT;
  if (d->bc != PERKS_BC_FRAME && d->bc != PERKS_BC_PERIODIC) return PERKS_ERR_INVALID_ARGUMENT;
  int r = 0;
  for (int p = 0; p < d->npoints; p++)
    for (int a = 0; a < 3; a++) {
      const int o = d->offsets[3 * p + a];
      if (a >= d->ndim && o != 0) return PERKS_ERR_INVALID_ARGUMENT;
      r = std::abs(o) > r ? std::abs(o) : r;
    }
  for (int p = 0; p < d->npoints; p++)
    if (!std::isfinite(d->weights[p])) return PERKS_ERR_INVALID_ARGUMENT;
  if (d->ndim == 2 && d->extent[2] != 1) return PERKS_ERR_INVALID_DOMAIN;
  for (int a = 0; a < 3; a++)
    if (d->extent[a] < 1) return PERKS_ERR_INVALID_DOMAIN;
  for (int a = 0; a < d->ndim; a++)
    if (d->extent[a] < 2 * r + 1) return PERKS_ERR_INVALID_DOMAIN;
  for (int a = 0; a < 3; a++)
    if (d->extent[a] > (int64_t)1 << 30) return PERKS_ERR_UNSUPPORTED;
  // PERIODIC (reading R1's alternative): single GPU, the general kernels of k2d_wide.cu /
  // k3d_wide.cu (wrapped tile and plane loads); slabs keep the FRAME boundary
  const bool periodic = d->bc == PERKS_BC_PERIODIC;
  if (periodic && nranks > 1) return PERKS_ERR_UNSUPPORTED;
  int shape = periodic ? -1 : find_shape(d->ndim, d->offsets, d->npoints);
  // 2D point sets without a specialised kernel (radius > 1, or another order / set): the general
  // kernels of k2d_wide.cu (radius <= 6)
  if (shape < 0 && d->ndim == 2 && r <= 6) shape = SHAPE_G2D;
  if (shape < 0 && d->ndim == 3 && r <= 3) shape = SHAPE_G3D;  // k3d_wide.cu
  if (shape < 0) return PERKS_ERR_UNSUPPORTED;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(e);
  if (device < 0 || device >= ndev) return PERKS_ERR_INVALID_ARGUMENT;
  perks_stencil_s *h = new (std::nothrow) perks_stencil_s();
  if (!h) return PERKS_ERR_OOM;
  Problem &p = h->p;
  p.ndim = d->ndim;
  p.nx = d->extent[0];
  p.ny = d->extent[1];
  p.nz = d->extent[2];
  p.shape = shape;
  p.dtype = d->dtype;
  p.bc = d->bc;
  p.npts = d->npoints;
  for (int i = 0; i < d->npoints; i++) {
    p.wd[i] = d->weights[i];
    p.wf[i] = (float)d->weights[i];  // reading R6: rounded once (RN-even) to the storage dtype
    p.off[i][0] = (int16_t)d->offsets[3 * i];
    p.off[i][1] = (int16_t)d->offsets[3 * i + 1];
    p.off3z[i] = (int16_t)d->offsets[3 * i + 2];
  }
  p.device = device;
  p.rank = rank;
  p.nranks = nranks;
  {
    DeviceGuard g(device);
    if (!g.ok) { delete h; return cuda_fail(cudaGetLastError()); }
    e = cudaDeviceGetAttribute(&p.num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess)
      e = cudaDeviceGetAttribute(&p.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e == cudaSuccess)
      e = cudaDeviceGetAttribute(&p.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    int l2 = 0;
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
    p.l2_bytes = l2;
    if (e != cudaSuccess) { delete h; return cuda_fail(e); }
    const int force_sms = env_int("PERKS_NUM_SMS", 0);  // sweeps only
    if (force_sms > 0 && force_sms < p.num_sms) p.num_sms = force_sms;
  }
  *out = h;
  return PERKS_OK;
}

perks_status perks_stencil_create(const perks_stencil_desc *d, int device, perks_stencil_t *out) {
  return create_impl(d, device, 0, 1, out);
}

perks_status perks_stencil_create_dist(const perks_stencil_desc *d, int device, int rank, int nranks,
                                       perks_stencil_t *out) {
  if (!d || !out || nranks < 1 || rank < 0 || rank >= nranks) return PERKS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (d->ndim != 3) return d->ndim == 2 ? PERKS_ERR_UNSUPPORTED : PERKS_ERR_INVALID_ARGUMENT;
  // a slab face with a neighbour is interior: the local slab needs only 2 planes (R9 applies to
  // the global extent, which is >= 2 * nranks >= 3 for nranks >= 2)
  perks_stencil_desc dd = *d;
  const int64_t nz_local = d->extent[2];
  if (nranks > 1) {
    if (nz_local < 2) return PERKS_ERR_INVALID_DOMAIN;
    if ((d->extent[0] * (d->dtype == PERKS_F64 ? 8 : 4)) % 16 != 0) return PERKS_ERR_UNSUPPORTED;
    dd.extent[2] = nz_local < 3 ? 3 : nz_local;  // validate x/y and the point set as usual
  }
  perks_status st = create_impl(&dd, device, rank, nranks, out);
  if (st != PERKS_OK) return st;
  perks_stencil_s *h = *out;
  h->p.nz = nz_local;
  if (nranks == 1) return PERKS_OK;
  if (h->p.shape == SHAPE_G3D) {  // slabs exchange faces only in the specialised r=1 kernels
    perks_stencil_destroy(h);
    *out = nullptr;
    return PERKS_ERR_UNSUPPORTED;
  }
  DistState &ds = h->dist;
  ds.on = true;
  DeviceGuard g(device);
  // G[12][ny][nx]: planes 0..3 for the one-step slab kernels, 4..11 for the two-steps-per-pass kernel
  ds.ghost_bytes = align256((size_t)12 * h->p.nx * h->p.ny * h->p.elem());
  ds.alloc_bytes = ds.ghost_bytes + 256;
  cudaError_t e = cudaMalloc(&ds.alloc, ds.alloc_bytes);
  if (e == cudaSuccess) e = cudaMemset(ds.alloc, 0, ds.alloc_bytes);
  if (e != cudaSuccess) {
    perks_stencil_destroy(h);
    *out = nullptr;
    return cuda_fail(e);
  }
  return PERKS_OK;
}

perks_status perks_stencil_dist_export(perks_stencil_t h, void *blob) {
  if (!h || !blob || !h->dist.on) return PERKS_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->p.device);
  DistBlob b;
  std::memset(&b, 0, sizeof(b));
  b.magic = kBlobMagic;
  b.version = 1;
  b.pid = (int32_t)getpid();
  b.device = h->p.device;
  b.rank = h->p.rank;
  b.nranks = h->p.nranks;
  b.nx = h->p.nx;
  b.ny = h->p.ny;
  b.dtype = (int32_t)h->p.dtype;
  b.dev_ptr = (uint64_t)(uintptr_t)h->dist.alloc;
  b.ghost_bytes = h->dist.ghost_bytes;
  cudaError_t e = cudaIpcGetMemHandle(&b.ipc, h->dist.alloc);
  if (e != cudaSuccess) return cuda_fail(e);
  std::memset(blob, 0, PERKS_DIST_BLOB_BYTES);
  std::memcpy(blob, &b, sizeof(b));
  return PERKS_OK;
}

static perks_status map_peer(perks_stencil_s *h, const void *blob, int want_rank, void **base, bool *ipc) {
  DistBlob b;
  std::memcpy(&b, blob, sizeof(b));
  const Problem &p = h->p;
  if (b.magic != kBlobMagic || b.version != 1 || b.rank != want_rank || b.nranks != p.nranks ||
      b.nx != p.nx || b.ny != p.ny || b.dtype != (int32_t)p.dtype || b.ghost_bytes != h->dist.ghost_bytes)
    return PERKS_ERR_COMM;
  if (b.pid == (int32_t)getpid()) {
    if (b.device != p.device) {
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, p.device, b.device);
      if (!ok) return PERKS_ERR_COMM;
      cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) return cuda_fail(e);
    }
    *base = (void *)(uintptr_t)b.dev_ptr;
    *ipc = false;
    return PERKS_OK;
  }
  cudaError_t e = cudaIpcOpenMemHandle(base, b.ipc, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e);
  *ipc = true;
  return PERKS_OK;
}

perks_status perks_stencil_dist_connect(perks_stencil_t h, const void *lower, const void *upper) {
  if (!h || !h->dist.on) return PERKS_ERR_INVALID_ARGUMENT;
  const Problem &p = h->p;
  if ((p.rank > 0) != (lower != nullptr) || (p.rank < p.nranks - 1) != (upper != nullptr))
    return PERKS_ERR_INVALID_ARGUMENT;
  if (h->dist.connected) return PERKS_ERR_INVALID_ARGUMENT;
  DeviceGuard g(p.device);
  perks_status st = PERKS_OK;
  if (lower && (st = map_peer(h, lower, p.rank - 1, &h->dist.lo_base, &h->dist.lo_ipc)) != PERKS_OK) return st;
  if (upper && (st = map_peer(h, upper, p.rank + 1, &h->dist.hi_base, &h->dist.hi_ipc)) != PERKS_OK) return st;
  h->dist.connected = true;
  return PERKS_OK;
}

perks_status perks_stencil_workspace_bytes(perks_stencil_t h, perks_variant v, size_t *bytes) {
  if (!h || !bytes || !valid_variant(v)) return PERKS_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->p.device);
  v = resolve(h, v);
  const Plan &pl = get_plan(h, v);
  if (!pl.ok) return PERKS_ERR_UNSUPPORTED;
  *bytes = pl.ws_bytes;
  return PERKS_OK;
}

perks_status perks_stencil_query(perks_stencil_t h, perks_variant v, perks_plan_info *info) {
  if (!h || !info || !valid_variant(v)) return PERKS_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->p.device);
  v = resolve(h, v);
  const Plan &pl = get_plan(h, v);
  if (!pl.ok) return PERKS_ERR_UNSUPPORTED;
  std::memset(info, 0, sizeof(*info));
  info->variant = (int32_t)v;
  info->grid = pl.grid;
  info->block = pl.block;
  info->ctas_per_sm = pl.ctas_per_sm;
  for (int a = 0; a < 3; a++) info->tile[a] = pl.tile[a];
  info->regs_per_thread = pl.regs;
  info->smem_per_cta = pl.smem;
  info->cached_cells_reg = pl.cached_reg;
  info->cached_cells_smem = pl.cached_smem;
  info->cached_cells_tmem = pl.cached_tmem;
  info->tmem_cols_per_cta = pl.tcols;
  info->total_cells = h->p.cells();
  info->dram_bytes_per_step = pl.dram_bytes_step;
  info->halo_bytes_per_step = pl.halo_bytes_step;
  info->workspace_bytes = pl.ws_bytes;
  std::strncpy(info->kernel_name, pl.name, sizeof(info->kernel_name) - 1);
  return PERKS_OK;
}

perks_status perks_stencil_launch_count(perks_stencil_t h, perks_variant v, int64_t steps,
                                        int64_t *launches) {
  if (!h || !launches || !valid_variant(v) || steps < 0) return PERKS_ERR_INVALID_ARGUMENT;
  DeviceGuard g(h->p.device);
  v = resolve(h, v);
  if (steps == 0) { *launches = 0; return PERKS_OK; }
  const Plan &pl = get_plan(h, v);
  if (pl.ok && pl.family == 5 && h->p.ndim == 2) {  // Tiled PERKS: one resident launch per tile and pass
    *launches = ((steps + pl.zchunk - 1) / pl.zchunk) * pl.units;
    return PERKS_OK;
  }
  *launches = v == PERKS_HOSTLOOP ? steps : 1;
  return PERKS_OK;
}

perks_status perks_stencil_run(perks_stencil_t h, perks_variant v, const void *d_in, void *d_out,
                               void *d_ws, size_t ws_bytes, int64_t steps, void *stream) {
  if (!h || !d_in || !d_out || !valid_variant(v) || steps < 0) return PERKS_ERR_INVALID_ARGUMENT;
  const Problem &p = h->p;
  const size_t bytes = (size_t)p.cells() * p.elem();
  const char *a = (const char *)d_in, *b = (const char *)d_out;
  if (a < b + bytes && b < a + bytes) return PERKS_ERR_ALIAS;
  DeviceGuard g(p.device);
  if (!g.ok) return cuda_fail(cudaGetLastError());
  cudaStream_t s = (cudaStream_t)stream;
  if (steps == 0) {  // N = 0 returns the input
    cudaError_t e = cudaMemcpyAsync(d_out, d_in, bytes, cudaMemcpyDeviceToDevice, s);
    return e == cudaSuccess ? PERKS_OK : cuda_fail(e);
  }
  v = resolve(h, v);
  const Plan &pl = get_plan(h, v);
  if (!pl.ok) return PERKS_ERR_UNSUPPORTED;
  if (pl.ws_bytes > 0) {
    if (!d_ws || ws_bytes < pl.ws_bytes || ((uintptr_t)d_ws & 255) != 0) return PERKS_ERR_WORKSPACE;
    const char *w = (const char *)d_ws;
    if ((w < a + bytes && a < w + pl.ws_bytes) || (w < b + bytes && b < w + pl.ws_bytes))
      return PERKS_ERR_ALIAS;
  }
  if ((((uintptr_t)d_in) & 15) != 0 || (((uintptr_t)d_out) & 15) != 0) return PERKS_ERR_INVALID_ARGUMENT;
  cudaError_t e = cudaSuccess;
  if (h->dist.on) {
    if (!h->dist.connected) return PERKS_ERR_COMM;
    DistRun dr = dist_run(h);
    e = pl.family == 7 ? run_tb3d(p, pl, d_in, d_out, d_ws, steps, s, &dr)
                       : run_stream3d(p, pl, d_in, d_out, d_ws, steps, s, &dr);
    if (e != cudaSuccess) return cuda_fail(e);
    dist_advance(h->dist, pl, steps);
    return PERKS_OK;
  }
  if (pl.family == 5 && p.ndim == 2) {  // Tiled PERKS (2D, beyond the on-chip capacity)
    e = run_tiled2d(p, pl, d_in, d_out, d_ws, steps, s);
    return e == cudaSuccess ? PERKS_OK : cuda_fail(e);
  }
  if (p.shape == SHAPE_G2D || p.shape == SHAPE_G3D) {
    cudaError_t e2 = p.shape == SHAPE_G2D ? run_wide2d(p, pl, d_in, d_out, d_ws, steps, s)
                                          : run_wide3d(p, pl, d_in, d_out, d_ws, steps, s);
    return e2 == cudaSuccess ? PERKS_OK : cuda_fail(e2);
  }
  switch (v) {
    case PERKS_HOSTLOOP:
    case PERKS_PERSISTENT:
      e = p.ndim == 2 ? run_stream2d(p, pl, d_in, d_out, d_ws, steps, s)
                      : run_stream3d(p, pl, d_in, d_out, d_ws, steps, s);
      break;
    case PERKS_PERKS:
      if (p.ndim == 2)
        e = pl.family == 1 ? run_perks2d_cluster(p, pl, d_in, d_out, steps, s)
            : pl.family == 3 ? run_perks2d_strip(p, pl, d_in, d_out, d_ws, steps, s)
                             : run_perks2d(p, pl, d_in, d_out, d_ws, steps, s);
      else if (pl.family == 6)
        e = run_brick3d(p, pl, d_in, d_out, d_ws, steps, s);
      else if (pl.family == 7)
        e = run_tb3d(p, pl, d_in, d_out, d_ws, steps, s);
      else
        e = run_stream3d(p, pl, d_in, d_out, d_ws, steps, s);
      break;
    default:
      return PERKS_ERR_INVALID_ARGUMENT;
  }
  return e == cudaSuccess ? PERKS_OK : cuda_fail(e);
}

perks_status perks_stencil_run_host(perks_stencil_t h, perks_variant v, const void *h_in,
                                    void *h_out, int64_t steps) {
  if (!h || !h_in || !h_out || !valid_variant(v) || steps < 0) return PERKS_ERR_INVALID_ARGUMENT;
  const Problem &p = h->p;
  DeviceGuard g(p.device);
  if (!g.ok) return cuda_fail(cudaGetLastError());
  const size_t bytes = (size_t)p.cells() * p.elem();
  size_t ws = 0;
  if (steps > 0) {
    perks_status st = perks_stencil_workspace_bytes(h, v, &ws);
    if (st != PERKS_OK) return st;
  }
  cudaError_t e = cudaSuccess;
  if (!h->h_stream) {
    e = cudaStreamCreateWithFlags(&h->h_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  if (!h->h_in) {
    if ((e = cudaMalloc(&h->h_in, bytes)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMalloc(&h->h_out, bytes)) != cudaSuccess) return cuda_fail(e);
  }
  if (ws > h->h_ws_bytes) {
    if (h->h_ws) cudaFree(h->h_ws);
    h->h_ws = nullptr;
    h->h_ws_bytes = 0;
    if ((e = cudaMalloc(&h->h_ws, ws)) != cudaSuccess) return cuda_fail(e);
    h->h_ws_bytes = ws;
  }
  if ((e = cudaMemcpyAsync(h->h_in, h_in, bytes, cudaMemcpyHostToDevice, h->h_stream)) != cudaSuccess)
    return cuda_fail(e);
  perks_status st = perks_stencil_run(h, v, h->h_in, h->h_out, h->h_ws, h->h_ws_bytes, steps, h->h_stream);
  if (st != PERKS_OK) return st;
  if ((e = cudaMemcpyAsync(h_out, h->h_out, bytes, cudaMemcpyDeviceToHost, h->h_stream)) != cudaSuccess)
    return cuda_fail(e);
  if ((e = cudaStreamSynchronize(h->h_stream)) != cudaSuccess) return cuda_fail(e);
  return PERKS_OK;
}

perks_status perks_stencil_run_group(const perks_stencil_t *hs, int n, perks_variant v,
                                     const void *const *d_in, void *const *d_out,
                                     void *const *d_ws, const size_t *ws_bytes, int64_t steps,
                                     void *stream) {
  if (!hs || n < 1 || !d_in || !d_out || !d_ws || !ws_bytes || !valid_variant(v) || steps < 0)
    return PERKS_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < n; i++) {
    if (!hs[i] || !d_in[i] || !d_out[i]) return PERKS_ERR_INVALID_ARGUMENT;
    if (!hs[i]->dist.on || hs[i]->p.device != hs[0]->p.device || hs[i]->p.dtype != hs[0]->p.dtype ||
        hs[i]->p.shape != hs[0]->p.shape)
      return PERKS_ERR_INVALID_ARGUMENT;
    if (!hs[i]->dist.connected) return PERKS_ERR_COMM;
  }
  cudaStream_t s = (cudaStream_t)stream;
  DeviceGuard g(hs[0]->p.device);
  if (steps == 0) {
    for (int i = 0; i < n; i++) {
      perks_status st = perks_stencil_run(hs[i], v, d_in[i], d_out[i], d_ws[i], ws_bytes[i], 0, stream);
      if (st != PERKS_OK) return st;
    }
    return PERKS_OK;
  }
  std::vector<const Problem *> ps(n);
  std::vector<const Plan *> pls(n);
  std::vector<DistRun> drs(n);
  const perks_variant rv = resolve(hs[0], v);
  for (int i = 0; i < n; i++) {
    const Plan &pl = get_plan(hs[i], rv);
    if (!pl.ok) return PERKS_ERR_UNSUPPORTED;
    if (pl.ws_bytes > 0 && (!d_ws[i] || ws_bytes[i] < pl.ws_bytes || ((uintptr_t)d_ws[i] & 255) != 0))
      return PERKS_ERR_WORKSPACE;
    ps[i] = &hs[i]->p;
    pls[i] = &pl;
    drs[i] = dist_run(hs[i]);
    drs[i].noncoop = 1;
  }
  cudaError_t e = cudaSuccess;
  if (rv != PERKS_HOSTLOOP) {
    // every slab's persistent grid spins on its neighbours: all grids must be resident at once
    // (a grid that cannot start would leave the others waiting until the watchdog trap)
    // (capacity of the whole device: the slabs' plans may each see only PERKS_NUM_SMS of its SMs)
    int dev_sms = 0;
    if (cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, hs[0]->p.device) != cudaSuccess)
      return cuda_fail(cudaGetLastError());
    int64_t sum = 0, cap = INT64_MAX;
    for (int i = 0; i < n; i++) {
      sum += pls[i]->grid;
      cap = std::min<int64_t>(cap, (int64_t)pls[i]->ctas_per_sm * dev_sms);
    }
    if (sum > cap) return PERKS_ERR_NOT_CORESIDENT;
  }
  if (rv == PERKS_HOSTLOOP) {
    e = run_stream3d_hostloop_group(ps.data(), pls.data(), d_in, d_out, d_ws, drs.data(), n, steps, s);
  } else {
    // one persistent kernel per slab, each on its own stream, all resident together
    cudaEvent_t fork;
    if ((e = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e);
    cudaEventRecord(fork, s);
    std::vector<cudaEvent_t> joins(n);
    for (int i = 0; i < n && e == cudaSuccess; i++) {
      perks_stencil_s *h = hs[i];
      if (h->g_streams.empty()) {
        cudaStream_t gs;
        if ((e = cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking)) != cudaSuccess) break;
        h->g_streams.push_back(gs);
      }
      cudaStream_t gs = h->g_streams[0];
      cudaStreamWaitEvent(gs, fork, 0);
      e = pls[i]->family == 7 ? run_tb3d(*ps[i], *pls[i], d_in[i], d_out[i], d_ws[i], steps, gs, &drs[i])
                              : run_stream3d(*ps[i], *pls[i], d_in[i], d_out[i], d_ws[i], steps, gs, &drs[i]);
      if (e != cudaSuccess) break;
      cudaEventCreateWithFlags(&joins[i], cudaEventDisableTiming);
      cudaEventRecord(joins[i], gs);
      cudaStreamWaitEvent(s, joins[i], 0);
      cudaEventDestroy(joins[i]);
    }
    cudaEventDestroy(fork);
  }
  if (e != cudaSuccess) return cuda_fail(e);
  for (int i = 0; i < n; i++) dist_advance(hs[i]->dist, *pls[i], steps);
  return PERKS_OK;
}

perks_status perks_stencil_destroy(perks_stencil_t h) {
  if (!h) return PERKS_ERR_INVALID_ARGUMENT;
  {
    DeviceGuard g(h->p.device);
    if (h->h_stream) cudaStreamSynchronize(h->h_stream);
    if (h->h_in) cudaFree(h->h_in);
    if (h->h_out) cudaFree(h->h_out);
    if (h->h_ws) cudaFree(h->h_ws);
    if (h->h_stream) cudaStreamDestroy(h->h_stream);
    for (cudaStream_t gs : h->g_streams) cudaStreamDestroy(gs);
    if (h->dist.lo_ipc && h->dist.lo_base) cudaIpcCloseMemHandle(h->dist.lo_base);
    if (h->dist.hi_ipc && h->dist.hi_base) cudaIpcCloseMemHandle(h->dist.hi_base);
    if (h->dist.alloc) cudaFree(h->dist.alloc);
  }
  delete h;
  return PERKS_OK;
}

}  // extern "C"
