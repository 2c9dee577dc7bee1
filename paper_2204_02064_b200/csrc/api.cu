// api.cu — the C-ABI boundary (include/perks/perks_stencil.h): descriptor validation, shape
// matching, planning, workspace sizing, dispatch to the kernel families and error mapping.
// No C++ exception crosses the ABI; every CUDA failure maps to PERKS_ERR_CUDA with the CUDA
// error kept in a thread-local (perks_last_cuda_error).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>

#include "internal.h"
#include "shapes.cuh"

namespace perks {
int env_int(const char *name, int def) {
  const char *v = std::getenv(name);
  if (!v || !*v) return def;
  return std::atoi(v);
}
}  // namespace perks

using namespace perks;

static thread_local int g_last_cuda = 0;

struct perks_stencil_s {
  Problem p;
  std::mutex mu;
  Plan plans[4];
  bool planned[4] = {false, false, false, false};
  // run_host scratch (device), grown on demand
  void *h_in = nullptr, *h_out = nullptr, *h_ws = nullptr;
  size_t h_ws_bytes = 0;
  cudaStream_t h_stream = nullptr;
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
  }
  return -1;
}

const Plan &get_plan(perks_stencil_s *h, perks_variant v) {
  std::lock_guard<std::mutex> lk(h->mu);
  const int i = (int)v;
  if (!h->planned[i]) {
    const Problem &p = h->p;
    Plan pl;
    if (v == PERKS_HOSTLOOP || v == PERKS_PERSISTENT)
      pl = p.ndim == 2 ? plan_stream2d(p, v) : plan_stream3d(p, v);
    else if (v == PERKS_PERKS && p.ndim == 2) {
      pl = plan_perks2d_cluster(p);  // small domains: one cluster, registers only
      if (pl.ok) pl.family = 1;
      else pl = plan_perks2d(p);
    } else if (v == PERKS_PERKS)
      pl = plan_perks3d(p);
    h->plans[i] = pl;
    h->planned[i] = true;
  }
  return h->plans[i];
}

perks_variant resolve(perks_stencil_s *h, perks_variant v) {
  if (v != PERKS_AUTO) return v;
  if (get_plan(h, PERKS_PERKS).ok) return PERKS_PERKS;
  return PERKS_PERSISTENT;
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

perks_status perks_stencil_create(const perks_stencil_desc *d, int device, perks_stencil_t *out) {
  if (!d || !out) return PERKS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (d->ndim != 2 && d->ndim != 3) return PERKS_ERR_INVALID_ARGUMENT;
  if (d->npoints < 1 || d->npoints > 27 || !d->offsets || !d->weights)
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
  if (d->bc != PERKS_BC_FRAME) return PERKS_ERR_UNSUPPORTED;  // GPU kernels: FRAME only
  const int shape = find_shape(d->ndim, d->offsets, d->npoints);
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
  }
  p.device = device;
  {
    DeviceGuard g(device);
    if (!g.ok) { delete h; return cuda_fail(cudaGetLastError()); }
    e = cudaDeviceGetAttribute(&p.num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess)
      e = cudaDeviceGetAttribute(&p.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e == cudaSuccess)
      e = cudaDeviceGetAttribute(&p.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    if (e != cudaSuccess) { delete h; return cuda_fail(e); }
    const int force_sms = env_int("PERKS_NUM_SMS", 0);  // sweeps only
    if (force_sms > 0 && force_sms < p.num_sms) p.num_sms = force_sms;
  }
  *out = h;
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
  switch (v) {
    case PERKS_HOSTLOOP:
    case PERKS_PERSISTENT:
      e = p.ndim == 2 ? run_stream2d(p, pl, d_in, d_out, d_ws, steps, s)
                      : run_stream3d(p, pl, d_in, d_out, d_ws, steps, s);
      break;
    case PERKS_PERKS:
      if (p.ndim == 2)
        e = pl.family == 1 ? run_perks2d_cluster(p, pl, d_in, d_out, steps, s)
                           : run_perks2d(p, pl, d_in, d_out, d_ws, steps, s);
      else
        e = run_perks3d(p, pl, d_in, d_out, d_ws, steps, s);
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

perks_status perks_stencil_destroy(perks_stencil_t h) {
  if (!h) return PERKS_ERR_INVALID_ARGUMENT;
  {
    DeviceGuard g(h->p.device);
    if (h->h_stream) cudaStreamSynchronize(h->h_stream);
    if (h->h_in) cudaFree(h->h_in);
    if (h->h_out) cudaFree(h->h_out);
    if (h->h_ws) cudaFree(h->h_ws);
    if (h->h_stream) cudaStreamDestroy(h->h_stream);
  }
  delete h;
  return PERKS_OK;
}

}  // extern "C"
