/*
 * perks_stencil.h — C ABI of the B200-native PERKS stencil library.
 *
 * What the library computes (PAPER.md = /root/reference/PAPER.md, arXiv 2204.02064):
 *   the iterative explicit stencil  x^{k+1} = F(x^k)  (Eq. iterative),
 *   F(x)(c) = sum_p w_p * x(c + d_p)                    (Eq. iterativeStencil),
 *   applied `steps` times out of place (Jacobi; step k+1 sees only step-k values).
 * How (the three execution variants of the north star):
 *   PERKS_HOSTLOOP   (a) one kernel launch per time step, the host time loop of Fig. 3 left;
 *   PERKS_PERSISTENT (b) one cooperative launch, the time loop moved into the kernel with a
 *                        device-wide barrier between steps (Fig. 3 right);
 *   PERKS_PERKS      (c) (b) plus caching of the domain in registers and shared memory across
 *                        steps, halo-only re-reads through L2 (§3.3 P:342-356,
 *                        Fig. 6).  For 3D domains beyond the on-chip capacity the
 *                        7-point star's plan keeps the next time level of the planes in flight on
 *                        chip instead and advances two steps per pass over the domain (Tiled
 *                        PERKS in streaming form, [draft] P:416-441, reading R15;
 *                        kernel names perks3d_tb2_*; dram_bytes_per_step = S·cells).
 * All variants produce bit-identical results (the scheme "does not touch on the compute part",
 * P:285): each cell is  acc = w_0*x(c+d_0) rounded, then acc = fma(w_p, x(c+d_p), acc)
 * in list order (reading R5), in the storage dtype (R6).
 *
 * Conventions for every entry point:
 *   - extern "C", no C++ exceptions cross the ABI, every call returns perks_status.
 *   - Device pointers are CUDA device addresses on the handle's device; host pointers are
 *     ordinary (pageable or pinned) host memory.  The library never frees caller memory.
 *   - Layout: dense C order [z][y][x], x unit stride, no padding.  2D uses nz = 1.
 *   - Boundary: PERKS_BC_FRAME — cells within r of any face are never updated and are copied
 *     to `out` bit-exactly (reading R1; the paper is silent).
 */
#ifndef PERKS_STENCIL_H
#define PERKS_STENCIL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PERKS_OK = 0,
  PERKS_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, bad enum, steps < 0, bad offsets          */
  PERKS_ERR_INVALID_DOMAIN = 2,   /* an active extent < 2r+1, or nz != 1 in 2D   */
  PERKS_ERR_UNSUPPORTED = 3,      /* no kernel instantiated for (dtype, point set, bc, variant) */
  PERKS_ERR_ALIAS = 4,            /* d_in and d_out byte ranges overlap (Jacobi is out of place) */
  PERKS_ERR_WORKSPACE = 5,        /* workspace NULL/too small/not 256-B aligned                */
  PERKS_ERR_NOT_CORESIDENT = 6,   /* persistent grid cannot be co-resident            */
  PERKS_ERR_CUDA = 7,             /* a CUDA runtime call failed; see perks_last_cuda_error()   */
  PERKS_ERR_COMM = 8,             /* multi-GPU peer setup failed                               */
  PERKS_ERR_OOM = 9               /* host or device allocation failed                          */
} perks_status;

typedef enum { PERKS_F32 = 0, PERKS_F64 = 1 } perks_dtype;

typedef enum {
  PERKS_BC_FRAME = 0,    /* Dirichlet frame of width r (hot path)                               */
  PERKS_BC_PERIODIC = 1  /* wrap-around (R1): single GPU, the general kernels (2D radius
                            <= 6, 3D radius <= 3); PERKS runs the persistent body with an empty
                            cache split; UNSUPPORTED for multi-GPU slabs                        */
} perks_bc;

typedef enum {
  PERKS_AUTO = 0,        /* PERKS if a plan exists, else PERSISTENT                              */
  PERKS_HOSTLOOP = 1,
  PERKS_PERSISTENT = 2,
  PERKS_PERKS = 3
} perks_variant;

/* Problem descriptor (copied at create; the caller may free its arrays afterwards). */
typedef struct {
  int32_t ndim;            /* 2 or 3                                                           */
  int64_t extent[3];       /* {nx, ny, nz}; nz = 1 for 2D                                      */
  int32_t npoints;         /* |P|                                                              */
  const int32_t *offsets;  /* host, npoints*3 ints (dx, dy, dz); list order = accumulation order */
  const double *weights;   /* host, npoints; rounded ONCE to dtype at create (reading R6)      */
  perks_dtype dtype;
  perks_bc bc;
} perks_stencil_desc;

typedef struct perks_stencil_s *perks_stencil_t;

/* Plan summary for one variant (what the planner chose; P:342-356 caching policy, D7). */
typedef struct {
  int32_t variant;              /* resolved variant (never PERKS_AUTO)                          */
  int32_t grid;                 /* CTAs per launch                                              */
  int32_t block;                /* threads per CTA                                              */
  int32_t ctas_per_sm;          /* co-resident CTAs per SM used by the plan                     */
  int32_t tile[3];              /* cells per work unit (x, y, z)                                */
  int32_t regs_per_thread;      /* from cudaFuncGetAttributes                                   */
  int32_t smem_per_cta;         /* dynamic + static shared memory bytes                         */
  int64_t cached_cells_reg;     /* cells resident in registers across steps (PERKS)             */
  int64_t cached_cells_smem;    /* cells resident in shared memory across steps (PERKS)         */
  int64_t total_cells;          /* nx*ny*nz                                                     */
  double dram_bytes_per_step;   /* algorithmic DRAM bytes per step (model A_gm/N)        */
  double halo_bytes_per_step;   /* bytes re-read/published for halos per step       */
  size_t workspace_bytes;       /* required workspace                                           */
  char kernel_name[64];         /* short name of the kernel instantiation                       */
  int64_t cached_cells_tmem;    /* cells resident in Tensor Memory across steps (3D PERKS TMEM
                                   tier, sm_100a, [draft] P:395-404)       */
  int32_t tmem_cols_per_cta;    /* TMEM columns each CTA allocates (0 = no TMEM tier)           */
} perks_plan_info;

/* Create a handle for one device.  Validates the descriptor (errors above), matches the point
 * list against the instantiated shapes, copies coefficients.  Does not allocate device memory
 * except small constants.  `device` is a CUDA ordinal. */
perks_status perks_stencil_create(const perks_stencil_desc *desc, int device, perks_stencil_t *out);

/* Bytes of device workspace `run` needs for `variant` (ping-pong buffer + exchange slots +
 * barrier counters).  The caller allocates it (256-B aligned) and passes it to run. */
perks_status perks_stencil_workspace_bytes(perks_stencil_t h, perks_variant variant, size_t *bytes);

/* Enqueue `steps` time steps on `stream` (a cudaStream_t; 0 = legacy default stream).
 *   d_in  : device, read only, never written;   d_out : device, every cell written (frame too).
 *   steps == 0 copies d_in to d_out.  Asynchronous: PERKS_OK means enqueued; device faults
 *   surface at the caller's next synchronisation.  Runs on different streams need distinct
 *   workspaces; persistent variants must not overlap on one device (co-residency). */
perks_status perks_stencil_run(perks_stencil_t h, perks_variant variant, const void *d_in,
                               void *d_out, void *d_workspace, size_t workspace_bytes,
                               int64_t steps, void *stream);

/* End-to-end convenience entry: host buffers in and out.  Allocates device buffers and the
 * workspace, copies h_in to the device, runs, copies the result to h_out and synchronises.
 * Blocking.  The timed e2e leg of bench.py uses this call. */
perks_status perks_stencil_run_host(perks_stencil_t h, perks_variant variant, const void *h_in,
                                    void *h_out, int64_t steps);

/* Plan summary (see perks_plan_info). */
perks_status perks_stencil_query(perks_stencil_t h, perks_variant variant, perks_plan_info *info);

/* Number of kernel launches `run` issues for `steps` (host loop: steps; persistent: 1 + setup). */
perks_status perks_stencil_launch_count(perks_stencil_t h, perks_variant variant, int64_t steps,
                                        int64_t *launches);

/* ---- Multi-GPU slab decomposition (the paper's distributed suggestion) ----
 * The global 3D domain is split along z (the slowest axis) into `nranks` slabs, rank r owning
 * global planes [z_r, z_r + local nz).  `local` describes THIS rank's slab exactly as for
 * perks_stencil_create (extent = {nx, ny, local nz}, local nz >= 2; nx*S a multiple of 16).
 * The FRAME applies only at the global faces (rank 0's first plane, rank nranks-1's last plane);
 * every other slab face is updated with the neighbour's plane as its halo, so the N-slab result
 * equals the single-GPU result on the global domain bit-exactly (reading R12).
 * Exchange: every step, the CTAs that produce a slab's first/last plane store it straight into
 * the neighbour's library-owned ghost plane (P2P over NVLink when the neighbour is another GPU;
 * ghost planes double-buffered by exchange parity) and then bump the neighbour's arrival counter
 * with a system-scope release; only the CTAs that read a ghost plane wait (system-scope acquire),
 * so the exchange overlaps the interior planes.  No NCCL call is on the data path.
 * Ownership: the library allocates the ghost planes + counters (cudaMalloc, exportable by CUDA
 * IPC) at create_dist and frees them at destroy.  Ranks must call perks_stencil_run collectively
 * (same variant, same steps) after connecting; a rank that is not connected returns
 * PERKS_ERR_COMM.  Device-side waits carry a watchdog (~10 s) that traps instead of hanging. */
#define PERKS_DIST_BLOB_BYTES 128

perks_status perks_stencil_create_dist(const perks_stencil_desc *local, int device, int rank,
                                       int nranks, perks_stencil_t *out);
/* Write this rank's connection blob (PERKS_DIST_BLOB_BYTES bytes, host memory): an IPC handle of
 * the ghost/counter allocation plus its geometry.  Exchange blobs with the neighbours by any
 * means (bench.py and the tests use torch.distributed all_gather). */
perks_status perks_stencil_dist_export(perks_stencil_t h, void *blob);
/* Connect to rank-1 (`lower_blob`) and rank+1 (`upper_blob`); pass NULL for a missing neighbour
 * (rank 0's lower, rank nranks-1's upper).  Blobs from the same process are used as plain device
 * pointers (peer access enabled if on another device); others are opened with cudaIpcOpenMemHandle.
 * Geometry/dtype/rank mismatches return PERKS_ERR_COMM. */
perks_status perks_stencil_dist_connect(perks_stencil_t h, const void *lower_blob,
                                        const void *upper_blob);
/* Run `n` handles that all live on ONE device together (single-GPU emulation of n slabs, used by
 * the tests).  Host loop: the step kernels of all handles are interleaved in step order on
 * `stream`.  Persistent/PERKS: one kernel per handle on its own internal stream, all resident
 * together (create the handles with PERKS_NUM_SMS = SMs/n so their grids fit), joined back into
 * `stream`.  Arrays are indexed like `hs`; semantics per handle as perks_stencil_run. */
perks_status perks_stencil_run_group(const perks_stencil_t *hs, int n, perks_variant variant,
                                     const void *const *d_in, void *const *d_out,
                                     void *const *d_workspace, const size_t *workspace_bytes,
                                     int64_t steps, void *stream);

perks_status perks_stencil_destroy(perks_stencil_t h);
const char *perks_status_string(perks_status s);
/* Thread-local last cudaError_t behind PERKS_ERR_CUDA (0 if none). */
int perks_last_cuda_error(void);
/* Library version string. */
const char *perks_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PERKS_STENCIL_H */
