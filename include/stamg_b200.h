/* stamg_b200 — C ABI of the B200-native transport-sweep / angular-multigrid
 * hot path (arXiv 2010.04559). Plain pointers and sizes only; no torch or
 * CUDA types cross this boundary.
 *
 * Each entry point replaces one operator of the reference C++ API
 * (/root/reference/proj/include/stamg/*.hpp); the replaced declaration is
 * cited beside it. Vectors live on the device in the reference Layout
 * (layout.hpp:4-32): index((el,q,d,i)) = ((el*P + q)*D + d)*S + i, here with
 * D = 1 (Const angular basis) and S = 4 (2D bilinear cells).
 *
 * Levels: STAMG_OUTER (-1) is the full-order problem the Krylov solver sees
 * (ProblemOperators, transport.hpp:29-45); 0..n_levels-1 are the angular
 * multigrid levels (MgHierarchy::level, multigrid.hpp:43-47), 0 = coarsest.
 *
 * Errors: every call returns STAMG_OK or a code below; stamg_last_error()
 * returns the message of the last failure on the calling thread. The codes
 * map onto the reference's exceptions:
 *   STAMG_EINVAL  <- std::invalid_argument (layout mismatch, order > N, ...)
 *   STAMG_ELOGIC  <- std::logic_error (non-nested meshes)
 *   STAMG_ENAN    <- std::runtime_error("...: NaN residual")
 *   STAMG_ECUDA / STAMG_ENCCL for device and collective failures.
 * A context is externally synchronised (one host thread at a time); all work
 * is ordered on the context's CUDA stream.
 */
#ifndef STAMG_B200_H
#define STAMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  STAMG_OK = 0,
  STAMG_EINVAL = 1,
  STAMG_ELOGIC = 2,
  STAMG_ENAN = 3,
  STAMG_ECUDA = 4,
  STAMG_ENCCL = 5,
  STAMG_EUNSUPPORTED = 6
};

#define STAMG_OUTER (-1)

/* Problem description: geometry (HexMesh, spatial_disc.hpp:12-25, here 2D),
 * angular mesh recipe (sphere_mesh.hpp:45-53), per-material scatter kernels
 * (ScatterKernel, scatter.hpp:14-20), material map, source (SourceSpec,
 * transport.hpp:21-27) and the cycle (CycleSpec, multigrid.hpp:17-24). Same
 * field order as the oracle's orc_spec so one host description drives both. */
typedef struct {
  int dim, nx, ny, nz;
  double box;
  int basis;              /* 0 = Const (the only basis on the B200 path) */
  int p;                  /* 1 = bilinear (the only order on the B200 path) */
  int angular_kind;       /* 0 uniform, 1 banded (+z), 2 cone around +x */
  int angular_level, cone_levels;
  double cone_half_angle_deg;
  int N, n_mat;
  const double* sigma_t;  /* [n_mat] */
  const double* moments;  /* [n_mat][N+1], sigma_{s,n} */
  const int* mat_of_el;   /* [n_el] or NULL */
  const double* q_el;     /* [n_el] isotropic source density, or NULL */
  int beam;               /* 0 none, 2 unit beam on x=0 inside the cone */
  double strength, x0, x1, y0, y1;
  int nr, n_levels, nu_pre, nu_post, coarse_sweeps;
  double coarse_tol;
} stamg_problem;

/* Host-side collective: sum n doubles element-wise across all ranks, in place.
 * buf is pinned host memory owned by the context; the context's stream is
 * synchronised before the call and the result is copied back after it.
 * Return 0 on success (anything else fails the operator with STAMG_ENCCL).
 * For in-process multi-rank emulation, tests and custom transports; the
 * production multi-GPU path is NCCL (nccl_id). */
typedef int (*stamg_allreduce_fn)(void* user, double* buf, int64_t n);

typedef struct {
  int device;            /* CUDA device ordinal */
  int rank, world;       /* direction sharding; world = 1 for one GPU */
  const void* nccl_id;   /* 128-byte ncclUniqueId when world > 1, else NULL */
  int build_hierarchy;   /* 0: outer level only (sweep/scatter throughput) */
  /* world > 1 needs exactly one of: nccl_id, allreduce, shard_probe */
  stamg_allreduce_fn allreduce;  /* host collective (see above), or NULL */
  void* allreduce_user;          /* passed to allreduce */
  int shard_probe;       /* timing only: this rank's slice runs alone and every
                            collective is skipped, so scatter moments, dots and
                            the scalar flux are partial sums (tools/shard_probe.py) */
} stamg_options;

typedef struct {
  int iterations, converged, breakdown, preconditioner_applications;
  double final_residual, wall_time;
} stamg_report;

typedef struct stamg_ctx stamg_ctx;
typedef struct stamg_vec stamg_vec;

const char* stamg_last_error(void);
int stamg_version(void);

/* build_operators + build_sweep_plan + build_hierarchy
 * (transport.hpp:47-49, sweeps.hpp:22, multigrid.hpp:50): host setup, then
 * the per-level tables are uploaded once. */
int stamg_create(const stamg_problem* prob, const stamg_options* opt, stamg_ctx** out);
int stamg_destroy(stamg_ctx* ctx);
int stamg_nccl_unique_id(void* out128);
/* One-rank round trip through every NCCL call the sharded contexts make (dlopen, unique id,
 * ncclCommInitRank, ncclCommSplit, ncclAllReduce of n doubles, destroy) on `device`;
 * *version_out = ncclGetVersion. STAMG_ENCCL if any step fails. */
int stamg_nccl_selftest(int device, int64_t n, int* version_out);

/* Layout of a level (layout.hpp:16-32): out4 = {n_el, n_patch, S, D}. */
int stamg_layout(stamg_ctx* ctx, int level, int out4[4]);
/* patch range [q_begin, q_end) owned by this rank at `level` (first/last+1 of the list) */
int stamg_patch_range(stamg_ctx* ctx, int level, int* q_begin, int* q_end);
/* leaf-order positions of this rank's patches at `level` (vectors hold them in this order) */
int stamg_patch_list(stamg_ctx* ctx, int level, int* out, int cap, int* n);
/* host only, no device: the partition rank `rank` of `world` gets (level 0 = coarsest MG
 * level, replicated) and, for level >= 1, each patch's parent position in the coarser
 * level's list held by the same rank */
int stamg_partition(const stamg_problem* prob, int rank, int world, int level, int* qpos, int* up, int cap, int* n);
/* Host-only: the directions (global leaf positions, ascending) rank `rank` of `world` owns
 * in a context without a hierarchy: whole orbits of the mesh's reflection symmetry, so
 * every rank folds its own scatter (contiguous slices of 4 patches without symmetry). */
int stamg_shard_patches(const stamg_problem* prob, int rank, int world, int* out, int cap, int* n);
/* Host only, no device: an outer-level table as the host setup builds it ("X" couplings
 * [P*D][H], scatter.hpp:32-39; "B" diagonal blocks, transport.hpp:38; "C" inflow blocks;
 * "M1" patch mass row sums; "octant" per patch; "rhs" assemble_rhs, transport.hpp:62;
 * "layout" {n_el, P, S, D}).
 * Call with out = NULL to get the length in *n. */
int stamg_host_table(const stamg_problem* prob, const char* name, double* out, int64_t cap, int64_t* n);
int stamg_n_levels(stamg_ctx* ctx, int* n_levels, int* nr);
/* scatter order of a level's coupling table (ops.kernel.N) */
int stamg_level_order(stamg_ctx* ctx, int level, int* order);

/* ---- vectors (FluxVector, layout.hpp:14), device resident ---- */
int stamg_vec_create(stamg_ctx* ctx, int level, stamg_vec** out);
int stamg_vec_free(stamg_vec* v);
int stamg_vec_size(stamg_vec* v, int64_t* n);
/* Device storage order: the reference layout ((el*P+q)*D+d)*S+i, except on contexts
 * without a hierarchy whose level qualifies for 8-direction groups, which store the
 * "wavefront layout" (per 8-direction group, cells along the sweep's skewed
 * anti-diagonals; STAMG_WAVEFRONT_LAYOUT=0 disables it). Upload,
 * download, the host-buffer entry points and stamg_vec_size always use the
 * reference layout; only the raw device pointer exposes the internal order. */
int stamg_vec_device_ptr(stamg_vec* v, double** ptr);
int stamg_vec_upload(stamg_ctx* ctx, stamg_vec* v, const double* host, int64_t n);
int stamg_vec_download(stamg_ctx* ctx, const stamg_vec* v, double* host, int64_t n);
int stamg_vec_fill(stamg_ctx* ctx, stamg_vec* v, double value);
int stamg_vec_copy(stamg_ctx* ctx, const stamg_vec* src, stamg_vec* dst);
int stamg_vec_axpy(stamg_ctx* ctx, double a, const stamg_vec* x, stamg_vec* y);      /* y += a x */
int stamg_vec_dot(stamg_ctx* ctx, const stamg_vec* x, const stamg_vec* y, double* out);

/* ---- hot-path operators ---- */
/* apply_L_into (transport.hpp:52-53): y = L phi */
int stamg_apply_L(stamg_ctx* ctx, int level, const stamg_vec* phi, stamg_vec* y);
/* apply_scatter_into (scatter.hpp:53-57): y += scale * S_order phi */
int stamg_apply_scatter(stamg_ctx* ctx, int level, const stamg_vec* phi, int max_order, double scale,
                        stamg_vec* y);
/* apply_A_into (transport.hpp:57-58): y = (L - S_order) phi */
int stamg_apply_A(stamg_ctx* ctx, int level, const stamg_vec* phi, int order, stamg_vec* y);
/* standard_sweep (sweeps.hpp:25-26): z = L^{-1} rhs; z may alias rhs */
int stamg_sweep(stamg_ctx* ctx, int level, const stamg_vec* rhs, stamg_vec* z);
/* coarse_scatter_sweep (sweeps.hpp:32-33): nu scatter-implicit GS passes */
int stamg_coarse_gs(stamg_ctx* ctx, int level, const stamg_vec* rhs, int nu, stamg_vec* phi);
/* smoother_step (sweeps.hpp:36-37): phi += L^{-1}(f - A_order phi) */
int stamg_smoother_step(stamg_ctx* ctx, int level, const stamg_vec* f, int order, stamg_vec* phi);
/* prolongate / restrict_residual (multigrid.hpp:52-53), level l >= 1 */
int stamg_prolongate(stamg_ctx* ctx, int l, const stamg_vec* coarse, stamg_vec* fine);
int stamg_restrict(stamg_ctx* ctx, int l, const stamg_vec* fine, stamg_vec* coarse);
/* lmg_vcycle / mg_apply (multigrid.hpp:56-60) */
int stamg_vcycle(stamg_ctx* ctx, int l, const stamg_vec* f, stamg_vec* phi);
int stamg_mg_apply(stamg_ctx* ctx, const stamg_vec* r, stamg_vec* z);
/* assemble_rhs (transport.hpp:62) into an outer-level vector */
int stamg_rhs(stamg_ctx* ctx, stamg_vec* f);

/* Krylov: method 0 = BiCGSTAB (krylov.hpp:27-30), 1 = GMRES(restart) (new);
 * precond 0 = standard_sweep, 1 = mg_apply, 2 = none. x0 = 0. */
int stamg_solve(stamg_ctx* ctx, int method, int precond, const stamg_vec* b, stamg_vec* x, double tol,
                int max_iter, int restart, stamg_report* rep, double* history, int history_cap);

/* Host-buffer entry points (what a reference-side FFI binds): copy in, run,
 * copy out. stamg_sweep_host pipelines the copies with the sweep over chunks of
 * direction groups (host->device, sweep and device->host of different chunks
 * run concurrently); rhs and z may be the same buffer. */
int stamg_sweep_host(stamg_ctx* ctx, int level, const double* rhs, double* z, int64_t n);
int stamg_solve_host(stamg_ctx* ctx, int method, int precond, const double* b, double* x, int64_t n,
                     double tol, int max_iter, int restart, stamg_report* rep);

/* harness.cpp:183-205 scalar flux per element (integral / volume), host out */
int stamg_scalar_flux(stamg_ctx* ctx, const stamg_vec* phi, double* out_host);

/* Source iteration step (sweeps.cpp:106-113 with the moment-only storage of
 * SURVEY.md §8(f) rank 1): psi <- q_ext + S phi (M2D), psi <- L^{-1} psi
 * (in-place sweep), mom <- D2M(psi) (+ allreduce over ranks). */
int stamg_source_iteration(stamg_ctx* ctx, stamg_vec* psi, int n_iter);

/* table introspection for parity tests */
int stamg_get_table(stamg_ctx* ctx, int level, const char* name, double* out, int64_t cap, int64_t* n);

int stamg_synchronize(stamg_ctx* ctx);
/* FP64 tensor (DMMA) and FP64 FMA throughput probes, TFLOP/s (roofline denominators) */
int stamg_bench_fp64_peaks(stamg_ctx* ctx, double* dmma_tflops, double* dfma_tflops);
/* pinned host buffers for the host-buffer entry points */
int stamg_host_alloc(int64_t bytes, void** out);
int stamg_host_free(void* p);
/* chunks the last stamg_sweep_host was pipelined over (0: serial copy-sweep-copy) */
int stamg_host_pipeline_chunks(stamg_ctx* ctx, int* n);
/* kernel launches issued by this context since creation (for bench) */
int stamg_launch_count(stamg_ctx* ctx, int64_t* n);
/* per-kernel device time accounting: enable and read (ms) */
int stamg_timing_enable(stamg_ctx* ctx, int on);
int stamg_timing_read(stamg_ctx* ctx, const char* kernel, double* ms, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* STAMG_B200_H */
