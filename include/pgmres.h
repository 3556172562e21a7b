/* pgmres.h — C ABI of the B200-native deflated PGMRES library (libpgmres.so).
 *
 * Drop-in boundary for the reference's linear-solve path.  Each entry point
 * replaces one reference interface (file:line into /root/reference/proj):
 *
 *   pgm_solve ................ deflated_gmres(A, b, x, cfg, Deflator&, Executor&)
 *                              include/dgmres/deflation.hpp:97-98, and
 *                              gmres_restarted(opA=spmv, opM=nullptr, ...)
 *                              include/dgmres/gmres.hpp:110-113 (deflator NULL)
 *   pgm_context_create ....... Executor(Partition, deterministic)  parallel.hpp:86-91
 *                              + partition_rows                     parallel.hpp:43
 *   pgm_matrix_upload ........ CsrMatrix hand-off                   sparse.hpp:17-24
 *   pgm_matrix_update_values . assemble_jacobian value rewrite      assembly.cpp:253,288
 *   pgm_spmv ................. Executor::spmv                       parallel.hpp:93
 *   pgm_deflator_* ........... class Deflator                       deflation.hpp:35-89
 *   pgm_report_* ............. GmresReport / write_csv              gmres.hpp:31-44
 *   pgm_newton_solve ......... newton_solve (caller of the path)    newton.hpp:45-54
 *
 * Conventions: plain pointers and sizes; every function returns a pgm_status
 * (0 = OK).  The message of the last failure is pgm_last_error(ctx).  Host
 * pointers unless the PGM_DEVICE_PTRS flag says the arrays are CUDA device
 * memory on the context's device.  All arithmetic is fp64; indices are
 * uint32 like the reference's index_t (mesh.hpp:8).
 */
#ifndef PGMRES_H_
#define PGMRES_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PGM_OK = 0,
  PGM_EINVAL = 1,     /* std::invalid_argument in the reference            */
  PGM_ENONFINITE = 2, /* gmres.cpp:151-153,165-169,195-198 runtime_error   */
  PGM_ESINGULAR = 3,  /* gmres.cpp:97-99 singular projection               */
  PGM_ECUDA = 4,
  PGM_ENCCL = 5,
  PGM_ENOMEM = 6,
  PGM_ESTATE = 7
} pgm_status;

enum { PGM_DEVICE_PTRS = 1 };

typedef struct pgm_context pgm_context;
typedef struct pgm_matrix pgm_matrix;
typedef struct pgm_deflator pgm_deflator;
typedef struct pgm_loopback pgm_loopback;

#define PGM_DETERMINISTIC_PLANES 2

/* One rank of a z-slab row-block partition (parallel.cpp:50-71). */
typedef struct {
  int32_t device;         /* CUDA ordinal this rank drives                   */
  int32_t rank, world;    /* world = 1: single GPU                           */
  const void* nccl_id;    /* 128-byte ncclUniqueId from rank 0 (world > 1);  */
                          /* NULL with world > 1 and no loopback: peer-only  */
                          /* (no NCCL; solves need pgm_peer_import first)   */
  pgm_loopback* loopback; /* instead of NCCL: in-process group of `world`    */
                          /* contexts driven by one host thread each         */
  uint32_t n_axis;        /* node planes; plane = n_axis^2 rows.  Required   */
                          /* when world > 1 (z-slab partition); 0 = no mesh  */
                          /* structure, accepted for world = 1 only          */
  uint32_t n_global;      /* total rows                                      */
  int32_t deterministic;  /* 0 / 1: reductions in a fixed order (bitwise     */
                          /* reproducible run to run for a given partition); */
                          /* PGM_DETERMINISTIC_PLANES: every reduction is    */
                          /* per-plane sequential partials + the reference's */
                          /* pairwise fold (parallel.cpp:33-46,120-131) —    */
                          /* bit-identical for ANY rank count (and equal to  */
                          /* the reference executor's dot); slower; no peer  */
                          /* transport                                       */
} pgm_context_config;

typedef struct {
  uint32_t row_begin, row_end;  /* owned rows [begin, end)                   */
  uint32_t halo_lo, halo_hi;    /* halo rows read below / above              */
} pgm_partition;

typedef struct {
  uint32_t n;               /* rows in this view (owned rows of this rank)   */
  uint64_t nnz;
  const uint32_t* row_ptr;  /* n+1 offsets starting at 0                     */
  const uint32_t* col_idx;  /* GLOBAL column ids, ascending within a row     */
  const double* values;
} pgm_csr_view;

typedef struct { /* GmresConfig, gmres.hpp:17-23 */
  uint32_t m;
  uint32_t max_restarts;
  double rel_tol;
  int32_t fixed_iterations;
  double breakdown_scale;
} pgm_gmres_config;

typedef struct { /* DeflationConfig, deflation.hpp:15-22 */
  uint32_t r_max;
  uint32_t drop;
  double accept_tol;
  uint32_t inv_power_maxit;
  double inv_power_tol;
  uint32_t power_maxit;
} pgm_deflation_config;

typedef struct { /* GmresReport, gmres.hpp:31-44 (arrays owned; pgm_report_free) */
  double beta0;
  uint32_t restarts;
  uint64_t total_inner;
  int32_t converged;
  int32_t breakdown;
  double final_relative;
  uint32_t n_inner;            /* InnerRecord count                          */
  uint32_t* inner_restart;     /* [n_inner]                                  */
  uint32_t* inner_step;        /* [n_inner]                                  */
  double* inner_monitored;     /* [n_inner] |gamma_{k+1}|                    */
  double* explicit_residual;   /* [restarts]                                 */
  double solve_seconds;        /* device time of the solve (CUDA events)     */
} pgm_report;

typedef struct { /* DeflationRecord, deflation.hpp:24-29 */
  uint32_t restart;
  uint32_t r;
  double mu;
  double smallest_ritz;
} pgm_deflation_record;

/* ---- context ----------------------------------------------------------- */
pgm_status pgm_context_create(const pgm_context_config* cfg, pgm_context** out);
void pgm_context_destroy(pgm_context* ctx);
const char* pgm_last_error(const pgm_context* ctx);
pgm_status pgm_context_partition(const pgm_context* ctx, pgm_partition* out);
/* In-process communicator for world > 1 without NCCL (one host thread per
 * rank, typically all on one GPU): same kernels and partition as the NCCL
 * path, host-staged collectives.  Used to test the multi-rank path. */
pgm_status pgm_loopback_create(int32_t world, pgm_loopback** out);
void pgm_loopback_destroy(pgm_loopback* g);
/* partition_rows(mesh, p)[w] without a context (parallel.cpp:50-71). */
pgm_status pgm_partition_rows(uint32_t n_axis, uint32_t p, uint32_t w, pgm_partition* out);
/* Device stream the library enqueues on (cudaStream_t), for callers that
 * time or order work around it. */
void* pgm_context_stream(pgm_context* ctx);

/* ---- matrix ------------------------------------------------------------ */
pgm_status pgm_matrix_upload(pgm_context* ctx, const pgm_csr_view* a, int32_t flags,
                             pgm_matrix** out);
pgm_status pgm_matrix_update_values(pgm_matrix* a, const double* values, int32_t flags);
void pgm_matrix_destroy(pgm_matrix* a);
pgm_status pgm_matrix_info(const pgm_matrix* a, uint32_t* n, uint64_t* nnz,
                           uint64_t* stored, uint64_t* device_bytes);
/* y = A x over the owned rows (halo exchange included when world > 1). */
pgm_status pgm_spmv(pgm_matrix* a, const double* x, double* y, int32_t flags);

/* ---- deflation preconditioner -------------------------------------------- */
pgm_status pgm_deflator_create(pgm_context* ctx, const pgm_deflation_config* cfg,
                               pgm_deflator** out);
void pgm_deflator_destroy(pgm_deflator* d);
pgm_status pgm_deflator_reset(pgm_deflator* d);
pgm_status pgm_deflator_info(pgm_deflator* d, uint32_t* rank, double* mu, uint32_t* skipped,
                             uint32_t* n_history);
pgm_status pgm_deflator_history(pgm_deflator* d, pgm_deflation_record* out, uint32_t cap);
/* U (n_own x rank, column-major) and T (rank x rank, column-major). */
pgm_status pgm_deflator_basis(pgm_deflator* d, double* U, double* T);
/* Deflator::push_vector with opA = spmv(a) (deflation.cpp:123-184). */
pgm_status pgm_deflator_push(pgm_deflator* d, pgm_matrix* a, const double* candidate,
                             int32_t flags, int32_t* accepted);
pgm_status pgm_deflator_truncate(pgm_deflator* d);
pgm_status pgm_deflator_observe_ritz(pgm_deflator* d, double value);
/* w = v + U(|mu| T^{-1} - I) U^T v (deflation.cpp:104-117). */
pgm_status pgm_deflator_apply(pgm_deflator* d, const double* v, double* w, int32_t flags);

/* ---- the solve ----------------------------------------------------------- */
/* deflated_gmres when d != NULL, plain gmres_restarted otherwise.  x holds the
 * initial guess on entry and the iterate on return; b and x cover the owned
 * rows.  rep may be NULL. */
pgm_status pgm_solve(pgm_context* ctx, pgm_matrix* a, pgm_deflator* d, const double* b,
                     double* x, const pgm_gmres_config* cfg, int32_t flags, pgm_report* rep);
void pgm_report_free(pgm_report* rep);

/* Restart observer — the RestartHook of gmres_restarted (gmres.hpp:94-113,
 * gmres.cpp:189) for audits such as acceptance.cpp:100-122 (criterion 8):
 * called on the host after every restart cycle's x update and deflation
 * harvest, before the explicit residual, with the 0-based cycle index and
 * the Arnoldi steps it completed.  Inside the callback the cycle's basis and
 * Hessenberg matrix can be read (below) and the deflator inspected
 * (pgm_deflator_info / _history / _basis); no other pgm_* call on this
 * context is allowed.  A nonzero return stops the solve with PGM_ESTATE.
 * cb = NULL removes the observer (then nothing synchronises mid-solve). */
typedef int32_t (*pgm_restart_observer)(void* user, uint32_t restart, uint32_t steps);
pgm_status pgm_set_restart_observer(pgm_context* ctx, pgm_restart_observer cb, void* user);
/* v_j (j < steps, owned rows) into host memory: GmresWorkspace::basis(j). */
pgm_status pgm_restart_basis(pgm_context* ctx, uint32_t j, double* out);
/* The cycle's unrotated Hessenberg matrix, (m+1) x m column-major
 * (GmresWorkspace::hess(i, j) = out[i + j (m+1)], valid for j < steps). */
pgm_status pgm_restart_hessenberg(pgm_context* ctx, double* out);

/* 128-byte ncclUniqueId for pgm_context_config.nccl_id (call on rank 0 and
 * broadcast it, e.g. with torch.distributed). */
pgm_status pgm_nccl_unique_id(void* out128);

/* Peer-memory transport (world > 1, one process per GPU): every reduction
 * kernel all-reduces inside its last block by storing its sums into every
 * rank's window over NVLink (CUDA IPC mapping) — no NCCL call, no extra
 * kernel — and the halo planes go through mailboxes in the neighbours'
 * windows (k_halo_push / k_halo_pull).  Export this rank's 128-byte window
 * handle, gather all ranks' handles in rank order (e.g.
 * torch.distributed.all_gather), import them.  Without the import an NCCL
 * context keeps the NCCL allreduce and send/recv halos; a peer-only context
 * (nccl_id NULL) refuses to solve.  Requires CUDA_MODULE_LOADING=EAGER.  In-process
 * loopback groups use the peer transport by default (PGMRES_PEER=0: off). */
pgm_status pgm_peer_export(pgm_context* ctx, void* out128);
pgm_status pgm_peer_import(pgm_context* ctx, const void* all /* world * 128 bytes */);

/* Kernel launches of the last pgm_solve (evidence for the bench). */
uint64_t pgm_context_launch_count(const pgm_context* ctx);
/* Optional CUDA-event timing of every hot-path kernel of the next solves
 * (class ids: 0 step SpMV, 1 CGS2 pass B (CGS2 step only), 2 DCGS2 update / CGS2
 * pass C, 3 x update,
 * 4 Ritz, 5 push sweeps, 6 push SpMV, 7 rotate, 8 residual, 9 other;
 * world > 1: 10 halo planes — the reference Executor's "local" time,
 * parallel.cpp:249-253 — and 11 NCCL allreduce + replicated finisher — its
 * "global" time, parallel.cpp:297-300; on the peer transport the allreduce
 * runs inside the reduction kernels and is not separable). */
pgm_status pgm_context_set_profiling(pgm_context* ctx, int32_t on);
uint32_t pgm_context_profile(pgm_context* ctx, uint32_t* cls, uint32_t* cycle, uint32_t* k,
                             float* ms, uint32_t cap);

/* ---- caller side: FEM assembly of the Bratu system ---------------------- *
 * pattern_nnz / symbolic_pattern / assemble_jacobian / assemble_residual
 * (assembly.hpp:32-49) on the device for the context's owned rows: writes
 * row_ptr (n_own + 1), col_idx, values (nnz) and rhs = -R(u) (n_own).  u is the
 * global iterate (NULL = 0, the first Newton system).  Bit-identical to the
 * reference assembly at u = 0. */
pgm_status pgm_bratu_nnz(const pgm_context* ctx, uint32_t n_e, uint64_t* nnz);
pgm_status pgm_bratu_assemble(pgm_context* ctx, uint32_t n_e, double lambda, const double* u,
                              int32_t flags, uint32_t* row_ptr, uint32_t* col_idx,
                              double* values, double* rhs);

/* ---- caller side: the Newton driver -------------------------------------- *
 * newton_solve (newton.hpp:45-54, newton.cpp:31-97) for the Bratu problem on
 * the (2 n_e + 1)^3 mesh, device-resident: assembly, deflated PGMRES solve,
 * update and norms run on the GPU; the host reads two scalars per iteration.
 * u is the GLOBAL iterate (n_global entries; initial guess in, solution out:
 * every rank writes its owned rows).  Same stopping rule and records as the
 * reference: stop when ||delta||_inf <= update_tol, optional lambda
 * continuation.  Errors: EINVAL for max_iters = 0 ("newton: max_iters must be
 * positive"), plus every pgm_solve error. */
typedef struct { /* NewtonConfig, newton.hpp:15-23 */
  uint32_t max_iters;
  double update_tol;
  pgm_gmres_config gmres;
  pgm_deflation_config deflation;
  int32_t use_deflation;
  int32_t continuation;
  uint32_t continuation_steps;
} pgm_newton_config;

typedef struct { /* NewtonIterRecord, newton.hpp:25-32 */
  uint32_t iter;
  double lambda;
  double update_inf;
  double residual_norm;
  uint32_t gmres_restarts;
  uint64_t gmres_inner;
} pgm_newton_record;

typedef struct { /* NewtonReport, newton.hpp:34-43 (iters owned; pgm_newton_report_free) */
  pgm_newton_record* iters;
  uint32_t n_iters;
  int32_t converged;
  double final_residual;
  double final_update;
  uint64_t total_inner;
  double seconds; /* wall time of the driver (host clock) */
} pgm_newton_report;

pgm_status pgm_newton_solve(pgm_context* ctx, uint32_t n_e, double lambda, double* u,
                            int32_t flags, const pgm_newton_config* cfg, pgm_newton_report* rep);
void pgm_newton_report_free(pgm_newton_report* rep);

#ifdef __cplusplus
}
#endif
#endif /* PGMRES_H_ */
