// Shared device-side definitions of libpgmres: state structs, launch geometry,
// deterministic two-level grid reductions.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pgm {

// ---- launch geometry -------------------------------------------------------
#ifndef PGM_TILE
#define PGM_TILE 512
#endif
constexpr int TILE = PGM_TILE;        // rows per SpMV tile (SELL sort window)
constexpr int SPT = TILE / 32;        // 32-row slices per tile
#ifndef PGM_SPMV_THREADS
#define PGM_SPMV_THREADS 256  // threads per SpMV block (one TILE-row tile per block)
#endif
constexpr int SPMV_THREADS = PGM_SPMV_THREADS;
#ifndef PGM_SPMV_UNROLL
#define PGM_SPMV_UNROLL 4
#endif
#ifndef PGM_SPMV_PREFETCH
#define PGM_SPMV_PREFETCH 1
#endif
#ifndef PGM_SPMV_MINB
#define PGM_SPMV_MINB 4
#endif
constexpr int SPMV_UNROLL = PGM_SPMV_UNROLL;  // entries per lane per pipeline stage
constexpr int SPMV_MINB = PGM_SPMV_MINB;      // min resident blocks per SM (register cap)
constexpr int SW_THREADS = 128;       // sweep block: one row per thread
constexpr int CH = SW_THREADS;        // rows per sweep chunk
constexpr int GROUP = 32;             // first-level reduction group (blocks, one per lane)
constexpr int MAX_M = 112;            // Ritz harvest keeps [H | H^-1] in smem
constexpr int MAX_R1 = 32;            // r_max + 1 bound of the register fast path
constexpr int RITZ_THREADS = 256;

// ---- device state ------------------------------------------------------------
// Per-solve GMRES control word (gmres.cpp:132-218 loop variables + GmresReport
// scalars).  Lives in device memory; the host reads it once per restart.
struct GState {
  int active;       // inner loop of the current cycle still running
  int done;         // solve finished (converged, max restarts, or error)
  int error;        // pgm_status code
  int err_restart, err_step;
  int restart;      // current 0-based cycle
  int steps;        // Arnoldi steps completed in the current cycle
  int lucky;        // cycle ended on h < breakdown_scale * beta
  int converged, breakdown, restarts, n_inner;
  int dc_fallback;  // DCGS2 remainder hit rounding level: later cycles use CGS2
  unsigned long long total_inner;
  double beta0, beta, beta_cycle, final_relative;
  // configuration (GmresConfig)
  int m, max_restarts, fixed, harvest;
  double rel_tol, breakdown_scale;
};

// Deflator state (deflation.hpp:78-88) kept on the device across solves.
struct DState {
  int r, skipped, n_hist, hist_cap;
  double mu;
  int r_max, drop, inv_maxit, pow_maxit;
  double accept_tol, inv_tol;
  // restart-harvest pipeline (update_from_restart / push_vector)
  int push_ok;      // candidate still alive
  int rotate;       // truncation produced Q; U, AU need rotating
  int r0;           // rank before truncation (columns of Q)
  int trunc_fail;   // eigen decomposition failed (stderr in the reference)
  double theta, norm_in, pscale;
};

struct Params {
  GState* g;
  DState* d;
  // GMRES small arrays (m-sized, device)
  double *s;                      // lazy scale of stored basis column W_l: v_l = s_l W_l
  double *h_orig, *h_rot;         // (m+1) x m column-major
  double *gv, *cs, *sn;           // rotated rhs, Givens
  double *h1, *coefA, *coefB;     // CGS2 pass coefficients
  double *tU;                     // (m+1) x R1: U^T v_l for every basis vector
  double *c;                      // deflation coefficients for the next apply
  double *xc, *cx;                // x update: V y and U c' coefficients
  double *zl;                     // Ritz lift coefficients (V z)
  uint32_t *rec_restart, *rec_step;
  double *rec_mon, *expl;
  // deflation small arrays (R1-sized)
  double *T, *Tinv, *Q, *proj, *dwork;
  int* iwork;
  uint32_t *hist_restart, *hist_r;
  double *hist_mu, *hist_theta;
  // n-sized vectors: each a padded buffer of ld doubles, own rows at +lo
  double *V, *U, *AU, *x, *b, *u;
  size_t ld;
  int n, lo, m, R1;
  // reduction scratch
  double *part, *gpart, *g2part;
  unsigned* cnt;
  double* red_out;  // world > 1: block-reduced local sums for the allreduce
  int world;
  // fused peer-memory allreduce (world > 1, peer mode): every rank's comm
  // window is mapped into every other rank (NVLink P2P / CUDA IPC, or plain
  // pointers for in-process ranks)
  int peer, rank;
  double* const* peer_win;                  // [world] -> window [2][world][PEER_NV]
  unsigned long long* const* peer_flag;     // [world] -> flags  [2][world]
  const double* win_local;
  const unsigned long long* flag_local;
  unsigned long long* epoch;                // this rank's reduction counter
  // deterministic mode (pgm_context_config.deterministic = 2): every
  // reduction is recomputed as per-plane sequential partials + the
  // reference's pairwise fold (k_det_dots), bit-identical for any rank count
  int det;
  int plane;            // rows per node plane (n_axis^2; n for world = 1 without mesh)
  int nplanes;          // this rank's planes
  double* det_pp;       // [nv][nplanes] this rank's plane partials
  const double* det_all;  // world > 1: [nv][nplanes_global] gathered partials
  int nplanes_global;
  unsigned* det_cnt;    // completion counter of k_det_dots
};

constexpr int PEER_NV = 2 * MAX_R1 + MAX_M + 8;  // values per reduction slot

// ---- programmatic dependent launch (PDL) -------------------------------------
// The hot-path kernels are launched with programmatic stream serialization:
// kernel N+1 may become resident once every block of kernel N has passed
// pdl_trigger() (end of its main loop), runs its prologue (L2 prefetch of
// data written >= 2 kernels back, never data of kernel N), then blocks in
// pdl_wait() until kernel N has completed and its writes are visible.  Every
// kernel calls pdl_trigger() only after its own pdl_wait(), so "written >= 2
// kernels back" is always complete.  Without the launch attribute both are
// no-ops.
#ifndef PGM_PDL_ASM
#define PGM_PDL_ASM 1
#endif
#ifndef PGM_SPMV_EARLY_PF
#define PGM_SPMV_EARLY_PF 1
#endif
__device__ __forceinline__ void pdl_wait() {
#if PGM_PDL_ASM
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#if PGM_PDL_ASM
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// ---- reductions ---------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// bvals: the block's nv sums (smem).  Every block writes them; the last block
// of every GROUP sums its group in block order; the last group-reducer sums
// the groups in order and returns true (in every thread of that block) with
// red[0..nv) filled.  The summation order depends only on the grid size, so
// results are identical run to run.  Both levels handle VPW values per warp
// pass so that several dependent L2 round trips overlap (the tail of every
// reduction kernel is latency-bound).
#ifndef PGM_VPW
#define PGM_VPW 4
#endif
constexpr int VPW = PGM_VPW;
// G / bid: the reduction's block count and this block's index in it (a
// reduction may span several launches, e.g. the interior and boundary tiles
// of a halo-overlapped SpMV; partials are indexed by tile, so the order is
// the same however the launches interleave).
#ifndef PGM_TAIL_TIMING
#define PGM_TAIL_TIMING 0  // tuning variant: %globaltimer stamps of the reduction tail
#endif
#if PGM_TAIL_TIMING
__device__ unsigned long long g_tail_ns[16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__shared__ unsigned long long s_tail_t[3];
#endif
#ifndef PGM_RED_ACQREL
#define PGM_RED_ACQREL 1
#endif
// Arrival counter of the grid reduction: CTA barrier, then ONE acq_rel RMW by
// thread 0 (release: the CTA's partials, ordered before it by the barrier;
// acquire: every earlier arrival's partials) — the pattern of a semaphore
// arrive, instead of a block-wide __threadfence before and after a relaxed
// atomic (each fence is a full round trip on the reduction's critical path).
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
#if PGM_RED_ACQREL
#define PGM_ARRIVE(ctr, last_at)                                   \
  __syncthreads();                                                 \
  if (threadIdx.x == 0) s_flag = (atom_add_acqrel((ctr), 1u) == (unsigned)(last_at)); \
  __syncthreads();
#define PGM_ARRIVED_FENCE()
#else
#define PGM_ARRIVE(ctr, last_at)                                   \
  __threadfence();                                                 \
  __syncthreads();                                                 \
  if (threadIdx.x == 0) s_flag = (atomicAdd((ctr), 1u) == (unsigned)(last_at)); \
  __syncthreads();
#define PGM_ARRIVED_FENCE() __threadfence();
#endif
__device__ __forceinline__ bool grid_reduce_ex(const double* bvals, int nv, const Params& P,
                                               double* red, int G, int bid) {
  __shared__ int s_flag;
#if PGM_TAIL_TIMING
  if (threadIdx.x == 0) s_tail_t[0] = gtimer();
#endif
  const int NG = (G + GROUP - 1) / GROUP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int v = threadIdx.x; v < nv; v += blockDim.x) P.part[(size_t)v * G + bid] = bvals[v];
  const int grp = bid / GROUP;
  const int g0 = grp * GROUP;
  const int gsize = min(GROUP, G - g0);
  PGM_ARRIVE(&P.cnt[1 + grp], gsize - 1)
  if (!s_flag) return false;
  PGM_ARRIVED_FENCE()
  // level 1: lane = block of the group, VPW values per warp pass
  for (int v0 = warp * VPW; v0 < nv; v0 += nw * VPW) {
    double s[VPW];
#pragma unroll
    for (int q = 0; q < VPW; ++q)
      s[q] = (v0 + q < nv && lane < gsize) ? __ldcg(&P.part[(size_t)(v0 + q) * G + g0 + lane]) : 0.0;
#pragma unroll
    for (int q = 0; q < VPW; ++q) s[q] = warp_sum(s[q]);
    if (lane < VPW && v0 + lane < nv) {
      double o = s[0];
#pragma unroll
      for (int q = 1; q < VPW; ++q)
        if (lane == q) o = s[q];
      P.gpart[(size_t)(v0 + lane) * NG + grp] = o;
    }
  }
  if (threadIdx.x == 0) P.cnt[1 + grp] = 0;
  // level 2: with more than GROUP groups, super-groups of GROUP groups are
  // summed by their last group-reducer (distributed), so the final block
  // reads at most GROUP partials per value (a single block walking ~1000
  // groups per value was ~25 us of the step at n_e = 125)
  const int NS = (NG + GROUP - 1) / GROUP;
  const double* lvl = P.gpart;
  int nlvl = NG;
  if (NS > 1) {
    const int sg = grp / GROUP, s0 = sg * GROUP, ssize = min(GROUP, NG - s0);
    PGM_ARRIVE(&P.cnt[1 + NG + sg], ssize - 1)
    if (!s_flag) return false;
    PGM_ARRIVED_FENCE()
    for (int v0 = warp * VPW; v0 < nv; v0 += nw * VPW) {
      double s[VPW];
#pragma unroll
      for (int q = 0; q < VPW; ++q)
        s[q] = (v0 + q < nv && lane < ssize) ? __ldcg(&P.gpart[(size_t)(v0 + q) * NG + s0 + lane]) : 0.0;
#pragma unroll
      for (int q = 0; q < VPW; ++q) s[q] = warp_sum(s[q]);
      if (lane < VPW && v0 + lane < nv) {
        double o = s[0];
#pragma unroll
        for (int q = 1; q < VPW; ++q)
          if (lane == q) o = s[q];
        P.g2part[(size_t)(v0 + lane) * NS + sg] = o;
      }
    }
    if (threadIdx.x == 0) P.cnt[1 + NG + sg] = 0;
    lvl = P.g2part;
    nlvl = NS;
  }
  PGM_ARRIVE(&P.cnt[0], (NS > 1 ? NS : NG) - 1)
  if (!s_flag) return false;
  PGM_ARRIVED_FENCE()
#if PGM_TAIL_TIMING
  if (threadIdx.x == 0) s_tail_t[1] = gtimer();
#endif
  // final level: lanes stride over the partials, VPW values per warp pass
  for (int v0 = warp * VPW; v0 < nv; v0 += nw * VPW) {
    double s[VPW];
#pragma unroll
    for (int q = 0; q < VPW; ++q) s[q] = 0.0;
#pragma unroll 4
    for (int g = lane; g < nlvl; g += 32) {
      double t[VPW];
#pragma unroll
      for (int q = 0; q < VPW; ++q)
        t[q] = v0 + q < nv ? __ldcg(&lvl[(size_t)(v0 + q) * nlvl + g]) : 0.0;
#pragma unroll
      for (int q = 0; q < VPW; ++q) s[q] += t[q];
    }
#pragma unroll
    for (int q = 0; q < VPW; ++q) s[q] = warp_sum(s[q]);
    if (lane < VPW && v0 + lane < nv) {
      double o = s[0];
#pragma unroll
      for (int q = 1; q < VPW; ++q)
        if (lane == q) o = s[q];
      red[v0 + lane] = o;
    }
  }
  if (threadIdx.x == 0) P.cnt[0] = 0;
#if PGM_TAIL_TIMING
  if (threadIdx.x == 0) s_tail_t[2] = gtimer();
#endif
  __syncthreads();
  return true;
}

__device__ __forceinline__ bool grid_reduce(const double* bvals, int nv, const Params& P,
                                            double* red) {
  return grid_reduce_ex(bvals, nv, P, red, (int)gridDim.x, (int)blockIdx.x);
}

// ---- fused cross-GPU allreduce over peer memory --------------------------------
// Called by every thread of the reduction's last block with red[0..nv) = this
// rank's sums.  The block pushes them into slot [parity][rank] of EVERY
// rank's window with plain stores over NVLink, fences system-wide, raises its
// epoch flag in every window, waits until all ranks' flags reach the epoch,
// then sums the world slots in rank order: identical bits on every rank, no
// extra kernel, no NCCL call.  Epochs are per-rank counters that advance
// identically (every rank runs the same reduction sequence); two parities
// suffice because a rank can only run ahead by one reduction.  The wait is
// bounded: on timeout the block gives up and flags g->error.
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Wall-clock bound of every cross-rank wait (%globaltimer, ns): generous
// enough for time-sliced ranks (two processes on one GPU without MPS) and
// slow starters, yet a protocol fault still ends in PGM_ESTATE, not a hang.
constexpr unsigned long long PEER_WAIT_NS = 30ull * 1000000000ull;
__device__ __forceinline__ unsigned long long peer_clock_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifndef PGM_PEER_INLINE
#define PGM_PEER_INLINE __noinline__
#endif
// (noinline, arguments by value: the hot kernels keep their register
// allocation and do not spill Params to the stack for the call)
__device__ PGM_PEER_INLINE void peer_allreduce_impl(double* red, int nv, int W, int me,
                                                 double* const* peer_win,
                                                 unsigned long long* const* peer_flag,
                                                 const double* win_local,
                                                 const unsigned long long* flag_local,
                                                 unsigned long long* epoch, GState* g) {
  __shared__ unsigned long long s_e;
  __shared__ int s_timeout;
  if (threadIdx.x == 0) {
    s_e = ++(*epoch);
    s_timeout = 0;
  }
  __syncthreads();
  const unsigned long long e = s_e;
  const int par = (int)(e & 1ull);
#ifdef PGM_PEER_DEBUG
  if (threadIdx.x == 0 && e < 12) printf("peer rank %d e %llu nv %d grid %d\n", me, e, nv, (int)gridDim.x);
#endif
  for (int q = 0; q < W; ++q) {
    double* dst = peer_win[q] + ((size_t)par * W + me) * PEER_NV;
    for (int v = threadIdx.x; v < nv; v += blockDim.x) dst[v] = red[v];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < W) st_release_sys(peer_flag[threadIdx.x] + par * W + me, e);
  if (threadIdx.x < W) {
    const unsigned long long* f = flag_local + par * W + threadIdx.x;
    const unsigned long long t_start = peer_clock_ns();
    long long spins = 0;
    while (ld_acquire_sys(f) < e) {
      if ((++spins & 1023) == 0 && peer_clock_ns() - t_start > PEER_WAIT_NS) {
        s_timeout = 1;
        break;
      }
    }
  }
  __syncthreads();
#ifdef PGM_PEER_DEBUG
  if (s_timeout && threadIdx.x == 0) printf("peer TIMEOUT rank %d e %llu\n", me, e);
  if (threadIdx.x < W && e < 12) printf("peer rank %d sees flag[%d] = %llu\n", me, threadIdx.x, flag_local[par * W + threadIdx.x]);
#endif
  if (s_timeout && threadIdx.x == 0) {
    g->error = 7;  // PGM_ESTATE: a peer never arrived
    g->active = 0;
    g->done = 1;
  }
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < W; ++q) s += __ldcv(win_local + ((size_t)par * W + q) * PEER_NV + v);
    red[v] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ void peer_allreduce(double* red, int nv, const Params& P) {
  peer_allreduce_impl(red, nv, P.world, P.rank, P.peer_win, P.peer_flag, P.win_local,
                      P.flag_local, P.epoch, P.g);
}

// The reduction tail shared by every reduction kernel: local grid reduction,
// then either the finisher (one GPU, or peer mode after the fused allreduce)
// or red_out for the host-side collective (NCCL / loopback) + k_finish.
// Returns true in the block that must run the finisher on red.
__device__ __forceinline__ bool reduce_tail(const double* bvals, int nv, const Params& P,
                                            double* red, int G, int bid) {
  if (P.det) return false;  // k_det_dots recomputes this reduction and finishes it
  if (!grid_reduce_ex(bvals, nv, P, red, G, bid)) return false;
  if (P.world > 1 && !P.peer) {
    for (int v = threadIdx.x; v < nv; v += blockDim.x) P.red_out[v] = red[v];
    return false;
  }
  if (P.peer) peer_allreduce(red, nv, P);
  return true;
}

// Block-wide sum (fixed order), result broadcast to every thread.
__device__ __forceinline__ double block_sum(double v, double* scratch32) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch32[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += scratch32[w];
  return s;
}

}  // namespace pgm
