// libpgmres: B200-native deflated PGMRES behind the C ABI of include/pgmres.h.
//
// Host orchestration only: every vector operation of the hot path runs in the
// kernels of kernels.cuh; the host enqueues one restart cycle at a time and
// reads back a small status word once per restart (no per-step round trip).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <type_traits>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/pgmres.h"
#include <cub/cub.cuh>

#include "bratu.cuh"
#include "kernels.cuh"
#include "nccl_lite.h"

using namespace pgm;

namespace {

thread_local std::string g_tls_err;

struct Status {  // pgm_status + message
  pgm_status code = PGM_OK;
  std::string msg;
};

#define CU(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      return Status{PGM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};     \
    }                                                                                   \
  } while (0)

#define TRY(expr)                 \
  do {                            \
    Status s_ = (expr);           \
    if (s_.code != PGM_OK) return s_; \
  } while (0)

Status einval(const std::string& m) { return Status{PGM_EINVAL, m}; }

template <class T>
Status dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (e == cudaErrorMemoryAllocation) {
    // the stream-ordered pool keeps freed matrix memory (release threshold
    // = inf): hand it back to the device and retry once
    cudaGetLastError();
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      cudaDeviceSynchronize();
      cudaMemPoolTrimTo(pool, 0);
    }
    e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    return Status{PGM_ENOMEM, std::string("cudaMalloc(") + std::to_string(count * sizeof(T)) +
                                  " B): " + cudaGetErrorString(e)};
  }
  return {};
}
template <class T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

// Stream-ordered allocations for the per-matrix arrays (the pool keeps freed
// memory, so the e2e path's upload/destroy per solve does not pay cudaMalloc /
// cudaFree synchronisation).
template <class T>
Status dalloc_async(T** p, size_t count, cudaStream_t st) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), count * sizeof(T), st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return Status{PGM_ENOMEM, std::string("cudaMallocAsync(") +
                                  std::to_string(count * sizeof(T)) + " B): " +
                                  cudaGetErrorString(e)};
  }
  return {};
}
template <class T>
void dfree_async(T*& p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
  p = nullptr;
}

size_t round_up(size_t a, size_t b) { return (a + b - 1) / b * b; }

}  // namespace

// ---------------------------------------------------------------------------
struct pgm_deflator;
struct pgm_context;

// In-process communicator: `world` contexts driven by `world` host threads of
// one process (normally on one GPU).  It replaces only the NCCL transport, so
// the complete world > 1 code path (partitioned rows, halo planes, per-
// reduction allreduce + replicated finisher) runs and is testable on one GPU.
struct pgm_loopback {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<pgm_context*> ctx;
  std::vector<std::vector<double>> host;  // per-rank staging of reduced values
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct pgm_context {
  int device = 0, rank = 0, world = 1;
  // restart observer (pgm_set_restart_observer): called on the host after
  // each cycle's x update and deflation harvest, before the explicit residual
  pgm_restart_observer obs = nullptr;
  void* obs_user = nullptr;
  bool in_obs = false;
  int obs_steps = 0;
  // collective mode: reductions go through red_out + allreduce + k_finish.
  // world > 1, or a 1-rank NCCL communicator (world = 1 with an nccl_id:
  // exercises the NCCL path on one GPU).
  bool coll = false;
  uint32_t n_axis = 0, n_global = 0;
  pgm_partition part{};
  size_t n = 0, lo = 0, hi = 0, ld = 0;
  cudaStream_t stream = nullptr;
  int nsm = 148;
  std::string err;
  uint64_t launches = 0;
  // reduction scratch
  double *part_buf = nullptr, *gpart_buf = nullptr, *g2part_buf = nullptr, *red_out = nullptr;
  unsigned* cnt = nullptr;
  int gmax = 0, nvmax = 0;
  // GMRES workspace
  int ws_m = 0, ws_maxr = 0;
  double *V = nullptr, *x = nullptr, *b = nullptr, *tmp = nullptr;
  double *s = nullptr, *h_orig = nullptr, *h_rot = nullptr, *gv = nullptr, *cs = nullptr,
         *sn = nullptr, *h1 = nullptr, *coefA = nullptr, *coefB = nullptr, *tU = nullptr,
         *c = nullptr, *xc = nullptr, *cx = nullptr, *zl = nullptr;
  uint32_t *rec_restart = nullptr, *rec_step = nullptr;
  double *rec_mon = nullptr, *expl = nullptr;
  int ws_R1 = 0;
  GState* g = nullptr;
  GState* h_status = nullptr;  // pinned
  DState* h_dstate = nullptr;  // pinned copy of the running deflator's state (rank r)
  pgm_deflator* dummy = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // world > 1: halo planes move on hstream while the interior SpMV tiles run
  cudaStream_t hstream = nullptr;
  cudaEvent_t ev_halo_src = nullptr, ev_halo_done = nullptr;
  // multi-GPU: NCCL (one process per GPU) or an in-process loopback group
  void* nccl = nullptr;
  struct pgm_loopback* loop = nullptr;
  // deterministic mode (config.deterministic = PGM_DETERMINISTIC_PLANES):
  // every reduction = per-plane sequential partials + pairwise fold
  cudaStream_t cstream = nullptr;  // host -> device staging copies (matrix upload)
  void* hpin[2] = {nullptr, nullptr};  // pinned ring for pageable matrix sources
  size_t hpin_bytes = 0;
  cudaEvent_t ev_hdma[2] = {nullptr, nullptr};
  cudaEvent_t ev_copy[2] = {nullptr, nullptr}, ev_gath[2] = {nullptr, nullptr};
  bool det = false;
  int plane = 0, nplanes = 0, nplanes_global = 0, det_maxp = 0;
  std::vector<int> plane_off, plane_cnt;  // per rank (global plane order)
  double *det_pp = nullptr, *det_all = nullptr, *det_gbuf = nullptr;
  unsigned* det_cnt = nullptr;
  int det_nv = 0;
  pgm_deflator* cur_defl = nullptr;  // deflator of the running solve (halo of u)
  double* halo_ptr = nullptr;        // HV_PTR: ctx-layout view of a caller vector (Newton u)
  std::vector<pgm_matrix*> mats;     // live matrices (detached when the context dies first)
  // fused peer-memory allreduce (common.cuh peer_allreduce): one allocation
  // holding the window [2][world][PEER_NV] doubles + flags [2][world] + epoch
  bool peer = false;
  char* pbuf = nullptr;
  char** d_peer_base = nullptr;  // [world] window bases (char*) for the halo mailboxes
  double** d_peer_win = nullptr;
  unsigned long long** d_peer_flag = nullptr;
  std::vector<void*> peer_opened;  // IPC mappings to close
  // optional per-launch profiling (CUDA events around every hot-path kernel)
  bool prof_on = false;
  bool pdl = true;  // programmatic dependent launch of the hot-path kernels (PGMRES_PDL=0 disables)
  bool dcgs2 = true;  // delayed CGS2, one reduction per Arnoldi step (PGMRES_DCGS2=0: CGS2)
  bool dc_now = true;  // this solve runs DCGS2
  int prof_cycle = 0;
  struct Rec {
    uint32_t cls, cyc, k;
    cudaEvent_t a, b;
  };
  std::vector<Rec> prof;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
};

struct pgm_matrix {
  pgm_context* ctx = nullptr;
  uint32_t n = 0;
  uint64_t nnz = 0, stored = 0;
  int nslices = 0, ntiles = 0;
  unsigned long long* sptr = nullptr;
  unsigned* lane_len = nullptr;
  unsigned short* lane_row = nullptr;
  double* val = nullptr;
  unsigned* col = nullptr;
  unsigned short* col16 = nullptr;  // 16-bit column deltas (col freed when set)
  unsigned* lane_base = nullptr;
  unsigned* rp = nullptr;      // device CSR row_ptr (kept for value updates)
  // host-array transfers are staged through a bounded device buffer, a tile
  // range at a time (no resident nnz-sized staging copy)
  struct Chunk {
    int s0, count;                // slices
    unsigned long long lo, hi;    // CSR entries [lo, hi)
  };
  std::vector<Chunk> chunks;      // plan for host sources (built on first use)
  unsigned long long chunk_cap = 0;
  unsigned col_shift = 0;
  // tiles [0, t_lo_end) and [t_hi_begin, ntiles) read halo rows; the rest is
  // interior (world > 1: runs while the halo planes are in flight)
  int t_lo_end = 0, t_hi_begin = 0;
  Sell view() const {
    Sell S;
    S.sptr = sptr;
    S.lane_len = lane_len;
    S.lane_row = lane_row;
    S.val = val;
    S.col = col;
    S.col16 = col16;
    S.lane_base = lane_base;
    S.ntiles = ntiles;
    S.n = (int)n;
    return S;
  }
};

struct pgm_deflator {
  pgm_context* ctx = nullptr;
  pgm_deflation_config cfg{};
  int R1 = 0;
  DState* d = nullptr;
  double *U = nullptr, *AU = nullptr, *u = nullptr;
  double *T = nullptr, *Tinv = nullptr, *Q = nullptr, *proj = nullptr, *dwork = nullptr;
  int* iwork = nullptr;
  uint32_t *hist_restart = nullptr, *hist_r = nullptr;
  double *hist_mu = nullptr, *hist_theta = nullptr;
  int hist_cap = 0;
  bool dummy = false;
};

namespace {

pgm_status fail(pgm_context* ctx, const Status& s) {
  if (ctx) ctx->err = s.msg;
  g_tls_err = s.msg;
  return s.code;
}

// ---------------------------------------------------------------------------
// Launch geometry
template <class K>
int occupancy(K kernel, int threads, size_t smem) {
  int nb = 0;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem);
  return std::max(1, nb);
}

// Launch with programmatic stream serialization (PDL, common.cuh) when the
// context allows it; the kernel's griddepcontrol instructions order it.
template <class... KArgs, class... Args>
cudaError_t launch_pdl(pgm_context* ctx, void (*kernel)(KArgs...), int grid, int block,
                       size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (ctx->pdl && !ctx->prof_on) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

constexpr int MAX_BLOCKS_PER_SM = 8;  // bounds the grid-reduction tail
constexpr int MAX_SPLIT_BLOCKS_PER_SM = 32;  // warp-split CGS2 sweeps (64-128 threads)

// Kernel classes of the profile (pgm_context_profile).
enum ProfClass : uint32_t {
  PC_STEP_SPMV = 0, PC_SWEEP_B = 1, PC_SWEEP_C = 2, PC_XUPDATE = 3, PC_RITZ = 4,
  PC_PUSH = 5, PC_PUSH_SPMV = 6, PC_ROTATE = 7, PC_RESIDUAL = 8, PC_OTHER = 9,
  // world > 1: halo planes (NCCL send/recv or loopback copies; the reference's
  // "local" time) and the collective reduction + replicated finisher (its
  // "global" time; inside the reduction kernels on the peer transport)
  PC_HALO = 10, PC_ALLREDUCE = 11
};

cudaEvent_t prof_event(pgm_context* ctx) {
  if (ctx->ev_used == ctx->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->ev_pool.push_back(e);
  }
  return ctx->ev_pool[ctx->ev_used++];
}

struct ProfScope {
  pgm_context* ctx;
  cudaStream_t st;
  pgm_context::Rec rec{};
  ProfScope(pgm_context* c, uint32_t cls, uint32_t k, cudaStream_t s = nullptr)
      : ctx(c), st(s ? s : c->stream) {
    if (!ctx->prof_on) return;
    rec.cls = cls;
    rec.cyc = (uint32_t)ctx->prof_cycle;
    rec.k = k;
    rec.a = prof_event(ctx);
    rec.b = prof_event(ctx);
    cudaEventRecord(rec.a, st);
  }
  ~ProfScope() {
    if (!ctx->prof_on) return;
    cudaEventRecord(rec.b, st);
    ctx->prof.push_back(rec);
  }
};

template <class Epi>
uint32_t prof_class_of() {
  return PC_OTHER;
}
template <>
uint32_t prof_class_of<StepEpi>() {
  return PC_STEP_SPMV;
}
template <>
uint32_t prof_class_of<DStepEpi>() {
  return PC_STEP_SPMV;
}
template <>
uint32_t prof_class_of<ResidualEpi>() {
  return PC_RESIDUAL;
}
template <>
uint32_t prof_class_of<PushEpi>() {
  return PC_PUSH_SPMV;
}
template <int MODE>
uint32_t prof_class_sweep() {
  return MODE == SW_CGS2_B ? PC_SWEEP_B
       : MODE == SW_CGS2_C ? PC_SWEEP_C
       : MODE == SW_XUPDATE ? PC_XUPDATE
       : (MODE >= SW_PUSH1 && MODE <= SW_PUSH3) ? PC_PUSH : PC_OTHER;
}

size_t spmv_smem(int nv) { return sizeof(double) * spmv_smem_doubles(nv); }

// seg: 0 = every tile; 1 = interior tiles; 2 = halo-reading boundary tiles
// (1 and 2 together form one reduction over all tiles, world > 1; step SpMV only).
template <class Epi, bool SEG, bool C16>
Status launch_spmv_k(pgm_context* ctx, int G, size_t smem, const Sell& sv, const Params& P,
                     const Epi& E, const SpmvSeg& sg) {
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_spmv<Epi, SEG, C16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  CU(launch_pdl(ctx, k_spmv<Epi, SEG, C16>, G, SPMV_THREADS, smem, sv, P, E, sg));
  return {};
}

template <class Epi>
Status launch_spmv(pgm_context* ctx, const pgm_matrix* A, const Params& P, const Epi& E,
                   int nvmax, uint32_t prof_k = 0, int seg = 0) {
  const size_t smem = std::is_same<Epi, StepEpi>::value
                          ? sizeof(double) * spmv_step_smem_doubles(nvmax)
                          : std::is_same<Epi, DStepEpi>::value
                                ? sizeof(double) * (spmv_step_smem_doubles(nvmax) + TILE)
                                : spmv_smem(nvmax);
  Sell sv = A->view();
  SpmvSeg sg{0, 0, 0};
  int G = std::max(1, A->ntiles);
  if (seg == 1) {
    sg = SpmvSeg{A->t_lo_end, A->t_hi_begin - A->t_lo_end, 0};
    G = sg.len0;
  } else if (seg == 2) {
    sg = SpmvSeg{0, A->t_lo_end, A->t_hi_begin};
    G = A->t_lo_end + (A->ntiles - A->t_hi_begin);
  }
  if (G <= 0) return {};
  ProfScope ps(ctx, prof_class_of<Epi>(), prof_k);
  // one tile per block: the hardware scheduler balances the tiles
  const bool c16 = A->col16 != nullptr;
  if constexpr (std::is_same<Epi, StepEpi>::value || std::is_same<Epi, DStepEpi>::value) {
    if (seg != 0) {
      const Status st = c16 ? launch_spmv_k<Epi, true, true>(ctx, G, smem, sv, P, E, sg)
                            : launch_spmv_k<Epi, true, false>(ctx, G, smem, sv, P, E, sg);
      TRY(st);
      ctx->launches++;
      CU(cudaGetLastError());
      return {};
    }
  }
  const Status st = c16 ? launch_spmv_k<Epi, false, true>(ctx, G, smem, sv, P, E, sg)
                        : launch_spmv_k<Epi, false, false>(ctx, G, smem, sv, P, E, sg);
  TRY(st);
  ctx->launches++;
  CU(cudaGetLastError());
  return {};
}

template <int MODE, int NP>
Status launch_sweep_np(pgm_context* ctx, const Params& P, int k, int nv, int np) {
  const size_t smem = sizeof(double) * sweep_smem_doubles(nv, np);
  const int occ = std::min(MAX_BLOCKS_PER_SM, occupancy(k_sweep<MODE, NP>, SW_BLOCK, smem));
  const int nchunks = (int)((ctx->n + 31) / 32);
  const int G = std::max(1, std::min((nchunks + SW_WARPS - 1) / SW_WARPS, occ * ctx->nsm));
  ProfScope ps(ctx, prof_class_sweep<MODE>(), (uint32_t)k);
  k_sweep<MODE, NP><<<G, SW_BLOCK, smem, ctx->stream>>>(P, k);
  ctx->launches++;
  CU(cudaGetLastError());
  return {};
}

// CGS2 sweeps (np = k + 1): warp-split kernels; 4 warps per block (8 above
// 64 vectors), 2 rows per lane (tools/sweepbench.cu, tools/run_variants.sh).
template <int MODE, int NW, int RPL, int NUW, int NPW>
Status launch_cgs2_cfg(pgm_context* ctx, const Params& P, int k) {
  static int occ = 0;  // per instantiation; same device geometry for every context
  if (occ == 0)
    occ = std::min(MAX_SPLIT_BLOCKS_PER_SM, occupancy(k_cgs2<MODE, NW, RPL, NUW, NPW>, NW * 32, 0));
  const int nchunks = (int)((ctx->n + 32 * RPL - 1) / (32 * RPL));
  const int G = std::max(1, std::min(nchunks, occ * ctx->nsm));
  ProfScope ps(ctx, prof_class_sweep<MODE>(), (uint32_t)k);
  CU(launch_pdl(ctx, k_cgs2<MODE, NW, RPL, NUW, NPW>, G, NW * 32, 0, P, k));
  ctx->launches++;
  CU(cudaGetLastError());
  return {};
}

template <int MODE, int NW, int RPL, int NUW, int... Is>
Status launch_cgs2_table(pgm_context* ctx, const Params& P, int k, int npw,
                         std::integer_sequence<int, Is...>) {
  using Fn = Status (*)(pgm_context*, const Params&, int);
  static constexpr Fn table[] = {&launch_cgs2_cfg<MODE, NW, RPL, NUW, Is + 1>...};
  return table[npw - 1](ctx, P, k);
}

constexpr int CGS2_SPLIT_MAX = 112;  // = MAX_M: 8 warps x 14 vectors

#ifndef PGM_CGS2_RPL
#define PGM_CGS2_RPL 2  // rows per lane (tools/run_variants.sh study: 2 beats 1)
#endif
Status launch_dcgs2_update(pgm_context* ctx, const Params& P, int k) {
  static int occ = 0;
  if (occ == 0) occ = std::min(MAX_BLOCKS_PER_SM, occupancy(k_dcgs2_update, UPD_BLOCK, 0));
  const int nchunks = (int)((ctx->n + 63) / 64);
  const int G = std::max(1, std::min((nchunks + UPD_BLOCK / 32 - 1) / (UPD_BLOCK / 32),
                                     occ * ctx->nsm));
  ProfScope ps(ctx, PC_SWEEP_C, (uint32_t)k);
  CU(launch_pdl(ctx, k_dcgs2_update, G, UPD_BLOCK, 0, P, k));
  ctx->launches++;
  CU(cudaGetLastError());
  return {};
}

Status launch_cgs2_update(pgm_context* ctx, const Params& P, int k) {
  static int occ = 0;
  if (occ == 0) occ = std::min(MAX_BLOCKS_PER_SM, occupancy(k_cgs2_update, UPD_BLOCK, 0));
  const int nchunks = (int)((ctx->n + 63) / 64);
  const int G = std::max(1, std::min((nchunks + UPD_BLOCK / 32 - 1) / (UPD_BLOCK / 32),
                                     occ * ctx->nsm));
  ProfScope ps(ctx, PC_SWEEP_C, (uint32_t)k);
  CU(launch_pdl(ctx, k_cgs2_update, G, UPD_BLOCK, 0, P, k));
  ctx->launches++;
  CU(cudaGetLastError());
  return {};
}

// NUW (deflation vectors per warp) is chosen from the deflator's current rank
// r (constant within a cycle; read with the restart status word), so early
// cycles with a small basis do not pay registers for U.
template <int NW, int R, int NUW, int NPWMAX>
Status launch_cgs2_nuw(pgm_context* ctx, const Params& P, int k, int npw) {
  return launch_cgs2_table<SW_CGS2_B, NW, R, NUW>(ctx, P, k, npw,
                                                  std::make_integer_sequence<int, NPWMAX>{});
}

template <int NW, int R, int NPWMAX>
Status launch_cgs2_r(pgm_context* ctx, const Params& P, int k, int npw, int r) {
  const int nuw = (r + NW - 1) / NW;
  if (nuw == 0) return launch_cgs2_nuw<NW, R, 0, NPWMAX>(ctx, P, k, npw);
  if (nuw <= 1) return launch_cgs2_nuw<NW, R, 1, NPWMAX>(ctx, P, k, npw);
  if (nuw <= 2) return launch_cgs2_nuw<NW, R, 2, NPWMAX>(ctx, P, k, npw);
  if (nuw <= 4) return launch_cgs2_nuw<NW, R, 4, NPWMAX>(ctx, P, k, npw);
  if constexpr (NW == 4) {
    if (nuw <= 6) return launch_cgs2_nuw<NW, R, 6, NPWMAX>(ctx, P, k, npw);
  }
  return launch_cgs2_nuw<NW, R, (MAX_R1 + NW - 1) / NW, NPWMAX>(ctx, P, k, npw);
}

Status launch_cgs2_b(pgm_context* ctx, const Params& P, int k, int nv, int r) {
  constexpr int R = PGM_CGS2_RPL;
  const int np = k + 1;
#ifndef PGM_B_NW
#define PGM_B_NW 4
#endif
  constexpr int BNW = PGM_B_NW;
  if (np <= 64) return launch_cgs2_r<BNW, R, (64 + BNW - 1) / BNW>(ctx, P, k, (np + BNW - 1) / BNW, r);
  if (np <= CGS2_SPLIT_MAX) return launch_cgs2_r<8, R, 14>(ctx, P, k, (np + 7) / 8, r);
  return launch_sweep_np<SW_CGS2_B, 0>(ctx, P, k, nv, np);
}

// np / nv: upper bounds of the register-streamed set and of the reduced values;
// np picks the register-resident template (0 = generic path for np > 64).
template <int MODE>
Status launch_sweep(pgm_context* ctx, const Params& P, int k, int np, int /*np2*/, int nv, bool) {
  // register-resident vector set up to NPMAX; above it the 16-wide generic
  // loop (measured at cfg3: the push_vector sweeps are faster generic, the x
  // update register-resident)
  constexpr int NPMAX = MODE == SW_XUPDATE ? 64 : 16;
  if (np <= 8) return launch_sweep_np<MODE, 8>(ctx, P, k, nv, np);
  if (np <= 16) return launch_sweep_np<MODE, 16>(ctx, P, k, nv, np);
  if constexpr (NPMAX >= 64) {
    if (np <= 32) return launch_sweep_np<MODE, 32>(ctx, P, k, nv, np);
    if (np <= 64) return launch_sweep_np<MODE, 64>(ctx, P, k, nv, np);
  }
  return launch_sweep_np<MODE, 0>(ctx, P, k, nv, np);
}

// ---------------------------------------------------------------------------
// Context-owned buffers

Status ensure_reduction(pgm_context* ctx, int nv, int gneed = 0) {
  const int gmax = std::max(ctx->nsm * MAX_SPLIT_BLOCKS_PER_SM, gneed);
  if (ctx->part_buf && ctx->nvmax >= nv && ctx->gmax >= gmax) return {};
  dfree(ctx->part_buf);
  dfree(ctx->gpart_buf);
  dfree(ctx->g2part_buf);
  dfree(ctx->cnt);
  dfree(ctx->red_out);
  ctx->nvmax = std::max(nv, 2 * MAX_R1 + MAX_M + 8);
  ctx->gmax = gmax;
  const int ng = (gmax + GROUP - 1) / GROUP;
  const int ns = (ng + GROUP - 1) / GROUP;
  TRY(dalloc(&ctx->part_buf, (size_t)ctx->nvmax * gmax));
  TRY(dalloc(&ctx->gpart_buf, (size_t)ctx->nvmax * ng));
  TRY(dalloc(&ctx->g2part_buf, (size_t)ctx->nvmax * ns));
  // counters: [0] final, [1, 1 + ng) groups, [1 + ng, 1 + ng + ns) super-groups
  // (a reduction with NG groups uses [1 + NG, ...): sized for the largest)
  TRY(dalloc(&ctx->cnt, (size_t)ng + 1 + ns));
  TRY(dalloc(&ctx->red_out, (size_t)ctx->nvmax));
  CU(cudaMemset(ctx->cnt, 0, sizeof(unsigned) * (ng + 1 + ns)));
  if (ctx->det) {
    dfree(ctx->det_pp);
    dfree(ctx->det_all);
    dfree(ctx->det_gbuf);
    dfree(ctx->det_cnt);
    TRY(dalloc(&ctx->det_pp, (size_t)ctx->nvmax * std::max(1, ctx->det_maxp)));
    TRY(dalloc(&ctx->det_all, (size_t)ctx->nvmax * std::max(1, ctx->nplanes_global)));
    if (ctx->world > 1 && !ctx->loop)
      TRY(dalloc(&ctx->det_gbuf, (size_t)ctx->world * ctx->nvmax * std::max(1, ctx->det_maxp)));
    TRY(dalloc(&ctx->det_cnt, 1));
    CU(cudaMemset(ctx->det_cnt, 0, sizeof(unsigned)));
  }
  return {};
}

void free_workspace(pgm_context* ctx) {
  dfree(ctx->V);
  dfree(ctx->s);
  dfree(ctx->h_orig);
  dfree(ctx->h_rot);
  dfree(ctx->gv);
  dfree(ctx->cs);
  dfree(ctx->sn);
  dfree(ctx->h1);
  dfree(ctx->coefA);
  dfree(ctx->coefB);
  dfree(ctx->tU);
  dfree(ctx->c);
  dfree(ctx->xc);
  dfree(ctx->cx);
  dfree(ctx->zl);
  dfree(ctx->rec_restart);
  dfree(ctx->rec_step);
  dfree(ctx->rec_mon);
  dfree(ctx->expl);
  ctx->ws_m = ctx->ws_maxr = ctx->ws_R1 = 0;
}

Status ensure_workspace(pgm_context* ctx, int m, int max_restarts, int R1) {
  if (ctx->V && ctx->ws_m == m && ctx->ws_maxr >= max_restarts && ctx->ws_R1 >= R1) return {};
  free_workspace(ctx);
  const size_t ld = ctx->ld;
  TRY(dalloc(&ctx->V, (size_t)(m + 1) * ld));
  CU(cudaMemset(ctx->V, 0, sizeof(double) * (m + 1) * ld));
  const size_t hm = (size_t)(m + 1) * m;
  TRY(dalloc(&ctx->s, m + 2));
  TRY(dalloc(&ctx->h_orig, hm));
  TRY(dalloc(&ctx->h_rot, hm));
  CU(cudaMemset(ctx->h_orig, 0, sizeof(double) * hm));
  CU(cudaMemset(ctx->h_rot, 0, sizeof(double) * hm));
  TRY(dalloc(&ctx->gv, m + 2));
  TRY(dalloc(&ctx->cs, m + 1));
  TRY(dalloc(&ctx->sn, m + 1));
  TRY(dalloc(&ctx->h1, m + 2));
  TRY(dalloc(&ctx->coefA, m + 2));
  TRY(dalloc(&ctx->coefB, m + 2));
  TRY(dalloc(&ctx->tU, (size_t)(m + 2) * R1));
  TRY(dalloc(&ctx->c, R1 + 1));
  TRY(dalloc(&ctx->xc, m + 2));
  TRY(dalloc(&ctx->cx, R1 + 1));
  TRY(dalloc(&ctx->zl, m + 2));
  const size_t cap = (size_t)std::max(1, max_restarts) * m;
  TRY(dalloc(&ctx->rec_restart, cap));
  TRY(dalloc(&ctx->rec_step, cap));
  TRY(dalloc(&ctx->rec_mon, cap));
  TRY(dalloc(&ctx->expl, std::max(1, max_restarts)));
  ctx->ws_m = m;
  ctx->ws_maxr = max_restarts;
  ctx->ws_R1 = R1;
  return {};
}

Status defl_alloc_vectors(pgm_deflator* d) {
  if (d->U) return {};
  pgm_context* ctx = d->ctx;
  const size_t ld = ctx->ld;
  const int R1 = d->dummy ? 1 : d->R1;
  TRY(dalloc(&d->U, (size_t)R1 * ld));
  TRY(dalloc(&d->AU, (size_t)R1 * ld));
  TRY(dalloc(&d->u, ld));
  CU(cudaMemset(d->U, 0, sizeof(double) * R1 * ld));
  CU(cudaMemset(d->AU, 0, sizeof(double) * R1 * ld));
  CU(cudaMemset(d->u, 0, sizeof(double) * ld));
  return {};
}

Status defl_ensure_hist(pgm_deflator* d, int need) {
  if (need <= d->hist_cap) return {};
  int cap = std::max(need, 2 * d->hist_cap + 64);
  uint32_t *hr = nullptr, *hrr = nullptr;
  double *hm = nullptr, *ht = nullptr;
  TRY(dalloc(&hr, cap));
  TRY(dalloc(&hrr, cap));
  TRY(dalloc(&hm, cap));
  TRY(dalloc(&ht, cap));
  DState hs;
  CU(cudaMemcpy(&hs, d->d, sizeof(DState), cudaMemcpyDeviceToHost));
  const int keep = std::min(hs.n_hist, d->hist_cap);
  if (keep > 0) {
    CU(cudaMemcpy(hr, d->hist_restart, 4 * keep, cudaMemcpyDeviceToDevice));
    CU(cudaMemcpy(hrr, d->hist_r, 4 * keep, cudaMemcpyDeviceToDevice));
    CU(cudaMemcpy(hm, d->hist_mu, 8 * keep, cudaMemcpyDeviceToDevice));
    CU(cudaMemcpy(ht, d->hist_theta, 8 * keep, cudaMemcpyDeviceToDevice));
  }
  dfree(d->hist_restart);
  dfree(d->hist_r);
  dfree(d->hist_mu);
  dfree(d->hist_theta);
  d->hist_restart = hr;
  d->hist_r = hrr;
  d->hist_mu = hm;
  d->hist_theta = ht;
  d->hist_cap = cap;
  hs.hist_cap = cap;
  CU(cudaMemcpy(&d->d->hist_cap, &cap, sizeof(int), cudaMemcpyHostToDevice));
  return {};
}

size_t peer_win_bytes(const pgm_context* ctx) {
  return sizeof(double) * 2 * (size_t)ctx->world * PEER_NV;
}
// halo mailboxes after the reduction window + flags: [2 par][2 dir][hmax]
// doubles, then flags [2 par][2 dir], the halo epoch and the push counter
size_t peer_halo_rows(const pgm_context* ctx) {
  return std::max<size_t>(std::max(ctx->lo, ctx->hi), 1);
}
size_t peer_mb_offset(const pgm_context* ctx) {
  return round_up(peer_win_bytes(ctx) + sizeof(unsigned long long) * (2 * (size_t)ctx->world + 2),
                  256);
}
size_t peer_hf_offset(const pgm_context* ctx) {
  return peer_mb_offset(ctx) + sizeof(double) * 4 * peer_halo_rows(ctx);
}
size_t peer_buf_bytes(const pgm_context* ctx) {
  return peer_hf_offset(ctx) + sizeof(unsigned long long) * 8;
}

// Peer-pointer tables: wins[q] / flags[q] = rank q's window and flags as
// addressable from this rank.
Status peer_set_tables(pgm_context* ctx, const std::vector<char*>& bufs) {
  const int W = ctx->world;
  std::vector<double*> w(W);
  std::vector<unsigned long long*> f(W);
  for (int q = 0; q < W; ++q) {
    w[q] = reinterpret_cast<double*>(bufs[q]);
    f[q] = reinterpret_cast<unsigned long long*>(bufs[q] + peer_win_bytes(ctx));
  }
  if (!ctx->d_peer_win) TRY(dalloc(&ctx->d_peer_win, W));
  if (!ctx->d_peer_flag) TRY(dalloc(&ctx->d_peer_flag, W));
  if (!ctx->d_peer_base) TRY(dalloc(&ctx->d_peer_base, W));
  CU(cudaMemcpy(ctx->d_peer_win, w.data(), sizeof(double*) * W, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(ctx->d_peer_flag, f.data(), sizeof(void*) * W, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(ctx->d_peer_base, bufs.data(), sizeof(char*) * W, cudaMemcpyHostToDevice));
  ctx->peer = true;
  return {};
}

Params make_params(pgm_context* ctx, pgm_deflator* d) {
  Params P{};
  P.g = ctx->g;
  P.d = d->d;
  P.s = ctx->s;
  P.h_orig = ctx->h_orig;
  P.h_rot = ctx->h_rot;
  P.gv = ctx->gv;
  P.cs = ctx->cs;
  P.sn = ctx->sn;
  P.h1 = ctx->h1;
  P.coefA = ctx->coefA;
  P.coefB = ctx->coefB;
  P.tU = ctx->tU;
  P.c = ctx->c;
  P.xc = ctx->xc;
  P.cx = ctx->cx;
  P.zl = ctx->zl;
  P.rec_restart = ctx->rec_restart;
  P.rec_step = ctx->rec_step;
  P.rec_mon = ctx->rec_mon;
  P.expl = ctx->expl;
  P.T = d->T;
  P.Tinv = d->Tinv;
  P.Q = d->Q;
  P.proj = d->proj;
  P.dwork = d->dwork;
  P.iwork = d->iwork;
  P.hist_restart = d->hist_restart;
  P.hist_r = d->hist_r;
  P.hist_mu = d->hist_mu;
  P.hist_theta = d->hist_theta;
  P.V = ctx->V;
  P.U = d->U;
  P.AU = d->AU;
  P.x = ctx->x;
  P.b = ctx->b;
  P.u = d->u;
  P.ld = ctx->ld;
  P.n = (int)ctx->n;
  P.lo = (int)ctx->lo;
  P.m = ctx->ws_m;
  P.R1 = d->R1;
  P.part = ctx->part_buf;
  P.gpart = ctx->gpart_buf;
  P.g2part = ctx->g2part_buf;
  P.det = ctx->det ? 1 : 0;
  P.plane = ctx->plane;
  P.nplanes = ctx->nplanes;
  P.det_pp = ctx->det_pp;
  P.det_all = ctx->det_all;
  P.nplanes_global = ctx->nplanes_global;
  P.det_cnt = ctx->det_cnt;
  P.cnt = ctx->cnt;
  P.red_out = ctx->red_out;
  P.world = ctx->coll ? std::max(ctx->world, 2) : 1;
  P.peer = ctx->peer ? 1 : 0;
  P.rank = ctx->rank;
  P.peer_win = ctx->d_peer_win;
  P.peer_flag = ctx->d_peer_flag;
  if (ctx->pbuf) {
    P.win_local = reinterpret_cast<const double*>(ctx->pbuf);
    P.flag_local = reinterpret_cast<const unsigned long long*>(ctx->pbuf + peer_win_bytes(ctx));
    P.epoch = reinterpret_cast<unsigned long long*>(ctx->pbuf + peer_win_bytes(ctx)) +
              2 * ctx->world;
  }
  return P;
}

// Small-state workspace for the standalone deflator entry points.
Status ensure_min_workspace(pgm_context* ctx, int R1) {
  if (ctx->V && ctx->ws_R1 >= R1) return {};
  return ensure_workspace(ctx, std::max(1, ctx->ws_m), std::max(1, ctx->ws_maxr),
                          std::max(R1, ctx->ws_R1));
}

Status set_gstate_idle(pgm_context* ctx) {
  GState gs{};
  gs.harvest = 0;
  CU(cudaMemcpyAsync(ctx->g, &gs, sizeof(GState), cudaMemcpyHostToDevice, ctx->stream));
  return {};
}

// ---------------------------------------------------------------------------
// Multi-GPU collectives (world > 1): allreduce of the block-reduced sums,
// then the scalar finisher on every rank.
enum HaloKind { HV_V = 0, HV_X = 1, HV_U = 2, HV_TMP = 3, HV_PTR = 4 };
Status allreduce_red(pgm_context* ctx, int nv);
Status halo_exchange(pgm_context* ctx, HaloKind kind, int slot = 0, cudaStream_t st = nullptr);

// Deterministic mode: gather every rank's plane partials ([v][planes of the
// rank], nv rows) into det_all ([v][global plane]) on every rank.
Status det_gather(pgm_context* ctx, int nv) {
  const int npg = ctx->nplanes_global;
  if (ctx->loop) {
    pgm_loopback* L = ctx->loop;
    CU(cudaStreamSynchronize(ctx->stream));
    L->barrier();  // every rank's k_det_dots has finished
    for (int q = 0; q < ctx->world; ++q) {
      const pgm_context* o = L->ctx[q];
      if (ctx->plane_cnt[q] == 0) continue;
      CU(cudaMemcpy2DAsync(ctx->det_all + ctx->plane_off[q], 8 * (size_t)npg, o->det_pp,
                           8 * (size_t)ctx->plane_cnt[q], 8 * (size_t)ctx->plane_cnt[q], nv,
                           cudaMemcpyDeviceToDevice, ctx->stream));
    }
    CU(cudaStreamSynchronize(ctx->stream));
    L->barrier();  // nobody overwrites its partials before all have copied them
    return {};
  }
  // NCCL: every rank contributes nv x det_maxp (its planes, padded)
  const size_t per = (size_t)nv * ctx->det_maxp;
  {
    // pack [v][nplanes] -> [v][det_maxp] (columns beyond nplanes unused)
    CU(cudaMemcpy2DAsync(ctx->det_gbuf + (size_t)ctx->rank * per, 8 * (size_t)ctx->det_maxp,
                         ctx->det_pp, 8 * (size_t)ctx->nplanes, 8 * (size_t)ctx->nplanes, nv,
                         cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (nccl_lite::allgather_f64(ctx->det_gbuf + (size_t)ctx->rank * per, ctx->det_gbuf, per,
                               ctx->nccl, ctx->stream) != 0)
    return Status{PGM_ENCCL, "ncclAllGather (deterministic plane partials) failed"};
  for (int q = 0; q < ctx->world; ++q) {
    if (ctx->plane_cnt[q] == 0) continue;
    CU(cudaMemcpy2DAsync(ctx->det_all + ctx->plane_off[q], 8 * (size_t)npg,
                         ctx->det_gbuf + (size_t)q * per, 8 * (size_t)ctx->det_maxp,
                         8 * (size_t)ctx->plane_cnt[q], nv, cudaMemcpyDeviceToDevice,
                         ctx->stream));
  }
  return {};
}

template <int KIND>
Status finish_global(pgm_context* ctx, const Params& P, int k, int nv) {
  if (ctx->det) {
    // the reduction kernel skipped its tail (P.det): recompute the values as
    // per-plane sequential partials + pairwise fold, then finish
    if (nv <= 0 || nv > ctx->nvmax) return Status{PGM_ESTATE, "finish_global: bad reduction size"};
    const long threads = (long)std::max(1, ctx->nplanes) * nv;
    const int G = (int)((threads + DET_THREADS - 1) / DET_THREADS);
    {
      ProfScope ps(ctx, PC_ALLREDUCE, (uint32_t)k);
      k_det_dots<KIND><<<G, DET_THREADS, 0, ctx->stream>>>(P, k);
      ctx->launches++;
      CU(cudaGetLastError());
      if (ctx->world > 1) {
        TRY(det_gather(ctx, nv));
        k_det_finish<KIND><<<1, DET_THREADS, 0, ctx->stream>>>(P, k);
        ctx->launches++;
        CU(cudaGetLastError());
      }
    }
    return {};
  }
  if (!ctx->coll || ctx->peer) return {};  // peer mode: all-reduced inside the kernel
  if (nv <= 0 || nv > ctx->nvmax) return Status{PGM_ESTATE, "finish_global: bad reduction size"};
  ProfScope ps(ctx, PC_ALLREDUCE, (uint32_t)k);
  TRY(allreduce_red(ctx, nv));
  k_finish<KIND><<<1, 32, 0, ctx->stream>>>(P, k);
  ctx->launches++;
  CU(cudaGetLastError());
  return {};
}

// One restart cycle of the solve: m Arnoldi steps (3 fused kernels each), the
// x update, the deflation harvest and the explicit residual.
Status enqueue_residual(pgm_context* ctx, pgm_matrix* A, pgm_deflator* d, const Params& P) {
  if (ctx->world > 1) TRY(halo_exchange(ctx, HV_X));
  TRY(launch_spmv(ctx, A, P, ResidualEpi{0}, d->R1 + 1));
  TRY(finish_global<101>(ctx, P, 0, d->R1 + 1));
  return {};
}

Status enqueue_cycle(pgm_context* ctx, pgm_matrix* A, pgm_deflator* d, const Params& P,
                     bool harvest, bool residual = true) {
  const int m = ctx->ws_m;
  const int R1 = d->R1;
  const bool overlap = ctx->world > 1 && A->t_hi_begin > A->t_lo_end;
  if (ctx->dc_now) {
    // delayed CGS2: SpMV (+ the step's one reduction) and one update per step,
    // the cycle closes with a dots-only pass for column m-1
    for (int k = 0; k < m; ++k) {
      DStepEpi se{k};
      if (overlap) {
        // halo planes of W_k (= u_k) on hstream while the interior tiles run
        CU(cudaEventRecord(ctx->ev_halo_src, ctx->stream));
        CU(cudaStreamWaitEvent(ctx->hstream, ctx->ev_halo_src, 0));
        TRY(halo_exchange(ctx, HV_V, k, ctx->hstream));
        CU(cudaEventRecord(ctx->ev_halo_done, ctx->hstream));
        TRY(launch_spmv(ctx, A, P, se, 2 * m + 2 + R1, (uint32_t)k, 1));
        CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo_done, 0));
        TRY(launch_spmv(ctx, A, P, se, 2 * m + 2 + R1, (uint32_t)k, 2));
      } else {
        if (ctx->world > 1) TRY(halo_exchange(ctx, HV_V, k));
        TRY(launch_spmv(ctx, A, P, se, 2 * m + 2 + R1, (uint32_t)k));
      }
      TRY(finish_global<103>(ctx, P, k, std::max(k, 1) + k + 2 + R1));
      TRY(launch_dcgs2_update(ctx, P, k));
    }
    {
      const int nt = (int)((ctx->n + TILE - 1) / TILE);
      const size_t smem = sizeof(double) * ((size_t)TILE + 2 * (m + 1) + 2);
      ProfScope ps(ctx, PC_OTHER, (uint32_t)m);
      CU(launch_pdl(ctx, k_dclose, nt, SPMV_THREADS, smem, P, nt));
      ctx->launches++;
      CU(cudaGetLastError());
    }
    TRY(finish_global<SW_DCLOSE>(ctx, P, m, m + 1));
  }
  for (int k = 0; k < (ctx->dc_now ? 0 : m); ++k) {
    if (overlap) {
      // halo planes of W_k on hstream (NVLink P2P through NCCL send/recv)
      // while the interior tiles run; then the boundary tiles.  NCCL calls
      // stay totally ordered: the halo completes before the next allreduce
      // is enqueued behind the boundary tiles.
      CU(cudaEventRecord(ctx->ev_halo_src, ctx->stream));
      CU(cudaStreamWaitEvent(ctx->hstream, ctx->ev_halo_src, 0));
      TRY(halo_exchange(ctx, HV_V, k, ctx->hstream));
      CU(cudaEventRecord(ctx->ev_halo_done, ctx->hstream));
      StepEpi se{k};
      TRY(launch_spmv(ctx, A, P, se, m + 1, (uint32_t)k, 1));
      CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo_done, 0));
      TRY(launch_spmv(ctx, A, P, se, m + 1, (uint32_t)k, 2));
      TRY(finish_global<100>(ctx, P, k, k + 1));
      TRY(launch_cgs2_b(ctx, P, k, k + 2 + R1, ctx->cur_defl ? ctx->h_dstate->r : R1));
      TRY(finish_global<SW_CGS2_B>(ctx, P, k, k + 2 + R1));
      TRY(launch_cgs2_update(ctx, P, k));
      continue;
    }
    if (ctx->world > 1) TRY(halo_exchange(ctx, HV_V, k));
    // (alternating the walk direction kernel to kernel, to reuse the previous
    // kernel's L2 tail, measured slower on B200: all kernels walk forward)
    StepEpi se{k};
    TRY(launch_spmv(ctx, A, P, se, m + 1, (uint32_t)k));
    TRY(finish_global<100>(ctx, P, k, k + 1));
    TRY(launch_cgs2_b(ctx, P, k, k + 2 + R1, ctx->cur_defl ? ctx->h_dstate->r : R1));
    TRY(finish_global<SW_CGS2_B>(ctx, P, k, k + 2 + R1));
    TRY(launch_cgs2_update(ctx, P, k));
  }
  {
    const size_t esmem = sizeof(double) * ((size_t)m * m + m + MAX_R1);
    if (esmem > 48 * 1024)
      CU(cudaFuncSetAttribute(k_end_cycle, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esmem));
    ProfScope ps(ctx, PC_OTHER, 0);
    k_end_cycle<<<1, 256, esmem, ctx->stream>>>(P);
    ctx->launches++;
    CU(cudaGetLastError());
  }
  {
    ProfScope ps(ctx, PC_XUPDATE, 0);
    const int occ = std::min(MAX_BLOCKS_PER_SM, occupancy(k_xupdate, XU_BLOCK, 0));
    const int nch = (int)((ctx->n + 63) / 64);
    const int G = std::max(1, std::min((nch + XU_BLOCK / 32 - 1) / (XU_BLOCK / 32), occ * ctx->nsm));
    k_xupdate<<<G, XU_BLOCK, 0, ctx->stream>>>(P);
    ctx->launches++;
    CU(cudaGetLastError());
  }
  if (harvest) {
    // [H | H^-1] + 4 vectors, plus a copy of H for the matvecs when it fits
    const int hcopy = sizeof(double) * (3 * (size_t)m * m + 4 * m) <= 227 * 1024 ? 1 : 0;
    const size_t rsmem = sizeof(double) * ((2 + hcopy) * (size_t)m * m + 4 * m);
    if (rsmem > 48 * 1024)
      CU(cudaFuncSetAttribute(k_ritz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem));
    {
      ProfScope ps(ctx, PC_RITZ, 0);
      // CTA 0: Gauss-Jordan + inverse iteration; CTA 1: power iteration
      k_ritz<<<2, RITZ_THREADS, rsmem, ctx->stream>>>(P, hcopy);
    }
    ctx->launches++;
    CU(cudaGetLastError());
    TRY(launch_sweep<SW_PUSH1>(ctx, P, 1, m, 0, R1 + 1, false));
    TRY(finish_global<SW_PUSH1>(ctx, P, 1, R1 + 1));
    TRY(launch_sweep<SW_PUSH2>(ctx, P, 0, R1, 0, R1, true));
    TRY(finish_global<SW_PUSH2>(ctx, P, 0, R1));
    TRY(launch_sweep<SW_PUSH3>(ctx, P, 0, R1, 0, 1, false));
    TRY(finish_global<SW_PUSH3>(ctx, P, 0, 1));
    if (ctx->world > 1) TRY(halo_exchange(ctx, HV_U));
    TRY(launch_spmv(ctx, A, P, PushEpi{}, 2 * R1 + 1));
    TRY(finish_global<102>(ctx, P, 0, 2 * R1 + 1));
    {
      ProfScope ps(ctx, PC_ROTATE, 0);
      k_rotate<true><<<ctx->nsm * 4, 256, 0, ctx->stream>>>(P);
    }
    ctx->launches++;
    CU(cudaGetLastError());
  }
  if (residual) TRY(enqueue_residual(ctx, A, d, P));
  return {};
}

// Restart observer: the cycle (x update + harvest) has been enqueued; wait for
// it and hand the host the restart index and step count.  The basis and H stay
// readable (pgm_restart_basis / pgm_restart_hessenberg) until the callback
// returns; the explicit residual (which reuses W_0) is enqueued afterwards.
Status observe_restart(pgm_context* ctx) {
  CU(cudaStreamSynchronize(ctx->stream));
  GState gs;
  CU(cudaMemcpy(&gs, ctx->g, sizeof(GState), cudaMemcpyDeviceToHost));
  if (gs.error) return {};
  ctx->in_obs = true;
  ctx->obs_steps = gs.steps;
  const int rc = ctx->obs(ctx->obs_user, (uint32_t)gs.restart, (uint32_t)gs.steps);
  ctx->in_obs = false;
  if (rc != 0) return Status{PGM_ESTATE, "restart observer requested the solve to stop"};
  return {};
}

Status read_status(pgm_context* ctx) {
  if (ctx->cur_defl)
    CU(cudaMemcpyAsync(ctx->h_dstate, ctx->cur_defl->d, sizeof(DState), cudaMemcpyDeviceToHost,
                       ctx->stream));
  CU(cudaMemcpyAsync(ctx->h_status, ctx->g, sizeof(GState), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return {};
}

Status error_of(const GState& gs) {
  switch (gs.error) {
    case 0:
      return {};
    case 2:
      if (gs.err_restart < 0) return Status{PGM_ENONFINITE, "gmres: initial residual is not finite"};
      if (gs.err_step < 0)
        return Status{PGM_ENONFINITE, "gmres: non-finite residual after restart " +
                                          std::to_string(gs.err_restart)};
      return Status{PGM_ENONFINITE, "gmres: non-finite Arnoldi coefficient at restart " +
                                        std::to_string(gs.err_restart) + ", step " +
                                        std::to_string(gs.err_step)};
    case 3:
      return Status{PGM_ESINGULAR, "gmres: singular projection in least squares"};
    default:
      return Status{(pgm_status)gs.error, "device error"};
  }
}

Status copy_in(pgm_context* ctx, double* dst_own, const double* src, size_t n, int32_t flags) {
  CU(cudaMemcpyAsync(dst_own, src, n * sizeof(double),
                     (flags & PGM_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     ctx->stream));
  return {};
}
Status copy_out(pgm_context* ctx, double* dst, const double* src_own, size_t n, int32_t flags) {
  CU(cudaMemcpyAsync(dst, src_own, n * sizeof(double),
                     (flags & PGM_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                     ctx->stream));
  return {};
}

#ifndef PGM_L2WIN
#define PGM_L2WIN 1
#endif
// L2 persistence for the small dense solver state the finishers and the SpMV
// prologues chase every step (Hessenberg, rotations, scales, coefficients,
// U^T V, T^-1, the status words): written by one step's finisher and read by
// the next, they would otherwise be evicted by the basis / matrix streams in
// between (18 GB per step at config 3).  One access-policy window over the
// span of these allocations when it is compact (<= 4 MB).
void set_l2_window(pgm_context* ctx, pgm_deflator* d) {
  if (!PGM_L2WIN) return;
  if (const char* e = std::getenv("PGMRES_L2WIN"))
    if (e[0] == '0') return;
  const size_t m = (size_t)ctx->ws_m, R1 = (size_t)std::max(d->R1, 1);
  const std::pair<const void*, size_t> r[] = {
      {ctx->s, 8 * (m + 2)},          {ctx->h_orig, 8 * (m + 1) * m}, {ctx->h_rot, 8 * (m + 1) * m},
      {ctx->gv, 8 * (m + 2)},         {ctx->cs, 8 * (m + 1)},         {ctx->sn, 8 * (m + 1)},
      {ctx->coefA, 8 * (m + 2)},      {ctx->coefB, 8 * (m + 2)},      {ctx->tU, 8 * (m + 2) * R1},
      {ctx->c, 8 * (R1 + 1)},         {ctx->g, sizeof(GState)},       {d->d, sizeof(DState)},
      {d->Tinv, 8 * R1 * R1},         {ctx->cnt, 64}};
  uintptr_t lo = UINTPTR_MAX, hi = 0;
  for (const auto& e : r) {
    if (!e.first) continue;
    lo = std::min(lo, (uintptr_t)e.first);
    hi = std::max(hi, (uintptr_t)e.first + e.second);
  }
  if (hi <= lo || hi - lo > ((size_t)4 << 20)) return;
  static bool limit = false;
  if (!limit) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)4 << 20);
    limit = true;
  }
  cudaStreamAttrValue v{};
  v.accessPolicyWindow.base_ptr = (void*)lo;
  v.accessPolicyWindow.num_bytes = hi - lo;
  v.accessPolicyWindow.hitRatio = 1.0f;
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &v);
  cudaGetLastError();  // best effort
}

Status solve_impl(pgm_context* ctx, pgm_matrix* A, pgm_deflator* dflt, const double* b, double* x,
                  const pgm_gmres_config* cfg, int32_t flags, pgm_report* rep) {
  if (!cfg) return einval("pgm_solve: null config");
  if (cfg->m == 0) return einval("GmresWorkspace: m must be positive");
  if (ctx->world > 1 && !ctx->loop && !ctx->nccl && !ctx->peer)
    return einval("pgm_solve: a world > 1 context without NCCL needs pgm_peer_import first");
  if (!A || A->ctx != ctx) return einval("pgm_solve: matrix belongs to another context");
  if (A->n != ctx->n) return einval("pgm_solve: matrix rows do not match the partition");
  const bool harvest = dflt != nullptr;
  // the finishers and update passes keep a cycle's Hessenberg column and
  // coefficients in shared memory (MAX_M + O(1) doubles), the Ritz harvest
  // keeps [H | H^-1]: every path is bounded by MAX_M (BASELINE's largest
  // restart length is 100)
  if (cfg->m > (uint32_t)MAX_M)
    return einval("pgm_solve: restart length m > " + std::to_string(MAX_M) +
                  " is not supported on the device path");
  pgm_deflator* d = harvest ? dflt : ctx->dummy;
  if (d->ctx != ctx) return einval("pgm_solve: deflator belongs to another context");
  const int m = (int)cfg->m;
  const int maxr = (int)cfg->max_restarts;
  TRY(ensure_reduction(ctx, std::max(std::max(m + 1, 2 * d->R1 + 1), 2 * m + 2 + d->R1),
                       A->ntiles));
  // the peer window slot bounds the DCGS2 reduction (2m + 2 + r values):
  // larger restart lengths use CGS2 on the peer transport
  ctx->dc_now = ctx->dcgs2 && !(ctx->peer && 2 * m + 2 + d->R1 > PEER_NV);
  TRY(ensure_workspace(ctx, m, maxr, std::max(d->R1, 1)));
  TRY(defl_alloc_vectors(d));
  set_l2_window(ctx, d);
  if (harvest) {
    DState hs;
    CU(cudaMemcpy(&hs, d->d, sizeof(DState), cudaMemcpyDeviceToHost));
    TRY(defl_ensure_hist(d, hs.n_hist + maxr + 1));
  }
  const size_t n = ctx->n;
  TRY(copy_in(ctx, ctx->b + ctx->lo, b, n, flags));
  TRY(copy_in(ctx, ctx->x + ctx->lo, x, n, flags));
  GState gs{};
  gs.m = m;
  gs.max_restarts = maxr;
  gs.fixed = cfg->fixed_iterations != 0;
  gs.harvest = harvest ? 1 : 0;
  gs.rel_tol = cfg->rel_tol;
  gs.breakdown_scale = cfg->breakdown_scale;
  CU(cudaMemcpyAsync(ctx->g, &gs, sizeof(GState), cudaMemcpyHostToDevice, ctx->stream));
  const Params P = make_params(ctx, d);
  // In-process peer ranks share one GPU: a device-synchronising call on one
  // rank (cudaFree, ...) would wait for another rank's kernel spinning on the
  // first rank's reductions.  Every rank finishes its set-up before any
  // launches a reduction kernel.
  if (ctx->loop && ctx->peer) {
    CU(cudaStreamSynchronize(ctx->stream));
    ctx->loop->barrier();
  }
  ctx->cur_defl = d;
  ctx->launches = 0;
  ctx->prof.clear();
  ctx->ev_used = 0;
  ctx->prof_cycle = -1;
  CU(cudaEventRecord(ctx->ev0, ctx->stream));
  if (ctx->world > 1) TRY(halo_exchange(ctx, HV_X));
  TRY(launch_spmv(ctx, A, P, ResidualEpi{1}, d->R1 + 1));
  TRY(finish_global<101>(ctx, P, 1, d->R1 + 1));
  TRY(read_status(ctx));
  while (!ctx->h_status->done) {
    ctx->prof_cycle = ctx->h_status->restart;
    if (ctx->obs) {
      TRY(enqueue_cycle(ctx, A, d, P, harvest, false));
      TRY(observe_restart(ctx));
      TRY(enqueue_residual(ctx, A, d, P));
    } else {
      TRY(enqueue_cycle(ctx, A, d, P, harvest));
    }
    TRY(read_status(ctx));
    // a DCGS2 remainder at rounding level (finish.cuh dcgs2_column) closed the
    // cycle early: the remaining cycles of this solve run the CGS2 step
    if (ctx->dc_now && ctx->h_status->dc_fallback) ctx->dc_now = false;
    if (const char* e = std::getenv("PGMRES_DC_SWITCH_AT"))  // test knob: forced switch
      if (ctx->h_status->restart >= std::atoi(e)) ctx->dc_now = false;
  }
  CU(cudaEventRecord(ctx->ev1, ctx->stream));
  const GState hs = *ctx->h_status;
  TRY(copy_out(ctx, x, ctx->x + ctx->lo, n, flags));
  CU(cudaStreamSynchronize(ctx->stream));
  TRY(error_of(hs));
  if (rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->beta0 = hs.beta0;
    rep->restarts = (uint32_t)hs.restarts;
    rep->total_inner = hs.total_inner;
    rep->converged = hs.converged;
    rep->breakdown = hs.breakdown;
    rep->final_relative = hs.final_relative;
    rep->n_inner = (uint32_t)hs.n_inner;
    const size_t ni = std::max<size_t>(1, hs.n_inner), nr = std::max<size_t>(1, hs.restarts);
    rep->inner_restart = (uint32_t*)std::malloc(4 * ni);
    rep->inner_step = (uint32_t*)std::malloc(4 * ni);
    rep->inner_monitored = (double*)std::malloc(8 * ni);
    rep->explicit_residual = (double*)std::malloc(8 * nr);
    if (hs.n_inner > 0) {
      CU(cudaMemcpy(rep->inner_restart, ctx->rec_restart, 4 * hs.n_inner, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(rep->inner_step, ctx->rec_step, 4 * hs.n_inner, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(rep->inner_monitored, ctx->rec_mon, 8 * hs.n_inner, cudaMemcpyDeviceToHost));
    }
    if (hs.restarts > 0)
      CU(cudaMemcpy(rep->explicit_residual, ctx->expl, 8 * hs.restarts, cudaMemcpyDeviceToHost));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    rep->solve_seconds = 1e-3 * ms;
  }
  return {};
}

// ---------------------------------------------------------------------------
// Matrix upload: CSR (owned rows, global columns) -> SELL-32 tiles, layout
// built on the device (k_sell_layout: per-tile stable sort by row length).
// CSR values (and, on upload, column ids) -> the SELL arrays.  Device
// sources are gathered in place by one launch; host sources go through a
// bounded staging buffer one tile range at a time (<= STAGE_ENTRIES CSR
// entries, or one tile if a single tile holds more), so no nnz-sized staging
// copy is ever resident.  rp_src: the caller's row_ptr (host or device, as
// `dev` says); a host plan needs the host row_ptr, so a device-uploaded
// matrix that later receives host values copies row_ptr back once.
constexpr unsigned long long STAGE_ENTRIES = 1ull << 25;  // 32 M entries: 384 MB

Status gather_values(pgm_context* ctx, pgm_matrix* M, const uint32_t* rp_src,
                     const uint32_t* ci_src, const double* v_src, bool dev, bool write_cols) {
  cudaStream_t st = ctx->stream;
  if (M->nslices == 0) return {};
  const int threads = 256;
  if (dev) {
    const size_t blocks = ((size_t)M->nslices * 32 + threads - 1) / threads;
    k_csr_to_sell<<<(unsigned)blocks, threads, 0, st>>>(M->view(), M->val, M->col, M->rp,
                                                        ci_src, v_src, M->col_shift, 0,
                                                        M->nslices, 0ull, write_cols ? 1 : 0);
    CU(cudaGetLastError());
    return {};
  }
  if (M->chunks.empty()) {
    std::vector<uint32_t> hrp;
    const uint32_t* rp = rp_src;
    if (!rp) {
      hrp.resize((size_t)M->n + 1);
      CU(cudaMemcpyAsync(hrp.data(), M->rp, 4 * ((size_t)M->n + 1), cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      rp = hrp.data();
    }
    unsigned long long cap = 0;
    int t = 0;
    while (t < M->ntiles) {
      const int t0 = t;
      const unsigned long long lo = rp[(size_t)t0 * TILE];
      unsigned long long hi = lo;
      while (t < M->ntiles) {
        const size_t row_end = std::min<size_t>(M->n, (size_t)(t + 1) * TILE);
        const unsigned long long h = rp[row_end];
        if (t > t0 && h - lo > STAGE_ENTRIES) break;
        hi = h;
        ++t;
      }
      M->chunks.push_back({t0 * SPT, (t - t0) * SPT, lo, hi});
      cap = std::max(cap, hi - lo);
    }
    M->chunk_cap = cap;
  }
  // two staging buffers: the copy of chunk i+1 (copy stream) overlaps the
  // gather of chunk i (library stream); events order buffer reuse
  if (!ctx->cstream) {
    CU(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      CU(cudaEventCreateWithFlags(&ctx->ev_copy[b], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&ctx->ev_gath[b], cudaEventDisableTiming));
    }
  }
  double* sv[2] = {nullptr, nullptr};
  unsigned* sc[2] = {nullptr, nullptr};
  const size_t cap = std::max<unsigned long long>(M->chunk_cap, 1);
  const int nbuf = M->chunks.size() > 1 ? 2 : 1;
  Status s;
  for (int b = 0; b < nbuf && !s.code; ++b) {
    s = dalloc_async(&sv[b], cap, st);
    if (!s.code && write_cols) s = dalloc_async(&sc[b], cap, st);
  }
  cudaError_t e = cudaSuccess;
  if (!s.code) e = cudaEventRecord(ctx->ev_gath[0], st);  // buffers allocated (stream order)
  if (e == cudaSuccess && nbuf > 1) e = cudaEventRecord(ctx->ev_gath[1], st);
  // pageable sources (a std::vector, a numpy array): the driver would stage
  // them through its own pinned buffer with one host thread (~13 GB/s); here
  // host threads copy chunk i into a pinned ring while the DMA moves chunk
  // i - 1 (PCIe rate)
  cudaPointerAttributes pa{};
  const bool pageable = cudaPointerGetAttributes(&pa, v_src) != cudaSuccess ||
                        pa.type == cudaMemoryTypeUnregistered;
  cudaGetLastError();
  const size_t pin_bytes = cap * (write_cols ? 12 : 8);
  if (pageable && ctx->hpin_bytes < pin_bytes) {
    for (int b = 0; b < 2; ++b) {
      if (ctx->hpin[b]) cudaFreeHost(ctx->hpin[b]);
      ctx->hpin[b] = nullptr;
      if (!ctx->ev_hdma[b]) CU(cudaEventCreateWithFlags(&ctx->ev_hdma[b], cudaEventDisableTiming));
    }
    ctx->hpin_bytes = 0;
    if (cudaHostAlloc(&ctx->hpin[0], pin_bytes, cudaHostAllocDefault) == cudaSuccess &&
        cudaHostAlloc(&ctx->hpin[1], pin_bytes, cudaHostAllocDefault) == cudaSuccess) {
      ctx->hpin_bytes = pin_bytes;
    } else {  // no pinned memory: the driver's own staging
      cudaGetLastError();
      for (int b = 0; b < 2; ++b)
        if (ctx->hpin[b]) cudaFreeHost(ctx->hpin[b]), ctx->hpin[b] = nullptr;
    }
  }
  const bool ring = pageable && ctx->hpin_bytes >= pin_bytes;
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  auto par_copy = [hw](char* dst, const char* src, size_t bytes) {
    const size_t per = (bytes + hw - 1) / hw;
    std::vector<std::thread> team;
    for (unsigned t = 1; t < hw && t * per < bytes; ++t)
      team.emplace_back([=] { std::memcpy(dst + t * per, src + t * per, std::min(per, bytes - t * per)); });
    std::memcpy(dst, src, std::min(per, bytes));
    for (auto& th : team) th.join();
  };
  for (size_t i = 0; i < M->chunks.size(); ++i) {
    if (s.code || e != cudaSuccess) break;
    const auto& c = M->chunks[i];
    const int b = (int)(i % nbuf);
    const size_t cnt = c.hi - c.lo;
    const double* vsrc = v_src + c.lo;
    const uint32_t* csrc = write_cols ? ci_src + c.lo : nullptr;
    if (ring) {
      // the DMA that last read pinned buffer b must be done before refilling it
      const int hb = (int)(i % 2);
      if (i >= 2) e = cudaEventSynchronize(ctx->ev_hdma[hb]);
      char* hp = static_cast<char*>(ctx->hpin[hb]);
      par_copy(hp, reinterpret_cast<const char*>(vsrc), 8 * cnt);
      if (write_cols) par_copy(hp + 8 * cnt, reinterpret_cast<const char*>(csrc), 4 * cnt);
      vsrc = reinterpret_cast<const double*>(hp);
      if (write_cols) csrc = reinterpret_cast<const uint32_t*>(hp + 8 * cnt);
    }
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->cstream, ctx->ev_gath[b], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(sv[b], vsrc, 8 * cnt, cudaMemcpyHostToDevice, ctx->cstream);
    if (e == cudaSuccess && write_cols)
      e = cudaMemcpyAsync(sc[b], csrc, 4 * cnt, cudaMemcpyHostToDevice, ctx->cstream);
    if (e == cudaSuccess && ring) e = cudaEventRecord(ctx->ev_hdma[i % 2], ctx->cstream);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_copy[b], ctx->cstream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ctx->ev_copy[b], 0);
    if (e == cudaSuccess) {
      const size_t blocks = ((size_t)c.count * 32 + threads - 1) / threads;
      k_csr_to_sell<<<(unsigned)blocks, threads, 0, st>>>(M->view(), M->val, M->col, M->rp,
                                                          sc[b], sv[b], M->col_shift, c.s0,
                                                          c.count, c.lo, write_cols ? 1 : 0);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_gath[b], st);
  }
  for (int b = 0; b < 2; ++b) {
    dfree_async(sv[b], st);
    dfree_async(sc[b], st);
  }
  if (s.code) return s;
  CU(e);
  return {};
}

Status matrix_upload(pgm_context* ctx, const pgm_csr_view* a, int32_t flags, pgm_matrix** out) {
  if (!a || !out) return einval("pgm_matrix_upload: null argument");
  if (a->n != ctx->n)
    return einval("pgm_matrix_upload: view has " + std::to_string(a->n) + " rows, partition owns " +
                  std::to_string(ctx->n));
  const bool dev = (flags & PGM_DEVICE_PTRS) != 0;
  cudaStream_t st = ctx->stream;
  auto* M = new pgm_matrix();
  M->ctx = ctx;
  M->n = a->n;
  M->nnz = a->nnz;
  M->ntiles = (int)((a->n + TILE - 1) / TILE);
  M->nslices = M->ntiles * SPT;
  M->col_shift = ctx->part.row_begin - ctx->part.halo_lo;
  auto cleanup = [&](Status s) {
    cudaStreamSynchronize(st);
    pgm_matrix_destroy(M);
    return s;
  };
  Status s;
  const cudaMemcpyKind kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  cudaError_t e = cudaSuccess;
  // row_ptr checks (start 0, end nnz, monotone) on the device copy
  if ((s = dalloc_async(&M->rp, (size_t)a->n + 1, st)).code) return cleanup(s);
  e = cudaMemcpyAsync(M->rp, a->row_ptr, 4 * ((size_t)a->n + 1), kind, st);
  const size_t ns = (size_t)M->nslices;
  if ((s = dalloc_async(&M->sptr, ns + 1, st)).code) return cleanup(s);
  if ((s = dalloc_async(&M->lane_len, ns * 32, st)).code) return cleanup(s);
  if ((s = dalloc_async(&M->lane_row, ns * 32, st)).code) return cleanup(s);
  int* dbad = nullptr;
  void* dtmp = nullptr;
  size_t tmp_bytes = 0;
  if ((s = dalloc_async(&dbad, 1, st)).code) return cleanup(s);
  e = e ? e : cudaMemsetAsync(dbad, 0, sizeof(int), st);
  if (e == cudaSuccess && M->ntiles > 0) {
    k_sell_layout<<<M->ntiles, 256, 0, st>>>(M->rp, (int)a->n, (unsigned long long)a->nnz,
                                             M->lane_len, M->lane_row, M->sptr, dbad);
    e = cudaGetLastError();
  }
  // sptr = exclusive scan of the slice sizes (k_sell_layout wrote them to sptr[s])
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, M->sptr, M->sptr, (int)(ns + 1), st);
  if ((s = dalloc_async((char**)&dtmp, tmp_bytes, st)).code) return cleanup(s);
  e = e ? e : cudaMemsetAsync(M->sptr + ns, 0, sizeof(unsigned long long), st);
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(dtmp, tmp_bytes, M->sptr, M->sptr, (int)(ns + 1), st);
  unsigned long long stored = 0;
  int bad = 0;
  e = e ? e : cudaMemcpyAsync(&stored, M->sptr + ns, 8, cudaMemcpyDeviceToHost, st);
  e = e ? e : cudaMemcpyAsync(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost, st);
  e = e ? e : cudaStreamSynchronize(st);
  cudaFreeAsync(dtmp, st);
  cudaFreeAsync(dbad, st);
  if (e != cudaSuccess)
    return cleanup(Status{PGM_ECUDA, std::string("upload layout: ") + cudaGetErrorString(e)});
  if (bad & 1) return cleanup(einval("pgm_matrix_upload: row_ptr must start at 0 and end at nnz"));
  if (bad & 2) return cleanup(einval("pgm_matrix_upload: row_ptr not monotone"));
  M->stored = stored;
  if ((s = dalloc_async(&M->val, M->stored, st)).code) return cleanup(s);
  if ((s = dalloc_async(&M->col, M->stored, st)).code) return cleanup(s);
  if ((s = gather_values(ctx, M, a->row_ptr, a->col_idx, a->values, dev, true)).code)
    return cleanup(s);
  const int threads = 256;
  const size_t blocks = ((size_t)M->nslices * 32 + threads - 1) / threads;
  unsigned* col32 = M->col;
  e = cudaGetLastError();
  if (e == cudaSuccess && M->nslices > 0 && !std::getenv("PGMRES_NO_C16")) {
    // 16-bit column deltas when every gap fits (10 instead of 12 B / nonzero)
    unsigned* dm = nullptr;
    unsigned hm = 0;
    e = cudaMallocAsync(reinterpret_cast<void**>(&dm), sizeof(unsigned), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(dm, 0, sizeof(unsigned), st);
    if (e == cudaSuccess) k_sell_delta_max<<<(unsigned)blocks, threads, 0, st>>>(M->view(), M->nslices, dm);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hm, dm, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFreeAsync(dm, st);
    if (e == cudaSuccess && hm <= 0xFFFFu) {
      if (cudaMallocAsync(reinterpret_cast<void**>(&M->col16), 2 * M->stored, st) == cudaSuccess &&
          cudaMallocAsync(reinterpret_cast<void**>(&M->lane_base), 4 * (size_t)M->nslices * 32,
                          st) == cudaSuccess) {
        Sell v32 = M->view();
        v32.col16 = nullptr;
        k_sell_compress<<<(unsigned)blocks, threads, 0, st>>>(v32, M->nslices, M->col16,
                                                              M->lane_base);
        e = cudaGetLastError();
        if (e == cudaSuccess) M->col = nullptr;  // col32 freed after the halo scan
      } else {
        cudaGetLastError();  // not enough memory: keep 32-bit columns
        dfree_async(M->col16, st);
        dfree_async(M->lane_base, st);
      }
    }
  }
  M->t_lo_end = 0;
  M->t_hi_begin = M->ntiles;
  if (e == cudaSuccess && ctx->world > 1 && a->n > 0) {
    // halo tiles from the 32-bit SELL columns (k_sell_compress keeps `col`
    // until the stream reaches its free)
    int h[2] = {-1, (int)a->n};
    int* dh = nullptr;
    e = cudaMalloc(&dh, sizeof(h));
    if (e == cudaSuccess) e = cudaMemcpyAsync(dh, h, sizeof(h), cudaMemcpyHostToDevice, st);
    Sell v32 = M->view();
    v32.col16 = nullptr;
    v32.col = col32;
    if (e == cudaSuccess)
      k_halo_rows_sell<<<(unsigned)blocks, threads, 0, st>>>(
          v32, M->nslices, ctx->part.halo_lo, ctx->part.halo_lo + (unsigned)a->n, dh);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, dh, sizeof(h), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(dh);
    M->t_lo_end = (h[0] + 1 + TILE - 1) / TILE;
    M->t_hi_begin = std::max(M->t_lo_end, h[1] / TILE);
  }
  if (col32 != M->col) dfree_async(col32, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess)
    return cleanup(Status{PGM_ECUDA, std::string("csr->sell: ") + cudaGetErrorString(e)});
  ctx->mats.push_back(M);
  *out = M;
  return {};
}

}  // namespace

// ===========================================================================
// Multi-GPU plumbing (NCCL through a dlopen'ed libnccl: the library carries no
// link-time dependency, single-GPU use never loads it).
namespace {

Status allreduce_red(pgm_context* ctx, int nv) {
  if (ctx->peer) {  // through the peer windows (same epoch sequence as the reduction kernels)
    if (nv > PEER_NV) return Status{PGM_ESTATE, "allreduce_red: payload exceeds the peer slot"};
    const Params P = make_params(ctx, ctx->cur_defl ? ctx->cur_defl : ctx->dummy);
    k_peer_allreduce_buf<<<1, 128, 0, ctx->stream>>>(P, ctx->red_out, nv);
    ctx->launches++;
    CU(cudaGetLastError());
    return {};
  }
  if (ctx->loop) {
    pgm_loopback* L = ctx->loop;
    CU(cudaStreamSynchronize(ctx->stream));
    L->barrier();
    std::vector<double>& mine = L->host[ctx->rank];
    mine.resize((size_t)nv * L->world);
    for (int q = 0; q < L->world; ++q)
      CU(cudaMemcpy(mine.data() + (size_t)q * nv, L->ctx[q]->red_out, 8 * (size_t)nv,
                    cudaMemcpyDeviceToHost));
    L->barrier();
    std::vector<double> sum(nv, 0.0);
    for (int q = 0; q < L->world; ++q)  // fixed rank order: identical on every rank
      for (int v = 0; v < nv; ++v) sum[v] += mine[(size_t)q * nv + v];
    CU(cudaMemcpyAsync(ctx->red_out, sum.data(), 8 * (size_t)nv, cudaMemcpyHostToDevice,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return {};
  }
  if (!nccl_lite::available() || !ctx->nccl) return Status{PGM_ENCCL, "NCCL not initialised"};
  if (nccl_lite::allreduce_sum_f64(ctx->red_out, ctx->red_out, (size_t)nv, ctx->nccl, ctx->stream) != 0)
    return Status{PGM_ENCCL, "ncclAllReduce failed"};
  return {};
}

double* halo_vec(pgm_context* ctx, HaloKind kind, int slot) {
  switch (kind) {
    case HV_V: return ctx->V + (size_t)slot * ctx->ld;
    case HV_X: return ctx->x;
    case HV_U: return ctx->cur_defl ? ctx->cur_defl->u : nullptr;
    case HV_TMP: return ctx->tmp;
    case HV_PTR: return ctx->halo_ptr;
  }
  return nullptr;
}

// Exchange the two boundary planes of a vector with the z-neighbours: own rows
// [0, halo) go down into the lower neighbour's halo_hi region and own rows
// [n - halo, n) go up into the upper neighbour's halo_lo region (slabs are at
// least two planes thick, so halos only ever come from adjacent ranks).
Status halo_exchange(pgm_context* ctx, HaloKind kind, int slot, cudaStream_t st) {
  if (ctx->world == 1) return {};
  if (!st) st = ctx->stream;
  ProfScope ps(ctx, PC_HALO, (uint32_t)slot, st);
  double* vec = halo_vec(ctx, kind, slot);
  const size_t lo = ctx->lo, hi = ctx->hi, n = ctx->n;
  const int below = ctx->rank - 1, above = ctx->rank + 1;
  if (ctx->peer) {
    // boundary planes through the neighbours' peer-memory mailboxes
    HaloPeerArgs A{};
    A.win = ctx->d_peer_base;
    A.mine = ctx->pbuf;
    A.off_mb = peer_mb_offset(ctx);
    A.off_hf = peer_hf_offset(ctx);
    A.hmax = peer_halo_rows(ctx);
    A.me = ctx->rank;
    A.world = ctx->world;
    A.epoch = reinterpret_cast<unsigned long long*>(ctx->pbuf + A.off_hf) + 4;
    A.cnt = reinterpret_cast<unsigned*>(reinterpret_cast<unsigned long long*>(ctx->pbuf + A.off_hf) + 5);
    A.g = ctx->g;
    const int dn = below >= 0 ? (int)lo : 0, up = above < ctx->world ? (int)hi : 0;
    const int G = std::max(1, std::min(ctx->nsm / 4, (int)((std::max(lo, hi) + 2047) / 2048)));
    k_halo_push<<<G, 256, 0, st>>>(A, vec + lo, (int)n, dn, up);
    k_halo_pull<<<G, 256, 0, st>>>(A, vec, below >= 0 ? (int)lo : 0, (int)n,
                                   above < ctx->world ? (int)hi : 0);
    ctx->launches += 2;
    CU(cudaGetLastError());
    return {};
  }
  if (ctx->loop) {
    pgm_loopback* L = ctx->loop;
    CU(cudaStreamSynchronize(ctx->stream));
    L->barrier();
    if (below >= 0 && lo > 0) {
      pgm_context* nb = L->ctx[below];
      const double* src = halo_vec(nb, kind, slot) + nb->lo + nb->n - nb->hi;
      CU(cudaMemcpyAsync(vec, src, 8 * lo, cudaMemcpyDeviceToDevice, st));
    }
    if (above < ctx->world && hi > 0) {
      pgm_context* na = L->ctx[above];
      const double* src = halo_vec(na, kind, slot) + na->lo;
      CU(cudaMemcpyAsync(vec + lo + n, src, 8 * hi, cudaMemcpyDeviceToDevice, st));
    }
    CU(cudaStreamSynchronize(st));
    L->barrier();
    return {};
  }
  if (!ctx->nccl) return Status{PGM_ENCCL, "NCCL not initialised"};
  if (nccl_lite::group_start() != 0) return Status{PGM_ENCCL, "ncclGroupStart failed"};
  int rc = 0;
  if (below >= 0 && lo > 0) {
    rc |= nccl_lite::send_f64(vec + lo, lo, below, ctx->nccl, st);
    rc |= nccl_lite::recv_f64(vec, lo, below, ctx->nccl, st);
  }
  if (above < ctx->world && hi > 0) {
    rc |= nccl_lite::send_f64(vec + lo + n - hi, hi, above, ctx->nccl, st);
    rc |= nccl_lite::recv_f64(vec + lo + n, hi, above, ctx->nccl, st);
  }
  rc |= nccl_lite::group_end();
  if (rc) return Status{PGM_ENCCL, "halo exchange failed"};
  return {};
}

}  // namespace

// ===========================================================================
// C ABI
extern "C" {

const char* pgm_last_error(const pgm_context* ctx) {
  return ctx ? ctx->err.c_str() : g_tls_err.c_str();
}

pgm_status pgm_partition_rows(uint32_t n_axis, uint32_t p, uint32_t w, pgm_partition* out) {
  if (!out || p == 0 || p > n_axis || w >= p) {
    g_tls_err = "partition_rows: need 1 <= p <= n_axis";
    return PGM_EINVAL;
  }
  const uint64_t plane = (uint64_t)n_axis * n_axis;
  const uint32_t q = n_axis / p, rem = n_axis % p;
  uint32_t zb = 0;
  for (uint32_t i = 0; i < w; ++i) zb += q + (i < rem ? 1 : 0);
  const uint32_t ze = zb + q + (w < rem ? 1 : 0);
  const uint32_t lo = zb >= 2 ? zb - 2 : 0;
  const uint32_t hi = std::min(n_axis, ze + 2);
  out->row_begin = (uint32_t)(zb * plane);
  out->row_end = (uint32_t)(ze * plane);
  out->halo_lo = (uint32_t)((zb - lo) * plane);
  out->halo_hi = (uint32_t)((hi - ze) * plane);
  return PGM_OK;
}

pgm_status pgm_context_create(const pgm_context_config* cfg, pgm_context** out) {
  if (!cfg || !out) {
    g_tls_err = "pgm_context_create: null argument";
    return PGM_EINVAL;
  }
  *out = nullptr;
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world || cfg->n_global == 0) {
    g_tls_err = "pgm_context_create: bad rank/world/n_global";
    return PGM_EINVAL;
  }
  auto* ctx = new pgm_context();
  if (const char* e = std::getenv("PGMRES_PDL")) ctx->pdl = e[0] != '0';
  if (const char* e = std::getenv("PGMRES_DCGS2")) ctx->dcgs2 = e[0] != '0';
  ctx->device = cfg->device;
  ctx->rank = cfg->rank;
  ctx->world = cfg->world;
  ctx->n_axis = cfg->n_axis;
  ctx->n_global = cfg->n_global;
  if (cfg->world == 1) {
    ctx->part = pgm_partition{0, cfg->n_global, 0, 0};
  } else if (cfg->n_axis > 0) {
    if ((uint64_t)cfg->n_axis * cfg->n_axis * cfg->n_axis != cfg->n_global) {
      delete ctx;
      g_tls_err = "pgm_context_create: n_global != n_axis^3";
      return PGM_EINVAL;
    }
    if (pgm_partition_rows(cfg->n_axis, cfg->world, cfg->rank, &ctx->part) != PGM_OK) {
      delete ctx;
      return PGM_EINVAL;
    }
    if (cfg->n_axis / cfg->world < 2) {  // halos (2 planes) must come from adjacent ranks
      delete ctx;
      g_tls_err = "pgm_context_create: every z-slab needs at least two node planes";
      return PGM_EINVAL;
    }
  } else {
    delete ctx;
    g_tls_err = "pgm_context_create: world > 1 needs the mesh n_axis (z-slab partition)";
    return PGM_EINVAL;
  }
  ctx->n = ctx->part.row_end - ctx->part.row_begin;
  ctx->lo = ctx->part.halo_lo;
  ctx->hi = ctx->part.halo_hi;
  if (cfg->deterministic == PGM_DETERMINISTIC_PLANES) {
    // planes = the reference's deterministic reduction blocks (n_axis^2 rows,
    // partition_rows: slabs of whole planes); without mesh structure one plane
    ctx->det = true;
    ctx->plane = cfg->n_axis > 0 ? (int)(cfg->n_axis * cfg->n_axis) : (int)cfg->n_global;
    ctx->nplanes_global = cfg->n_axis > 0 ? (int)cfg->n_axis : 1;
    for (int q = 0; q < cfg->world; ++q) {
      pgm_partition pq = ctx->part;
      if (cfg->world > 1) pgm_partition_rows(cfg->n_axis, cfg->world, q, &pq);
      const int cnt = (int)((pq.row_end - pq.row_begin) / ctx->plane);
      ctx->plane_off.push_back(q == 0 ? 0 : ctx->plane_off.back() + ctx->plane_cnt.back());
      ctx->plane_cnt.push_back(cnt);
      ctx->det_maxp = std::max(ctx->det_maxp, cnt);
    }
    ctx->nplanes = ctx->plane_cnt[cfg->rank];
  }
  // +256: bulk copies read whole 256-row chunks past the last owned row
  ctx->ld = round_up(ctx->lo + ctx->n + ctx->hi + 256, 128);
  auto bail = [&](const Status& s) {
    pgm_status c = fail(nullptr, s);
    pgm_context_destroy(ctx);
    return c;
  };
  cudaError_t e = cudaSetDevice(cfg->device);
  if (e != cudaSuccess) return bail(Status{PGM_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)});
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cfg->device);
  ctx->nsm = nsm > 0 ? nsm : 148;
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, cfg->device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;  // keep freed matrix arrays cached in the pool
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return bail(Status{PGM_ECUDA, std::string("stream: ") + cudaGetErrorString(e)});
  cudaEventCreate(&ctx->ev0);
  cudaEventCreate(&ctx->ev1);
  if (ctx->world > 1) {
    cudaStreamCreateWithFlags(&ctx->hstream, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&ctx->ev_halo_src, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->ev_halo_done, cudaEventDisableTiming);
  }
  Status s;
  if ((s = dalloc(&ctx->g, 1)).code) return bail(s);
  if ((e = cudaMallocHost(&ctx->h_dstate, sizeof(DState))) != cudaSuccess)
    return bail(Status{PGM_ENOMEM, "cudaMallocHost"});
  std::memset(ctx->h_dstate, 0, sizeof(DState));
  if ((e = cudaMallocHost(&ctx->h_status, sizeof(GState))) != cudaSuccess)
    return bail(Status{PGM_ENOMEM, "pinned status"});
  std::memset(ctx->h_status, 0, sizeof(GState));
  if ((s = dalloc(&ctx->x, ctx->ld)).code) return bail(s);
  if ((s = dalloc(&ctx->b, ctx->ld)).code) return bail(s);
  if ((s = dalloc(&ctx->tmp, ctx->ld)).code) return bail(s);
  cudaMemset(ctx->x, 0, 8 * ctx->ld);
  cudaMemset(ctx->b, 0, 8 * ctx->ld);
  cudaMemset(ctx->tmp, 0, 8 * ctx->ld);
  if ((s = ensure_reduction(ctx, 2 * MAX_R1 + MAX_M + 8)).code) return bail(s);
  if ((s = set_gstate_idle(ctx)).code) return bail(s);
  if (cfg->world > 1) {
    if ((s = dalloc(&ctx->pbuf, peer_buf_bytes(ctx))).code) return bail(s);
    if (cudaMemset(ctx->pbuf, 0, peer_buf_bytes(ctx)) != cudaSuccess)
      return bail(Status{PGM_ECUDA, "cudaMemset(peer window)"});
  }
  if (cfg->world > 1 && cfg->loopback) {
    pgm_loopback* L = static_cast<pgm_loopback*>(cfg->loopback);
    if (L->world != cfg->world) return bail(Status{PGM_EINVAL, "loopback group size != world"});
    ctx->loop = L;
    {
      std::lock_guard<std::mutex> lk(L->mu);
      L->ctx[cfg->rank] = ctx;
    }
    // in-process ranks: the fused peer-memory allreduce with plain pointers
    // (PGMRES_PEER=0 keeps the host-staged loopback collective instead).  PDL
    // off: an early-launched next kernel could hold the SMs a spinning peer
    // rank on the same GPU needs.
    ctx->pdl = false;
    // Spinning peers need every kernel resident without a context-wide module
    // load in between: peer mode only with CUDA_MODULE_LOADING=EAGER (lazy
    // loading of a kernel's module waits for the other ranks' spinning kernels).
    const char* pe = std::getenv("PGMRES_PEER");
    const char* ml = std::getenv("CUDA_MODULE_LOADING");
    const bool want_peer =
        !ctx->det && !(pe && pe[0] == '0') && ml && std::string(ml) == "EAGER";
    L->barrier();  // every rank registered and has its window
    if (want_peer) {
      std::vector<char*> bufs(cfg->world);
      for (int q = 0; q < cfg->world; ++q) bufs[q] = L->ctx[q]->pbuf;
      if ((s = peer_set_tables(ctx, bufs)).code) return bail(s);
    }
    L->barrier();
  } else if (cfg->world > 1 && !cfg->nccl_id) {
    // peer-only: no NCCL; halos and reductions go through the CUDA-IPC peer
    // windows once pgm_peer_import has mapped them (solves refuse before)
  } else if (cfg->world > 1 || cfg->nccl_id) {
    if (!nccl_lite::available()) return bail(Status{PGM_ENCCL, "libnccl.so.2 not loadable"});
    if (!cfg->nccl_id) return bail(Status{PGM_EINVAL, "world > 1 needs an ncclUniqueId"});
    if (nccl_lite::comm_init_rank(&ctx->nccl, cfg->world, cfg->nccl_id, cfg->rank) != 0)
      return bail(Status{PGM_ENCCL, "ncclCommInitRank failed"});
  }
  ctx->coll = ctx->world > 1 || ctx->nccl != nullptr;
  // dummy deflator (r = 0 forever) for plain gmres_restarted solves
  pgm_deflation_config dc{1, 1, 1e-8, 1, 1e-10, 1};
  pgm_deflator* dd = nullptr;
  if (pgm_deflator_create(ctx, &dc, &dd) != PGM_OK) {
    pgm_status c = PGM_ENOMEM;
    pgm_context_destroy(ctx);
    return c;
  }
  dd->dummy = true;
  ctx->dummy = dd;
  cudaDeviceSynchronize();
  *out = ctx;
  return PGM_OK;
}

void pgm_context_destroy(pgm_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (pgm_matrix* m : ctx->mats) m->ctx = nullptr;  // destroyed later with plain frees
  ctx->mats.clear();
  for (void* p : ctx->peer_opened) cudaIpcCloseMemHandle(p);
  ctx->peer_opened.clear();
  dfree(ctx->d_peer_win);
  dfree(ctx->d_peer_flag);
  dfree(ctx->d_peer_base);
  dfree(ctx->pbuf);
  if (ctx->dummy) pgm_deflator_destroy(ctx->dummy);
  free_workspace(ctx);
  dfree(ctx->x);
  dfree(ctx->b);
  dfree(ctx->tmp);
  dfree(ctx->g);
  dfree(ctx->part_buf);
  dfree(ctx->gpart_buf);
  dfree(ctx->g2part_buf);
  dfree(ctx->cnt);
  dfree(ctx->red_out);
  dfree(ctx->det_pp);
  dfree(ctx->det_all);
  dfree(ctx->det_gbuf);
  dfree(ctx->det_cnt);
  if (ctx->cstream) cudaStreamDestroy(ctx->cstream);
  for (int b = 0; b < 2; ++b) {
    if (ctx->hpin[b]) cudaFreeHost(ctx->hpin[b]);
    if (ctx->ev_hdma[b]) cudaEventDestroy(ctx->ev_hdma[b]);
  }
  for (int b = 0; b < 2; ++b) {
    if (ctx->ev_copy[b]) cudaEventDestroy(ctx->ev_copy[b]);
    if (ctx->ev_gath[b]) cudaEventDestroy(ctx->ev_gath[b]);
  }
  if (ctx->h_status) cudaFreeHost(ctx->h_status);
  if (ctx->h_dstate) cudaFreeHost(ctx->h_dstate);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->ev_halo_src) cudaEventDestroy(ctx->ev_halo_src);
  if (ctx->ev_halo_done) cudaEventDestroy(ctx->ev_halo_done);
  if (ctx->hstream) cudaStreamDestroy(ctx->hstream);
  if (ctx->nccl) nccl_lite::comm_destroy(ctx->nccl);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

pgm_status pgm_loopback_create(int32_t world, pgm_loopback** out) {
  if (!out || world < 1) return PGM_EINVAL;
  auto* L = new pgm_loopback();
  L->world = world;
  L->ctx.assign(world, nullptr);
  L->host.resize(world);
  *out = L;
  return PGM_OK;
}

void pgm_loopback_destroy(pgm_loopback* g) { delete g; }

pgm_status pgm_context_partition(const pgm_context* ctx, pgm_partition* out) {
  if (!ctx || !out) return PGM_EINVAL;
  *out = ctx->part;
  return PGM_OK;
}

void* pgm_context_stream(pgm_context* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

uint64_t pgm_context_launch_count(const pgm_context* ctx) { return ctx ? ctx->launches : 0; }

pgm_status pgm_matrix_upload(pgm_context* ctx, const pgm_csr_view* a, int32_t flags,
                             pgm_matrix** out) {
  if (!ctx) return PGM_EINVAL;
  cudaSetDevice(ctx->device);
  Status s = matrix_upload(ctx, a, flags, out);
  return s.code ? fail(ctx, s) : PGM_OK;
}

pgm_status pgm_matrix_update_values(pgm_matrix* a, const double* values, int32_t flags) {
  if (!a) return PGM_EINVAL;
  if (!a->ctx) {
    g_tls_err = "pgm_matrix_update_values: the matrix's context was destroyed";
    return PGM_ESTATE;
  }
  pgm_context* ctx = a->ctx;
  cudaStream_t st = ctx->stream;
  Status s = gather_values(ctx, a, nullptr, nullptr, values, (flags & PGM_DEVICE_PTRS) != 0,
                           false);
  if (s.code) return fail(ctx, s);
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(ctx, Status{PGM_ECUDA, cudaGetErrorString(e)});
  return PGM_OK;
}

void pgm_matrix_destroy(pgm_matrix* a) {
  if (!a) return;
  pgm_context* ctx = a->ctx;
  if (ctx) {
    auto& v = ctx->mats;
    v.erase(std::remove(v.begin(), v.end(), a), v.end());
    cudaStream_t st = ctx->stream;
    dfree_async(a->sptr, st);
    dfree_async(a->lane_len, st);
    dfree_async(a->lane_row, st);
    dfree_async(a->val, st);
    dfree_async(a->col, st);
    dfree_async(a->col16, st);
    dfree_async(a->lane_base, st);
    dfree_async(a->rp, st);
  } else {  // its context was destroyed first: plain (synchronous) frees
    cudaDeviceSynchronize();
    dfree(a->sptr);
    dfree(a->lane_len);
    dfree(a->lane_row);
    dfree(a->val);
    dfree(a->col);
    dfree(a->col16);
    dfree(a->lane_base);
    dfree(a->rp);
  }
  delete a;
}
pgm_status pgm_matrix_info(const pgm_matrix* a, uint32_t* n, uint64_t* nnz, uint64_t* stored,
                           uint64_t* device_bytes) {
  if (!a) return PGM_EINVAL;
  if (n) *n = a->n;
  if (nnz) *nnz = a->nnz;
  if (stored) *stored = a->stored;
  if (device_bytes)
    *device_bytes = a->stored * (a->col16 ? 10 : 12) +
                    (uint64_t)a->nslices * (8 + 32 * (a->col16 ? 10 : 6)) + 4ull * (a->n + 1);
  return PGM_OK;
}

pgm_status pgm_spmv(pgm_matrix* a, const double* x, double* y, int32_t flags) {
  if (a && !a->ctx) {
    g_tls_err = "pgm_spmv: the matrix's context was destroyed";
    return PGM_ESTATE;
  }
  if (!a) return PGM_EINVAL;
  pgm_context* ctx = a->ctx;
  cudaSetDevice(ctx->device);
  auto run = [&]() -> Status {
    TRY(set_gstate_idle(ctx));
    if (ctx->loop && ctx->peer) {  // in-process peer ranks start the exchange together
      CU(cudaStreamSynchronize(ctx->stream));
      ctx->loop->barrier();
    }
    TRY(copy_in(ctx, ctx->tmp + ctx->lo, x, ctx->n, flags));
    if (ctx->world > 1) TRY(halo_exchange(ctx, HV_TMP));
    Params P = make_params(ctx, ctx->dummy);
    PlainEpi E{ctx->tmp, ctx->b + ctx->lo};
    TRY(launch_spmv(ctx, a, P, E, 0));
    TRY(copy_out(ctx, y, ctx->b + ctx->lo, ctx->n, flags));
    CU(cudaStreamSynchronize(ctx->stream));
    if (ctx->world > 1) {  // a halo wait that timed out flags the state
      int err = 0;
      CU(cudaMemcpy(&err, &ctx->g->error, sizeof(int), cudaMemcpyDeviceToHost));
      if (err) return Status{PGM_ESTATE, "pgm_spmv: a peer rank never delivered its halo planes"};
    }
    return {};
  };
  Status s = run();
  return s.code ? fail(ctx, s) : PGM_OK;
}

pgm_status pgm_deflator_create(pgm_context* ctx, const pgm_deflation_config* cfg,
                               pgm_deflator** out) {
  if (!ctx || !cfg || !out) return PGM_EINVAL;
  if (cfg->r_max == 0) return fail(ctx, einval("deflation: r_max must be positive"));
  if (cfg->drop == 0) return fail(ctx, einval("deflation: drop must be positive"));
  if (cfg->r_max + 1 > (uint32_t)MAX_R1)
    return fail(ctx, einval("deflation: r_max > " + std::to_string(MAX_R1 - 1) +
                                " is not supported by the device path"));
  cudaSetDevice(ctx->device);
  auto* d = new pgm_deflator();
  d->ctx = ctx;
  d->cfg = *cfg;
  d->R1 = (int)cfg->r_max + 1;
  auto run = [&]() -> Status {
    const int R1 = d->R1;
    TRY(dalloc(&d->d, 1));
    TRY(dalloc(&d->T, (size_t)R1 * R1));
    TRY(dalloc(&d->Tinv, (size_t)R1 * R1));
    TRY(dalloc(&d->Q, (size_t)R1 * R1));
    TRY(dalloc(&d->proj, R1 + 1));
    TRY(dalloc(&d->dwork, (size_t)16 * R1 * R1 + 32 * R1));
    TRY(dalloc(&d->iwork, 4 * R1));
    CU(cudaMemset(d->T, 0, 8 * R1 * R1));
    CU(cudaMemset(d->Tinv, 0, 8 * R1 * R1));
    DState ds{};
    ds.r_max = (int)cfg->r_max;
    ds.drop = (int)cfg->drop;
    ds.accept_tol = cfg->accept_tol;
    ds.inv_maxit = (int)cfg->inv_power_maxit;
    ds.inv_tol = cfg->inv_power_tol;
    ds.pow_maxit = (int)cfg->power_maxit;
    CU(cudaMemcpy(d->d, &ds, sizeof(DState), cudaMemcpyHostToDevice));
    TRY(defl_ensure_hist(d, 64));
    return {};
  };
  Status s = run();
  if (s.code) {
    pgm_deflator_destroy(d);
    return fail(ctx, s);
  }
  *out = d;
  return PGM_OK;
}

void pgm_deflator_destroy(pgm_deflator* d) {
  if (!d) return;
  dfree(d->d);
  dfree(d->U);
  dfree(d->AU);
  dfree(d->u);
  dfree(d->T);
  dfree(d->Tinv);
  dfree(d->Q);
  dfree(d->proj);
  dfree(d->dwork);
  dfree(d->iwork);
  dfree(d->hist_restart);
  dfree(d->hist_r);
  dfree(d->hist_mu);
  dfree(d->hist_theta);
  delete d;
}

pgm_status pgm_deflator_reset(pgm_deflator* d) {
  if (!d) return PGM_EINVAL;
  DState ds;
  cudaStreamSynchronize(d->ctx->stream);
  cudaMemcpy(&ds, d->d, sizeof(DState), cudaMemcpyDeviceToHost);
  ds.r = 0;
  ds.mu = 0.0;
  ds.skipped = 0;
  ds.n_hist = 0;
  ds.rotate = 0;
  ds.push_ok = 0;
  cudaError_t e = cudaMemcpy(d->d, &ds, sizeof(DState), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return fail(d->ctx, Status{PGM_ECUDA, cudaGetErrorString(e)});
  return PGM_OK;
}

pgm_status pgm_deflator_info(pgm_deflator* d, uint32_t* rank, double* mu, uint32_t* skipped,
                             uint32_t* n_history) {
  if (!d) return PGM_EINVAL;
  DState ds;
  cudaStreamSynchronize(d->ctx->stream);
  cudaError_t e = cudaMemcpy(&ds, d->d, sizeof(DState), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fail(d->ctx, Status{PGM_ECUDA, cudaGetErrorString(e)});
  if (rank) *rank = (uint32_t)ds.r;
  if (mu) *mu = ds.mu;
  if (skipped) *skipped = (uint32_t)ds.skipped;
  if (n_history) *n_history = (uint32_t)ds.n_hist;
  return PGM_OK;
}

pgm_status pgm_deflator_history(pgm_deflator* d, pgm_deflation_record* out, uint32_t cap) {
  if (!d || !out) return PGM_EINVAL;
  DState ds;
  cudaStreamSynchronize(d->ctx->stream);
  cudaMemcpy(&ds, d->d, sizeof(DState), cudaMemcpyDeviceToHost);
  const uint32_t n = std::min<uint32_t>(cap, (uint32_t)std::min(ds.n_hist, d->hist_cap));
  std::vector<uint32_t> hr(n), hrr(n);
  std::vector<double> hm(n), ht(n);
  if (n) {
    cudaMemcpy(hr.data(), d->hist_restart, 4 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(hrr.data(), d->hist_r, 4 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(hm.data(), d->hist_mu, 8 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(ht.data(), d->hist_theta, 8 * n, cudaMemcpyDeviceToHost);
  }
  for (uint32_t i = 0; i < n; ++i) out[i] = {hr[i], hrr[i], hm[i], ht[i]};
  return PGM_OK;
}

pgm_status pgm_deflator_basis(pgm_deflator* d, double* U, double* T) {
  if (!d) return PGM_EINVAL;
  pgm_context* ctx = d->ctx;
  DState ds;
  cudaStreamSynchronize(ctx->stream);
  cudaMemcpy(&ds, d->d, sizeof(DState), cudaMemcpyDeviceToHost);
  const int r = ds.r;
  if (U && d->U)
    for (int j = 0; j < r; ++j)
      cudaMemcpy(U + (size_t)j * ctx->n, d->U + (size_t)j * ctx->ld + ctx->lo, 8 * ctx->n,
                 cudaMemcpyDeviceToHost);
  if (T && r > 0) {
    std::vector<double> t((size_t)d->R1 * d->R1);
    cudaMemcpy(t.data(), d->T, 8 * t.size(), cudaMemcpyDeviceToHost);
    for (int j = 0; j < r; ++j)
      for (int i = 0; i < r; ++i) T[i + j * r] = t[i + (size_t)j * d->R1];
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, Status{PGM_ECUDA, cudaGetErrorString(e)});
  return PGM_OK;
}

}  // extern "C"

namespace {
__global__ void k_push_begin(DState* d, int R1) {
  if (d->r >= R1) {
    d->skipped++;
    d->push_ok = 0;
  } else {
    d->push_ok = 1;
  }
  d->rotate = 0;
}
}  // namespace

extern "C" {

pgm_status pgm_deflator_push(pgm_deflator* d, pgm_matrix* a, const double* candidate,
                             int32_t flags, int32_t* accepted) {
  if (!d || !a || !candidate) return PGM_EINVAL;
  pgm_context* ctx = d->ctx;
  cudaSetDevice(ctx->device);
  auto run = [&]() -> Status {
    if (a->ctx != ctx) return einval("pgm_deflator_push: matrix from another context");
    TRY(ensure_min_workspace(ctx, d->R1));
    TRY(ensure_reduction(ctx, 2 * d->R1 + 1, a->ntiles));
    TRY(defl_alloc_vectors(d));
    TRY(set_gstate_idle(ctx));
    DState before;
    CU(cudaMemcpy(&before, d->d, sizeof(DState), cudaMemcpyDeviceToHost));
    TRY(copy_in(ctx, d->u + ctx->lo, candidate, ctx->n, flags));
    const Params P = make_params(ctx, d);
    ctx->cur_defl = d;
    const int R1 = d->R1;
    k_push_begin<<<1, 1, 0, ctx->stream>>>(d->d, R1);
    TRY(launch_sweep<SW_PUSH1>(ctx, P, 0, 0, 0, R1 + 1, false));
    TRY(finish_global<SW_PUSH1>(ctx, P, 0, R1 + 1));
    TRY(launch_sweep<SW_PUSH2>(ctx, P, 0, R1, 0, R1, true));
    TRY(finish_global<SW_PUSH2>(ctx, P, 0, R1));
    TRY(launch_sweep<SW_PUSH3>(ctx, P, 0, R1, 0, 1, false));
    TRY(finish_global<SW_PUSH3>(ctx, P, 0, 1));
    if (ctx->world > 1) TRY(halo_exchange(ctx, HV_U));
    TRY(launch_spmv(ctx, a, P, PushEpi{}, 2 * R1 + 1));
    TRY(finish_global<102>(ctx, P, 0, 2 * R1 + 1));
    k_rotate<false><<<ctx->nsm * 4, 256, 0, ctx->stream>>>(P);
    k_clear_rotate<<<1, 1, 0, ctx->stream>>>(d->d);
    CU(cudaGetLastError());
    DState after;
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaMemcpy(&after, d->d, sizeof(DState), cudaMemcpyDeviceToHost));
    if (accepted) *accepted = after.push_ok && (after.skipped == before.skipped);
    return {};
  };
  Status s = run();
  return s.code ? fail(ctx, s) : PGM_OK;
}

pgm_status pgm_deflator_truncate(pgm_deflator* d) {
  if (!d) return PGM_EINVAL;
  pgm_context* ctx = d->ctx;
  cudaSetDevice(ctx->device);
  auto run = [&]() -> Status {
    TRY(ensure_min_workspace(ctx, d->R1));
    TRY(defl_alloc_vectors(d));
    const Params P = make_params(ctx, d);
    k_truncate_once<<<1, 32, 0, ctx->stream>>>(P);
    k_rotate<false><<<ctx->nsm * 4, 256, 0, ctx->stream>>>(P);
    k_clear_rotate<<<1, 1, 0, ctx->stream>>>(d->d);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(ctx->stream));
    return {};
  };
  Status s = run();
  return s.code ? fail(ctx, s) : PGM_OK;
}

pgm_status pgm_deflator_observe_ritz(pgm_deflator* d, double value) {
  if (!d) return PGM_EINVAL;
  cudaSetDevice(d->ctx->device);
  k_observe<<<1, 1, 0, d->ctx->stream>>>(d->d, value);
  cudaError_t e = cudaStreamSynchronize(d->ctx->stream);
  if (e != cudaSuccess) return fail(d->ctx, Status{PGM_ECUDA, cudaGetErrorString(e)});
  return PGM_OK;
}

pgm_status pgm_deflator_apply(pgm_deflator* d, const double* v, double* w, int32_t flags) {
  if (!d || !v || !w) return PGM_EINVAL;
  pgm_context* ctx = d->ctx;
  cudaSetDevice(ctx->device);
  auto run = [&]() -> Status {
    TRY(ensure_min_workspace(ctx, d->R1));
    TRY(defl_alloc_vectors(d));
    TRY(set_gstate_idle(ctx));
    TRY(copy_in(ctx, d->u + ctx->lo, v, ctx->n, flags));
    const Params P = make_params(ctx, d);
    TRY(launch_sweep<SW_DOTS_U>(ctx, P, 0, 0, 0, d->R1, false));
    TRY(finish_global<SW_DOTS_U>(ctx, P, 0, d->R1));
    TRY(launch_sweep<SW_AXPY_U>(ctx, P, 0, d->R1, 0, 0, false));
    TRY(copy_out(ctx, w, d->u + ctx->lo, ctx->n, flags));
    CU(cudaStreamSynchronize(ctx->stream));
    return {};
  };
  Status s = run();
  return s.code ? fail(ctx, s) : PGM_OK;
}

#if PGM_TAIL_TIMING
// tuning variant only: accumulated reduction-tail stamps of the DCGS2 step
// SpMV (ns): [level-1 chain, level 2, finisher, launches, Ritz x5, finisher
// phases x4]; out must hold 16 values; reset after read
int pgm_debug_tail(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_tail_ns, 16 * sizeof(unsigned long long));
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(g_tail_ns, z, sizeof(z));
  return 0;
}
#endif

pgm_status pgm_set_restart_observer(pgm_context* ctx, pgm_restart_observer cb, void* user) {
  if (!ctx) return PGM_EINVAL;
  ctx->obs = cb;
  ctx->obs_user = user;
  return PGM_OK;
}

pgm_status pgm_restart_basis(pgm_context* ctx, uint32_t j, double* out) {
  if (!ctx || !out) return PGM_EINVAL;
  if (!ctx->in_obs) {
    ctx->err = "pgm_restart_basis: only valid inside a restart observer";
    return PGM_ESTATE;
  }
  if ((int)j >= ctx->obs_steps) {
    ctx->err = "pgm_restart_basis: basis vector " + std::to_string(j) + " of " +
               std::to_string(ctx->obs_steps);
    return PGM_EINVAL;
  }
  double sj = 0.0;
  cudaError_t e = cudaMemcpy(&sj, ctx->s + j, sizeof(double), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess)
    e = cudaMemcpy(out, ctx->V + (size_t)j * ctx->ld + ctx->lo, 8 * ctx->n, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fail(ctx, Status{PGM_ECUDA, cudaGetErrorString(e)});
  for (size_t i = 0; i < ctx->n; ++i) out[i] *= sj;  // v_j = s_j W_j (lazy scale)
  return PGM_OK;
}

pgm_status pgm_restart_hessenberg(pgm_context* ctx, double* out) {
  if (!ctx || !out) return PGM_EINVAL;
  if (!ctx->in_obs) {
    ctx->err = "pgm_restart_hessenberg: only valid inside a restart observer";
    return PGM_ESTATE;
  }
  const size_t hm = (size_t)(ctx->ws_m + 1) * ctx->ws_m;
  cudaError_t e = cudaMemcpy(out, ctx->h_orig, 8 * hm, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fail(ctx, Status{PGM_ECUDA, cudaGetErrorString(e)});
  return PGM_OK;
}

pgm_status pgm_solve(pgm_context* ctx, pgm_matrix* a, pgm_deflator* d, const double* b, double* x,
                     const pgm_gmres_config* cfg, int32_t flags, pgm_report* rep) {
  if (!ctx) return PGM_EINVAL;
  cudaSetDevice(ctx->device);
  Status s = solve_impl(ctx, a, d, b, x, cfg, flags, rep);
  return s.code ? fail(ctx, s) : PGM_OK;
}

void pgm_report_free(pgm_report* rep) {
  if (!rep) return;
  std::free(rep->inner_restart);
  std::free(rep->inner_step);
  std::free(rep->inner_monitored);
  std::free(rep->explicit_residual);
  rep->inner_restart = rep->inner_step = nullptr;
  rep->inner_monitored = rep->explicit_residual = nullptr;
}

}  // extern "C"

// ===========================================================================
// Profiling + device FEM assembly entry points
namespace {

uint64_t bratu_rows_nnz(uint32_t n_e, uint32_t row_begin, uint32_t row_end) {
  const uint32_t na = 2 * n_e + 1, last = na - 1;
  uint64_t total = 0;
  uint32_t lo;
  for (uint64_t v = row_begin; v < row_end; ++v) {
    const uint32_t ix = (uint32_t)(v % na), iy = (uint32_t)((v / na) % na),
                   iz = (uint32_t)(v / ((uint64_t)na * na));
    if (ix == 0 || ix == last || iy == 0 || iy == last)
      total += 1;
    else
      total += (uint64_t)bratu::reach(ix, last, &lo) * bratu::reach(iy, last, &lo) *
               bratu::reach(iz, last, &lo);
  }
  return total;
}

Status bratu_assemble(pgm_context* ctx, uint32_t n_e, double lambda, const double* u,
                      int32_t flags, uint32_t* row_ptr, uint32_t* col_idx, double* values,
                      double* rhs) {
  const uint64_t na = 2ull * n_e + 1;
  if (n_e == 0) return einval("build_mesh: n_e must be positive");
  if (na * na * na != ctx->n_global)
    return einval("bratu: (2 n_e + 1)^3 != context n_global");
  static std::once_flag table_once;
  static cudaError_t table_err = cudaSuccess;
  std::call_once(table_once, [] {
    bratu::Table t;
    bratu::build_table(t);
    table_err = cudaMemcpyToSymbol(bratu::c_tab, &t, sizeof(t));
  });
  CU(table_err);
  const uint32_t rb = ctx->part.row_begin, re = ctx->part.row_end;
  const uint64_t nnz = bratu_rows_nnz(n_e, rb, re);
  if (nnz > 0xFFFFFFFFull) return Status{PGM_EINVAL, "symbolic_pattern: nnz exceeds 32-bit offsets"};
  const bool dev = (flags & PGM_DEVICE_PTRS) != 0;
  const uint32_t nrows = re - rb;
  cudaStream_t st = ctx->stream;
  unsigned* d_rp = nullptr;
  unsigned* d_ci = nullptr;
  double *d_va = nullptr, *d_rhs = nullptr, *d_u = nullptr, *d_f = nullptr;
  void* d_tmp = nullptr;
  struct Guard {
    std::vector<void*> p;
    ~Guard() {
      for (void* q : p) cudaFree(q);
    }
  } guard;
  auto own = [&](auto** ptr, size_t count) -> Status {
    TRY(dalloc(ptr, count));
    guard.p.push_back((void*)*ptr);
    return {};
  };
  if (dev) {
    d_rp = row_ptr;
    d_ci = col_idx;
    d_va = values;
    d_rhs = rhs;
  } else {
    TRY(own(&d_rp, (size_t)nrows + 1));
    TRY(own(&d_ci, nnz));
    TRY(own(&d_va, nnz));
    TRY(own(&d_rhs, nrows));
  }
  if (u) {
    if (dev) {
      d_u = const_cast<double*>(u);
    } else {
      TRY(own(&d_u, ctx->n_global));
      CU(cudaMemcpyAsync(d_u, u, 8 * (size_t)ctx->n_global, cudaMemcpyHostToDevice, st));
    }
  }
  bratu::Mesh M;
  M.n_e = n_e;
  M.na = (uint32_t)na;
  M.plane = na * na;
  M.row_begin = rb;
  M.nrows = nrows;
  M.lambda = lambda;
  const double h_e = 1.0 / n_e;
  M.vol = std::pow(h_e / 2.0, 3);
  M.stiff_sc = h_e / 2.0;
  const unsigned T = 256;
  bratu::k_row_len<<<(unsigned)((nrows + T - 1) / T), T, 0, st>>>(M, d_rp);
  size_t tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, d_rp + 1, d_rp + 1, (int)nrows, st);
  TRY(own((char**)&d_tmp, tmp_bytes));
  cub::DeviceScan::InclusiveSum(d_tmp, tmp_bytes, d_rp + 1, d_rp + 1, (int)nrows, st);
  bratu::k_cols<<<(unsigned)((nrows + T - 1) / T), T, 0, st>>>(M, d_rp, d_ci, d_va);
  const uint32_t zb = (uint32_t)(rb / M.plane), ze = (uint32_t)((re + M.plane - 1) / M.plane);
  const int lay_lo = std::max(0, (int)(zb >> 1) - 1);
  const int lay_hi = std::min((int)n_e - 1, (int)((ze - 1) >> 1));
  const uint64_t per_layer = (uint64_t)n_e * n_e;
  const uint64_t e0 = (uint64_t)lay_lo * per_layer;
  const uint64_t ecount = (uint64_t)(lay_hi - lay_lo + 1) * per_layer;
  TRY(own(&d_f, ecount * 27));
  bratu::k_elem_f<<<(unsigned)((ecount * 27 + T - 1) / T), T, 0, st>>>(M, d_u, d_f, e0, ecount);
  bratu::k_jac_values<<<(unsigned)(((uint64_t)nrows * 32 + T - 1) / T), T, 0, st>>>(M, d_rp, d_f,
                                                                                   e0, d_va);
  bratu::k_residual_rhs<<<(unsigned)((nrows + T - 1) / T), T, 0, st>>>(M, d_u, d_f, e0, d_rhs);
  CU(cudaGetLastError());
  if (!dev) {
    CU(cudaMemcpyAsync(row_ptr, d_rp, 4 * ((size_t)nrows + 1), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(col_idx, d_ci, 4 * nnz, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(values, d_va, 8 * nnz, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(rhs, d_rhs, 8 * (size_t)nrows, cudaMemcpyDeviceToHost, st));
  }
  CU(cudaStreamSynchronize(st));
  return {};
}

}  // namespace

extern "C" {

pgm_status pgm_peer_export(pgm_context* ctx, void* out128) {
  if (!ctx || !out128) return PGM_EINVAL;
  if (ctx->world < 2 || !ctx->pbuf)
    return fail(ctx, einval("pgm_peer_export: needs a world > 1 context"));
  cudaSetDevice(ctx->device);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ctx->pbuf);
  if (e != cudaSuccess) return fail(ctx, Status{PGM_ECUDA, std::string("cudaIpcGetMemHandle: ") +
                                                             cudaGetErrorString(e)});
  std::memset(out128, 0, 128);
  std::memcpy(out128, &h, sizeof(h));
  return PGM_OK;
}

pgm_status pgm_peer_import(pgm_context* ctx, const void* all) {
  if (!ctx || !all) return PGM_EINVAL;
  if (ctx->world < 2 || !ctx->pbuf || ctx->loop)
    return fail(ctx, einval("pgm_peer_import: needs a world > 1 NCCL context"));
  if (ctx->det)
    return fail(ctx, einval("pgm_peer_import: the deterministic mode gathers plane partials "
                            "(NCCL); the fused peer allreduce is not available in it"));
  const char* ml = std::getenv("CUDA_MODULE_LOADING");
  if (!ml || std::string(ml) != "EAGER")
    return fail(ctx, einval("pgm_peer_import: set CUDA_MODULE_LOADING=EAGER before CUDA starts "
                            "(lazy module loading can stall spinning peer kernels)"));
  cudaSetDevice(ctx->device);
  std::vector<char*> bufs(ctx->world);
  for (int q = 0; q < ctx->world; ++q) {
    if (q == ctx->rank) {
      bufs[q] = ctx->pbuf;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(all) + 128 * (size_t)q, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return fail(ctx, Status{PGM_ECUDA, std::string("cudaIpcOpenMemHandle: ") +
                                             cudaGetErrorString(e)});
    ctx->peer_opened.push_back(p);
    bufs[q] = static_cast<char*>(p);
  }
  Status s = peer_set_tables(ctx, bufs);
  return s.code ? fail(ctx, s) : PGM_OK;
}

pgm_status pgm_nccl_unique_id(void* out128) {
  if (!out128) return PGM_EINVAL;
  if (!nccl_lite::available() || nccl_lite::get_unique_id(out128) != 0) {
    g_tls_err = "ncclGetUniqueId unavailable";
    return PGM_ENCCL;
  }
  return PGM_OK;
}

pgm_status pgm_context_set_profiling(pgm_context* ctx, int32_t on) {
  if (!ctx) return PGM_EINVAL;
  ctx->prof_on = on != 0;
  return PGM_OK;
}

uint32_t pgm_context_profile(pgm_context* ctx, uint32_t* cls, uint32_t* cycle, uint32_t* k,
                             float* ms, uint32_t cap) {
  if (!ctx) return 0;
  cudaStreamSynchronize(ctx->stream);
  const uint32_t n = (uint32_t)std::min<size_t>(cap, ctx->prof.size());
  for (uint32_t i = 0; i < n; ++i) {
    const auto& r = ctx->prof[i];
    if (cls) cls[i] = r.cls;
    if (cycle) cycle[i] = r.cyc;
    if (k) k[i] = r.k;
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    if (ms) ms[i] = t;
  }
  return n;
}

pgm_status pgm_bratu_nnz(const pgm_context* ctx, uint32_t n_e, uint64_t* nnz) {
  if (!nnz || n_e == 0) return PGM_EINVAL;
  const uint64_t na = 2ull * n_e + 1;
  uint32_t rb = 0, re = (uint32_t)(na * na * na);
  if (ctx) {
    rb = ctx->part.row_begin;
    re = ctx->part.row_end;
  }
  *nnz = bratu_rows_nnz(n_e, rb, re);
  return PGM_OK;
}

pgm_status pgm_bratu_assemble(pgm_context* ctx, uint32_t n_e, double lambda, const double* u,
                              int32_t flags, uint32_t* row_ptr, uint32_t* col_idx, double* values,
                              double* rhs) {
  if (!ctx || !row_ptr || !col_idx || !values || !rhs) return PGM_EINVAL;
  cudaSetDevice(ctx->device);
  Status s = bratu_assemble(ctx, n_e, lambda, u, flags, row_ptr, col_idx, values, rhs);
  return s.code ? fail(ctx, s) : PGM_OK;
}

}  // extern "C"

// ===========================================================================
// Newton driver (newton.hpp:15-54, newton.cpp:31-97), device-resident: u, the
// Jacobian (pattern built once, values rewritten in place, assembly.cpp:253),
// -R(u), delta and the deflation basis stay in HBM; the host reads two
// scalars per Newton iteration (||R||_2, ||delta||_inf) plus the solve's
// per-restart status word.
namespace {

Status newton_scalars(pgm_context* ctx, const double* rhs_own, const double* delta_own,
                      double* u_own, double* res_norm, double* step) {
  // red_out[0] = sum rhs^2 (global), red_out[1 + q] = max|delta| of rank q
  const int nv = 1 + ctx->world;
  TRY(ensure_reduction(ctx, nv));
  const int G = ctx->nsm * 4;
  k_newton_partials<<<G, 256, 0, ctx->stream>>>(rhs_own, delta_own, u_own, (int)ctx->n,
                                                ctx->part_buf);
  k_newton_final<<<1, 256, 0, ctx->stream>>>(ctx->part_buf, G, ctx->red_out, nv, ctx->rank);
  ctx->launches += 2;
  CU(cudaGetLastError());
  if (ctx->coll) TRY(allreduce_red(ctx, nv));
  double h[1 + 64];
  CU(cudaMemcpyAsync(h, ctx->red_out, 8 * (size_t)nv, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (res_norm) *res_norm = std::sqrt(h[0]);
  if (step) {
    double m = 0.0;
    for (int q = 0; q < ctx->world; ++q) m = std::max(m, h[1 + q]);
    *step = m;
  }
  return {};
}

Status newton_impl(pgm_context* ctx, uint32_t n_e, double lambda, double* u, int32_t flags,
                   const pgm_newton_config* cfg, pgm_newton_report* rep) {
  if (!cfg) return einval("newton: null config");
  if (cfg->max_iters == 0) return einval("newton: max_iters must be positive");
  if (ctx->world > 64) return einval("newton: world > 64");
  const uint64_t na = 2ull * n_e + 1;
  if (n_e == 0 || na * na * na != ctx->n_global)
    return einval("newton: (2 n_e + 1)^3 != context n_global");
  const size_t N = ctx->n_global, n = ctx->n;
  const size_t rb = ctx->part.row_begin;
  uint64_t nnz = 0;
  nnz = bratu_rows_nnz(n_e, ctx->part.row_begin, ctx->part.row_end);
  struct Bufs {
    double *ug = nullptr, *va = nullptr, *rhs = nullptr, *delta = nullptr;
    unsigned *rp = nullptr, *ci = nullptr;
    pgm_matrix* J = nullptr;
    pgm_deflator* D = nullptr;
    ~Bufs() {
      dfree(ug);
      dfree(va);
      dfree(rhs);
      dfree(delta);
      dfree(rp);
      dfree(ci);
      if (J) pgm_matrix_destroy(J);
      if (D) pgm_deflator_destroy(D);
    }
  } B;
  // u: global iterate (every rank holds the full-size vector; only its
  // [halo_lo | own | halo_hi] window is kept current, which is all the
  // assembly of its rows reads)
  TRY(dalloc(&B.ug, N));
  TRY(dalloc(&B.va, nnz));
  TRY(dalloc(&B.rhs, n));
  TRY(dalloc(&B.delta, n));
  TRY(dalloc(&B.rp, n + 1));
  TRY(dalloc(&B.ci, nnz));
  CU(cudaMemcpyAsync(B.ug, u, 8 * N,
                     (flags & PGM_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     ctx->stream));
  double* u_own = B.ug + rb;
  ctx->halo_ptr = B.ug + rb - ctx->lo;  // ctx layout [halo_lo | own | halo_hi]
  if (cfg->use_deflation) {
    const pgm_status st = pgm_deflator_create(ctx, &cfg->deflation, &B.D);
    if (st != PGM_OK) return Status{st, ctx->err};
  }
  std::vector<double> stages;
  if (cfg->continuation && cfg->continuation_steps > 1) {
    for (uint32_t q = 1; q <= cfg->continuation_steps; ++q)
      stages.push_back(lambda * double(q) / double(cfg->continuation_steps));
  } else {
    stages.push_back(lambda);
  }
  std::vector<pgm_newton_record> recs;
  const auto t0 = std::chrono::steady_clock::now();
  uint32_t iter = 0;
  uint64_t total_inner = 0;
  double final_residual = 0.0, final_update = 0.0;
  bool converged = true;
  for (double lam : stages) {
    bool stage_done = false;
    for (uint32_t it = 0; it < cfg->max_iters; ++it) {
      // assemble_residual + assemble_jacobian (newton.cpp:53-57): rhs = -R(u)
      TRY(bratu_assemble(ctx, n_e, lam, B.ug, PGM_DEVICE_PTRS, B.rp, B.ci, B.va, B.rhs));
      double res_norm = 0.0;
      TRY(newton_scalars(ctx, B.rhs, nullptr, nullptr, &res_norm, nullptr));
      if (!B.J) {
        pgm_csr_view v{(uint32_t)n, nnz, B.rp, B.ci, B.va};
        TRY(matrix_upload(ctx, &v, PGM_DEVICE_PTRS, &B.J));
      } else {
        const pgm_status st = pgm_matrix_update_values(B.J, B.va, PGM_DEVICE_PTRS);
        if (st != PGM_OK) return Status{st, ctx->err};
      }
      CU(cudaMemsetAsync(B.delta, 0, 8 * n, ctx->stream));
      if (B.D) {
        const pgm_status st = pgm_deflator_reset(B.D);  // newton.cpp:62
        if (st != PGM_OK) return Status{st, ctx->err};
      }
      pgm_report lin{};
      Status ss = solve_impl(ctx, B.J, B.D, B.rhs, B.delta, &cfg->gmres, PGM_DEVICE_PTRS, &lin);
      const uint32_t lin_restarts = lin.restarts;
      const uint64_t lin_inner = lin.total_inner;
      pgm_report_free(&lin);
      TRY(ss);
      // u += delta, ||delta||_inf (newton.cpp:72-73)
      double step = 0.0;
      TRY(newton_scalars(ctx, nullptr, B.delta, u_own, nullptr, &step));
      if (ctx->world > 1) TRY(halo_exchange(ctx, HV_PTR));
      ++iter;
      recs.push_back(pgm_newton_record{iter, lam, step, res_norm, lin_restarts, lin_inner});
      total_inner += lin_inner;
      final_update = step;
      final_residual = res_norm;
      if (step <= cfg->update_tol) {
        stage_done = true;
        break;
      }
    }
    if (!stage_done) {
      converged = false;
      break;
    }
  }
  if (converged) {
    TRY(bratu_assemble(ctx, n_e, stages.back(), B.ug, PGM_DEVICE_PTRS, B.rp, B.ci, B.va, B.rhs));
    TRY(newton_scalars(ctx, B.rhs, nullptr, nullptr, &final_residual, nullptr));
  }
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  // u out: every rank writes its owned rows (the caller's global vector)
  CU(cudaMemcpyAsync(u + rb, u_own, 8 * n,
                     (flags & PGM_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->halo_ptr = nullptr;
  if (rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->n_iters = (uint32_t)recs.size();
    rep->iters = (pgm_newton_record*)std::malloc(sizeof(pgm_newton_record) *
                                                 std::max<size_t>(1, recs.size()));
    if (!recs.empty()) std::memcpy(rep->iters, recs.data(), sizeof(pgm_newton_record) * recs.size());
    rep->converged = converged;
    rep->final_residual = final_residual;
    rep->final_update = final_update;
    rep->total_inner = total_inner;
    rep->seconds = secs;
  }
  return {};
}

}  // namespace

extern "C" {

pgm_status pgm_newton_solve(pgm_context* ctx, uint32_t n_e, double lambda, double* u,
                            int32_t flags, const pgm_newton_config* cfg, pgm_newton_report* rep) {
  if (!ctx || !u) return PGM_EINVAL;
  cudaSetDevice(ctx->device);
  Status s = newton_impl(ctx, n_e, lambda, u, flags, cfg, rep);
  ctx->halo_ptr = nullptr;
  return s.code ? fail(ctx, s) : PGM_OK;
}

void pgm_newton_report_free(pgm_newton_report* rep) {
  if (!rep) return;
  std::free(rep->iters);
  rep->iters = nullptr;
  rep->n_iters = 0;
}

}  // extern "C"
