// Device kernels of libpgmres (sm_100a).  All fp64, HBM-bandwidth bound.
//
//   k_spmv<Epi> ... SELL-32 sparse matrix-vector product, one lane per row,
//                   ascending-column accumulation without FMA contraction
//                   (bit-identical to sparse.cpp:9-19), fused with a per-tile
//                   epilogue in natural row order (vector updates + the dot
//                   products of the following reduction) and the grid
//                   reduction + scalar finisher.
//   k_sweep<MODE>.. one streaming pass over a block of basis vectors:
//                   out = in + sum_l a_l P_l (+ second set), then dot products
//                   of out with a set of vectors (staged in smem when it is
//                   the set just streamed), then the grid reduction.
//   k_ritz ........ restart-time small dense Ritz iterations on H (one block).
//   k_rotate ...... U <- U Q, AU <- AU Q after truncation; history record.
#pragma once

#include <math.h>

#include <type_traits>

#include <cub/cub.cuh>

#include "common.cuh"
#include "finish.cuh"
#include "tma.cuh"

namespace pgm {

// ---------------------------------------------------------------------------
// SELL-32 with a per-tile length sort (sigma = TILE).
struct Sell {
  const unsigned long long* sptr;  // [nslices + 1] entry offsets (multiples of 32)
  const unsigned* lane_len;        // [nslices * 32] true row length
  const unsigned short* lane_row;  // [nslices * 32] row within tile, 0xFFFF = empty lane
  const double* val;
  const unsigned* col;             // local column (index into the padded x buffer)
  const unsigned short* col16;     // compressed: 16-bit column deltas (same entry layout)
  const unsigned* lane_base;       // compressed: first column of the lane's row
  int ntiles;
  int n;
};

// Slice layout: entry (lane, t) of a slice lives at base + (t/4)*128 + lane*4 + t%4,
// so each lane reads 4 consecutive column ids (one uint4) and 4 values (two
// double2) per group: every warp load instruction moves a contiguous 512 B or
// 1 KB block.  Slice lengths are padded to a multiple of 4.
// C16: column ids stored as 16-bit deltas to the previous entry of the row
// (first entry: delta 0 from lane_base), 8 B per 4 entries instead of 16 B:
// 10 instead of 12 bytes per nonzero.  Used when every delta of the matrix
// fits (columns ascending, gaps < 65536: all z-slab meshes up to n_e = 127).
template <bool C16>
__device__ __forceinline__ void spmv_tile(const Sell& A, const double* __restrict__ x, int tile,
                                          double* ys) {
  using CT = typename std::conditional<C16, uint2, uint4>::type;
  constexpr int UG = SPMV_UNROLL / 4;  // 4-entry groups in flight per lane
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  // Rows are sorted by length inside the tile, so slice lengths fall with the
  // slice index: warp w takes slices w and SPT-1-w (long + short), which
  // balances the warps ahead of the epilogue barrier.
  for (int it = 0; it < SPT / nw; ++it) {
    const int sl = (it & 1) ? (SPT - 1 - (it >> 1) * nw - warp) : ((it >> 1) * nw + warp);
    const size_t s = (size_t)tile * SPT + sl;
    const unsigned long long base = A.sptr[s];
    const int L4 = (int)((A.sptr[s + 1] - base) >> 7);
    if (L4 == 0) continue;
#if PGM_SPMV_PREFETCH
    // stream the slice (values + column ids) into L2 through the TMA engine;
    // the lane loads below then mostly hit L2.  The warp's first slice was
    // prefetched ahead of the PDL wait (k_spmv).
    if (sl != warp || !PGM_SPMV_EARLY_PF) {
      if (lane == 0) tma_prefetch_l2(A.val + base, (uint32_t)L4 * 128u * 8u);
      if (lane == 1) {
        if (C16) tma_prefetch_l2(A.col16 + base, (uint32_t)L4 * 128u * 2u);
        else tma_prefetch_l2(A.col + base, (uint32_t)L4 * 128u * 4u);
      }
    }
#endif
    const int len = (int)A.lane_len[s * 32 + lane];
    const unsigned short ro = A.lane_row[s * 32 + lane];
    const CT* cp = C16 ? reinterpret_cast<const CT*>(A.col16 + base) + lane
                       : reinterpret_cast<const CT*>(A.col + base) + lane;
    unsigned prev = C16 ? A.lane_base[s * 32 + lane] : 0u;
    const double2* vp = reinterpret_cast<const double2*>(A.val + base) + 2 * lane;
    double acc = 0.0;
    // software pipeline: the streaming loads of group g+UG are in flight while
    // the x gathers and the accumulation of group g run
    CT c[UG];
    double2 va[UG], vb[UG];
#pragma unroll
    for (int u = 0; u < UG; ++u) {
      if (u < L4) {
        c[u] = __ldcs(cp + (size_t)u * 32);
        va[u] = __ldcs(vp + (size_t)u * 64);
        vb[u] = __ldcs(vp + (size_t)u * 64 + 1);
      }
    }
    for (int g = 0; g < L4; g += UG) {
      CT cn[UG];
      double2 van[UG], vbn[UG];
#pragma unroll
      for (int u = 0; u < UG; ++u) {
        if (g + UG + u < L4) {
          cn[u] = __ldcs(cp + (size_t)(g + UG + u) * 32);
          van[u] = __ldcs(vp + (size_t)(g + UG + u) * 64);
          vbn[u] = __ldcs(vp + (size_t)(g + UG + u) * 64 + 1);
        }
      }
      double xv[UG][4];
#pragma unroll
      for (int u = 0; u < UG; ++u) {
        const int t = (g + u) * 4;
        unsigned c0, c1, c2, c3;
        if constexpr (C16) {
          c0 = prev + (c[u].x & 0xFFFFu);
          c1 = c0 + (c[u].x >> 16);
          c2 = c1 + (c[u].y & 0xFFFFu);
          c3 = c2 + (c[u].y >> 16);
          prev = c3;
        } else {
          c0 = c[u].x;
          c1 = c[u].y;
          c2 = c[u].z;
          c3 = c[u].w;
        }
        xv[u][0] = (t + 0 < len) ? __ldg(x + c0) : 0.0;
        xv[u][1] = (t + 1 < len) ? __ldg(x + c1) : 0.0;
        xv[u][2] = (t + 2 < len) ? __ldg(x + c2) : 0.0;
        xv[u][3] = (t + 3 < len) ? __ldg(x + c3) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UG; ++u) {
        const int t = (g + u) * 4;
        if (t + 0 < len) acc = __dadd_rn(acc, __dmul_rn(va[u].x, xv[u][0]));
        if (t + 1 < len) acc = __dadd_rn(acc, __dmul_rn(va[u].y, xv[u][1]));
        if (t + 2 < len) acc = __dadd_rn(acc, __dmul_rn(vb[u].x, xv[u][2]));
        if (t + 3 < len) acc = __dadd_rn(acc, __dmul_rn(vb[u].y, xv[u][3]));
      }
#pragma unroll
      for (int u = 0; u < UG; ++u) {
        c[u] = cn[u];
        va[u] = van[u];
        vb[u] = vbn[u];
      }
    }
    if (ro != 0xFFFF) ys[ro] = acc;
  }
}

// ---- warp-level row-chunk dot products ---------------------------------------
// A warp owns 32 consecutive rows (lane = row).  Dot products of the row
// values o with a set of vectors are formed 16 values at a time: every lane
// writes its 16 products into a per-warp transposed tile tp[16][33] (smem),
// then lane pairs (v, v+16) sum the 32 products of value v in a fixed order
// and the lower lane keeps the running sum in register slot v / 16.
// Deterministic (fixed order everywhere) and barrier-free (only __syncwarp).
constexpr int TPR = 16;                 // values per batch
constexpr int TPS = 33;                 // padded tile row (doubles)
constexpr int TP_DOUBLES = TPR * TPS;   // per-warp tile
constexpr int NVL = 9;                  // accumulator slots: up to 144 values

__device__ __forceinline__ double tp_sum16(const double* tp, int lane) {
  const double* p = tp + (lane & 15) * TPS + (lane >> 4) * 16;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int q = 0; q < 16; q += 4) {
    a0 += p[q];
    a1 += p[q + 1];
    a2 += p[q + 2];
    a3 += p[q + 3];
  }
  double s = (a0 + a1) + (a2 + a3);
  s += __shfl_xor_sync(0xffffffffu, s, 16);
  return s;
}

// Products for values [v0, v0 + cnt) supplied by prod(v); accumulated in slot.
template <class F>
__device__ __forceinline__ void tp_batch(double* tp, double& slot_acc, int v0, int cnt, int lane,
                                         F prod) {
  double p[TPR];
#pragma unroll
  for (int j = 0; j < TPR; ++j) p[j] = (j < cnt) ? prod(v0 + j) : 0.0;
  __syncwarp();  // scheduling fence: all loads of the batch issued before the stores
#pragma unroll
  for (int j = 0; j < TPR; ++j)
    if (j < cnt) tp[j * TPS + lane] = p[j];
  __syncwarp();
  const double s = tp_sum16(tp, lane);
  if (lane < cnt) slot_acc += s;
  __syncwarp();
}

// All nv values: prod(v) for v in [0, nv).
template <class F>
__device__ __forceinline__ void tp_all(double* tp, double (&acc)[NVL], int nv, int lane, F prod) {
#pragma unroll
  for (int sl = 0; sl < NVL; ++sl) {
    const int v0 = sl * TPR;
    if (v0 < nv) tp_batch(tp, acc[sl], v0, min(TPR, nv - v0), lane, prod);
  }
}

// Block combine of the per-warp accumulators (fixed warp order) into bvals[nv].
__device__ __forceinline__ void warps_to_block(const double (&acc)[NVL], int nv, double* wacc,
                                               double* bvals) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane < TPR) {
#pragma unroll
    for (int sl = 0; sl < NVL; ++sl) {
      const int v = sl * TPR + lane;
      if (v < nv) wacc[warp * (NVL * TPR) + v] = acc[sl];
    }
  }
  __syncthreads();
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += wacc[w * (NVL * TPR) + v];
    bvals[v] = s;
  }
  __syncthreads();
}

// ---- SpMV epilogues ---------------------------------------------------------------
// Each is called once per 32-row chunk of the tile by one warp: grow = global
// own-row index of this lane's row, yv = (A x)[grow].

// y = A x, nothing else (pgm_spmv).
struct PlainEpi {
  const double* xin;
  double* y;  // own region
  __device__ bool skip(const Params&) const { return false; }
  __device__ int nvals(const Params&) const { return 0; }
  __device__ void prologue(const Params&, double*) const {}
  __device__ void chunk(const Params&, int grow, bool ok, double yv, double*, double (&)[NVL],
                        const double*) const {
    if (ok) y[grow] = yv;
  }
  __device__ void finish(const Params&, const double*) const {}
};

// Arnoldi step k: w = s_k A W_k + AU c  (= A M^{-1} v_k, deflation folded through
// the cached AU), stored as W_{k+1}; CGS2 pass-1 dots W_l . w (sweep A).
struct StepEpi {
  int k;
  __device__ bool skip(const Params& P) const { return !P.g->active; }
  __device__ int nvals(const Params&) const { return k + 1; }
  __device__ void prologue(const Params& P, double* sm) const {
    // sm[0] = s_k, sm[1..r] = c
    if (threadIdx.x == 0) sm[0] = P.s[k];
    for (int l = threadIdx.x; l < P.d->r; l += blockDim.x) sm[1 + l] = P.c[l];
  }
  __device__ void chunk(const Params& P, int grow, bool ok, double yv, double* tp,
                        double (&acc)[NVL], const double* sm) const {
    const int lane = threadIdx.x & 31;
    const int r = P.d->r;
    const size_t ld = P.ld;
    const double* own = P.V + P.lo + grow;
    double y = 0.0;
    if (ok) {
      y = sm[0] * yv;
      const double* au = P.AU + P.lo + grow;
      for (int l = 0; l < r; ++l) y += sm[1 + l] * __ldg(au + (size_t)l * ld);
      P.V[(size_t)(k + 1) * ld + P.lo + grow] = y;
    }
    tp_all(tp, acc, k + 1, lane,
           [&](int v) { return ok ? __ldg(own + (size_t)v * ld) * y : 0.0; });
  }
  __device__ void finish(const Params& P, const double* red) const { fin_step_spmv(P, k, red); }
};

// DCGS2 step k: y = s_k A W_k + AU c (W_k = lagged u_k for k >= 1, s_k = 1),
// stored as W_{k+1}; ONE reduction: [W_l . y (nb), W_l . u (k), u.u, u.y,
// U_j . y (r)], nb = max(k, 1) (finish.cuh fin_dcgs2).
struct DStepEpi {
  int k;
  __device__ bool skip(const Params& P) const { return !P.g->active; }
  __device__ int nvals(const Params& P) const { return (k > 0 ? k : 1) + k + 2 + P.d->r; }
  __device__ void prologue(const Params& P, double* sm) const {
    if (threadIdx.x == 0) sm[0] = P.s[k];
    for (int l = threadIdx.x; l < P.d->r; l += blockDim.x) sm[1 + l] = P.c[l];
  }
  __device__ void chunk(const Params&, int, bool, double, double*, double (&)[NVL],
                        const double*) const {}
  __device__ void finish(const Params& P, const double* red) const { fin_dcgs2(P, k, red); }
};

// Explicit residual r = b - A x into W_0; dots ||r||^2 and U_l . r.
struct ResidualEpi {
  int initial;
  __device__ bool skip(const Params& P) const { return P.g->error != 0 || (!initial && P.g->done); }
  __device__ int nvals(const Params& P) const { return 1 + P.d->r; }
  __device__ void prologue(const Params&, double*) const {}
  __device__ void chunk(const Params& P, int grow, bool ok, double yv, double* tp,
                        double (&acc)[NVL], const double*) const {
    const int lane = threadIdx.x & 31;
    double rv = 0.0;
    if (ok) {
      rv = P.b[P.lo + grow] + (-yv);  // r = b; r += -1 * (A x)   (gmres.cpp:143-145)
      P.V[P.lo + grow] = rv;
    }
    const double* u = P.U + P.lo + grow;
    const size_t ld = P.ld;
    tp_all(tp, acc, 1 + P.d->r, lane, [&](int v) {
      if (!ok) return 0.0;
      return v == 0 ? rv * rv : __ldg(u + (size_t)(v - 1) * ld) * rv;
    });
  }
  __device__ void finish(const Params& P, const double* red) const {
    fin_residual(P, red, initial != 0);
  }
};

// push_vector tail: U_j = u / ||u||, AU_j = A U_j, T row/column dots.
struct PushEpi {
  __device__ bool skip(const Params& P) const { return !P.d->push_ok; }
  __device__ int nvals(const Params& P) const { return 2 * P.d->r + 1; }
  __device__ void prologue(const Params& P, double* sm) const {
    if (threadIdx.x == 0) sm[0] = P.d->pscale;
  }
  __device__ void chunk(const Params& P, int grow, bool ok, double yv, double* tp,
                        double (&acc)[NVL], const double* sm) const {
    const int lane = threadIdx.x & 31;
    const int j = P.d->r;
    const size_t ld = P.ld;
    const double ps = sm[0];
    double un = 0.0, an = 0.0;
    if (ok) {
      un = P.u[P.lo + grow] * ps;
      an = yv * ps;
      P.U[(size_t)j * ld + P.lo + grow] = un;
      P.AU[(size_t)j * ld + P.lo + grow] = an;
    }
    const double* U = P.U + P.lo + grow;
    const double* AU = P.AU + P.lo + grow;
    tp_all(tp, acc, 2 * j + 1, lane, [&](int v) {
      if (!ok) return 0.0;
      if (v < j) return __ldg(U + (size_t)v * ld) * an;   // U_l . AU_j
      if (v == j) return un * an;                          // U_j . AU_j
      return un * __ldg(AU + (size_t)(v - j - 1) * ld);    // U_j . AU_l
    });
  }
  __device__ void finish(const Params& P, const double* red) const {
    if (threadIdx.x == 0) fin_push_spmv(P, red);
  }
};

template <class Epi>
__device__ __forceinline__ const double* epi_input(const Params& P, const Epi& E);
template <>
__device__ __forceinline__ const double* epi_input(const Params&, const PlainEpi& E) {
  return E.xin;
}
template <>
__device__ __forceinline__ const double* epi_input(const Params& P, const StepEpi& E) {
  return P.V + (size_t)E.k * P.ld;
}
template <>
__device__ __forceinline__ const double* epi_input(const Params& P, const DStepEpi& E) {
  return P.V + (size_t)E.k * P.ld;
}
template <>
__device__ __forceinline__ const double* epi_input(const Params& P, const ResidualEpi&) {
  return P.x;
}
template <>
__device__ __forceinline__ const double* epi_input(const Params& P, const PushEpi&) {
  return P.u;
}

constexpr int EPI_SMALL = 8 + 64;  // prologue scratch (doubles)
constexpr int SPMV_WARPS = SPMV_THREADS / 32;

__host__ __device__ constexpr size_t spmv_step_smem_doubles(int nv) {
  return (size_t)EPI_SMALL + TILE + 2 * (size_t)nv + 2;
}
__host__ __device__ constexpr size_t spmv_smem_doubles(int nv) {
  return (size_t)EPI_SMALL + TILE + (size_t)SPMV_WARPS * TP_DOUBLES +
         (size_t)SPMV_WARPS * NVL * TPR + 2 * (size_t)nv + 2;
}

// One 512-row tile per block: SELL SpMV into smem, then every warp runs the
// epilogue on its 64 rows (2 x 32-row chunks), then the grid reduction.
// dynamic smem: [small | ys TILE | tp per warp | wacc | bvals nv | red nv]
// Tile segments of one launch of a halo-overlapped SpMV (world > 1): block b
// runs tile b0 + b for b < len0, else tile b1 + (b - len0); the reduction
// spans all ntiles tiles of the interior and boundary launches.
struct SpmvSeg {
  int b0, len0, b1;
};

template <class Epi, bool SEG, bool C16>
__global__ void __launch_bounds__(SPMV_THREADS, SPMV_MINB) k_spmv(Sell A, Params P, Epi E,
                                                                 SpmvSeg sg) {
  extern __shared__ double sm[];
  const int tile = SEG ? ((int)blockIdx.x < sg.len0 ? sg.b0 + (int)blockIdx.x
                                                    : sg.b1 + ((int)blockIdx.x - sg.len0))
                       : (int)blockIdx.x;
  // A step SpMV of a cycle that already stopped exits before touching the
  // matrix: g->active is written by pass B's finisher, >= 2 kernels back
  // (common.cuh PDL rule), so it is final here.
  if ((std::is_same<Epi, StepEpi>::value || std::is_same<Epi, DStepEpi>::value) &&
      !*(volatile const int*)&P.g->active)
    return;
#if PGM_SPMV_PREFETCH && PGM_SPMV_EARLY_PF
  {
    // L2 prefetch of this warp's first slice (values + column ids).  The
    // matrix is never written during a solve, so this runs ahead of the PDL
    // wait, overlapping the previous kernel's reduction tail.  (Prefetching
    // every slice up front overflows the L2 share of the SM: slower.)
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    {
      const int sl = w;
      const size_t sidx = (size_t)tile * SPT + sl;
      const unsigned long long base = A.sptr[sidx];
      const uint32_t L4 = (uint32_t)((A.sptr[sidx + 1] - base) >> 7);
      if (L4 > 0 && ln == 0) tma_prefetch_l2(A.val + base, L4 * 128u * 8u);
      if (L4 > 0 && ln == 1) {
        if (C16) tma_prefetch_l2(A.col16 + base, L4 * 128u * 2u);
        else tma_prefetch_l2(A.col + base, L4 * 128u * 4u);
      }
    }
  }
#endif
  pdl_wait();
  if (E.skip(P)) return;
  const int nv = E.nvals(P);
  double* small = sm;
  double* ys = sm + EPI_SMALL;
  // the step epilogue needs no transpose tiles: [small | ys | bvals | red]
  constexpr bool STEP = std::is_same<Epi, StepEpi>::value || std::is_same<Epi, DStepEpi>::value;
  double* tp = ys + TILE + (threadIdx.x >> 5) * TP_DOUBLES;
  double* wacc = ys + TILE + SPMV_WARPS * TP_DOUBLES;
  double* bvals = STEP ? ys + TILE * (std::is_same<Epi, DStepEpi>::value ? 2 : 1)
                      : wacc + SPMV_WARPS * NVL * TPR;
  double* red = bvals + nv;
  E.prologue(P, small);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* x = epi_input(P, E);
  // exactly one tile per block (grid = ntiles): the epilogue accumulators are
  // only live after the SpMV part, which keeps the SpMV loop's registers low
  spmv_tile<C16>(A, x, tile, ys);
  __syncthreads();
  if constexpr (std::is_same<Epi, DStepEpi>::value) {
    // (1) y per row -> W_{k+1}, ys; u = W_k rows -> us.  (2) one stream over
    // each W_l (l < k) gives both W_l . y and W_l . u; U_j . y; u.u and u.y
    // from smem.  Warp w owns vectors w, w + 8, ...
    const int k = E.k;
    const int r = P.d->r;
    const size_t ld = P.ld;
    const int row0 = tile * TILE;
    const int rows = min(TILE, A.n - row0);
    double* us = ys + TILE;
    double* wnext = P.V + (size_t)(k + 1) * ld + P.lo + row0;
    const double* uk = P.V + (size_t)k * ld + P.lo + row0;
    const double* au0 = P.AU + P.lo + row0;
    for (int i = threadIdx.x; i < TILE; i += SPMV_THREADS) {
      double y = 0.0, u = 0.0;
      if (i < rows) {
        y = small[0] * ys[i];
        for (int l = 0; l < r; ++l) y += small[1 + l] * __ldg(au0 + (size_t)l * ld + i);
        wnext[i] = y;
        u = uk[i];
      }
      ys[i] = y;
      us[i] = u;
    }
    __syncthreads();
    const int nb = k > 0 ? k : 1;
    const double* v0 = P.V + P.lo + row0;
    const int nvec = nb + r + 1;  // W_l (l < nb), U_j, and one slot for u.u / u.y
    for (int q = warp; q < nvec; q += SPMV_WARPS) {
      double ay = 0.0, au = 0.0;
      if (q < nb) {
        const double* v = v0 + (size_t)q * ld + lane;
        if (rows == TILE) {  // full tile: all 16 loads in flight, then the products
          double t[TILE / 32];
#pragma unroll
          for (int i = 0; i < TILE / 32; ++i) t[i] = __ldg(v + 32 * i);
#pragma unroll
          for (int i = 0; i < TILE / 32; ++i) {
            ay += t[i] * ys[lane + 32 * i];
            au += t[i] * us[lane + 32 * i];
          }
        } else {
          for (int t = 0; t < TILE / 32; ++t) {
            if (lane + 32 * t < rows) {
              const double w = __ldg(v + 32 * t);
              ay += w * ys[lane + 32 * t];
              au += w * us[lane + 32 * t];
            }
          }
        }
        ay = warp_sum(ay);
        au = warp_sum(au);
        if (lane == 0) {
          bvals[q] = ay;
          if (q < k) bvals[nb + q] = au;
        }
      } else if (q < nb + r) {
        const double* v = P.U + (size_t)(q - nb) * ld + P.lo + row0 + lane;
        if (rows == TILE) {
          double t[TILE / 32];
#pragma unroll
          for (int i = 0; i < TILE / 32; ++i) t[i] = __ldg(v + 32 * i);
#pragma unroll
          for (int i = 0; i < TILE / 32; ++i) ay += t[i] * ys[lane + 32 * i];
        } else {
          for (int t = 0; t < TILE / 32; ++t)
            if (lane + 32 * t < rows) ay += __ldg(v + 32 * t) * ys[lane + 32 * t];
        }
        ay = warp_sum(ay);
        if (lane == 0) bvals[nb + k + 2 + (q - nb)] = ay;
      } else {
        for (int t = 0; t < TILE / 32; ++t) {
          const double u = us[lane + 32 * t];
          ay += u * u;
          au += u * ys[lane + 32 * t];
        }
        ay = warp_sum(ay);
        au = warp_sum(au);
        if (lane == 0) {
          bvals[nb + k] = ay;
          bvals[nb + k + 1] = au;
        }
      }
    }
    pdl_trigger();
    __syncthreads();
    const int G = SEG ? A.ntiles : (int)gridDim.x;
    if (reduce_tail(bvals, nv, P, red, G, tile)) {
      E.finish(P, red);
#if PGM_TAIL_TIMING
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned long long t3 = gtimer();
        atomicAdd(&g_tail_ns[0], s_tail_t[1] - s_tail_t[0]);  // level-1 chain (final block)
        atomicAdd(&g_tail_ns[1], s_tail_t[2] - s_tail_t[1]);  // level 2
        atomicAdd(&g_tail_ns[2], t3 - s_tail_t[2]);           // finisher
        atomicAdd(&g_tail_ns[3], 1ull);
      }
#endif
    }
    return;
  }
  if constexpr (std::is_same<Epi, StepEpi>::value) {
    // Step epilogue, two phases.  (1) y = s_k (A W_k) + AU c -> W_{k+1} and
    // ys, thread per row.  (2) pass-1 dots W_l . y: warp w owns the basis
    // vectors l = w, w + 8, ... and streams its 512 rows with 16 independent
    // loads per lane; one warp sum per vector, no cross-warp combine.
    const int k = E.k;
    const int r = P.d->r;
    const size_t ld = P.ld;
    const int row0 = tile * TILE;
    const int rows = min(TILE, A.n - row0);
    double* wnext = P.V + (size_t)(k + 1) * ld + P.lo + row0;
    const double* au0 = P.AU + P.lo + row0;
    for (int i = threadIdx.x; i < TILE; i += SPMV_THREADS) {
      double y = 0.0;
      if (i < rows) {
        y = small[0] * ys[i];
        int l = 0;
        for (; l + 1 < r; l += 2) {
          const double t0 = __ldg(au0 + (size_t)l * ld + i);
          const double t1 = __ldg(au0 + (size_t)(l + 1) * ld + i);
          y += small[1 + l] * t0;
          y += small[2 + l] * t1;
        }
        if (l < r) y += small[1 + l] * __ldg(au0 + (size_t)l * ld + i);
        wnext[i] = y;
      }
      ys[i] = y;
    }
    __syncthreads();
    const int np = k + 1;
    const double* v0 = P.V + P.lo + row0;
    for (int l = warp; l < np; l += SPMV_WARPS) {
      const double* v = v0 + (size_t)l * ld + lane;
      double a[4] = {0.0, 0.0, 0.0, 0.0};
      if (rows == TILE) {
        double t[TILE / 32];
#pragma unroll
        for (int q = 0; q < TILE / 32; ++q) t[q] = __ldg(v + 32 * q);
#pragma unroll
        for (int q = 0; q < TILE / 32; ++q) a[q & 3] += t[q] * ys[lane + 32 * q];
      } else {
        for (int q = 0; q < TILE / 32; ++q)
          if (lane + 32 * q < rows) a[q & 3] += __ldg(v + 32 * q) * ys[lane + 32 * q];
      }
      const double sum = warp_sum((a[0] + a[1]) + (a[2] + a[3]));
      if (lane == 0) bvals[l] = sum;
    }
    pdl_trigger();
    __syncthreads();
    const int G = SEG ? A.ntiles : (int)gridDim.x;
    if (reduce_tail(bvals, nv, P, red, G, tile)) E.finish(P, red);
    return;
  }
  if constexpr (std::is_same<Epi, PushEpi>::value) {
    // push_vector tail (deflation.cpp:160-174), same two-phase scheme as the
    // step epilogue: (1) U_j = u ps, AU_j = (A u) ps per row into smem;
    // (2) the 2j+1 T row/column dots, warp-split over the vector families
    // U_l . AU_j (l < j), U_j . AU_j, U_j . AU_l (l < j).
    const int j = P.d->r;
    const size_t ld = P.ld;
    const int row0 = tile * TILE;
    const int rows = min(TILE, A.n - row0);
    const double ps = small[0];
    double* an = ys;      // (A u) ps, in place
    double* un = tp - (threadIdx.x >> 5) * TP_DOUBLES;  // the transpose area: TILE doubles
    for (int i = threadIdx.x; i < TILE; i += SPMV_THREADS) {
      double a = 0.0, uu = 0.0;
      if (i < rows) {
        uu = P.u[P.lo + row0 + i] * ps;
        a = ys[i] * ps;
        P.U[(size_t)j * ld + P.lo + row0 + i] = uu;
        P.AU[(size_t)j * ld + P.lo + row0 + i] = a;
      }
      an[i] = a;
      un[i] = uu;
    }
    __syncthreads();
    for (int v = warp; v < nv; v += SPMV_WARPS) {
      double a[4] = {0.0, 0.0, 0.0, 0.0};
      if (v == j) {
        for (int q = 0; q < TILE / 32; ++q) a[q & 3] += un[lane + 32 * q] * an[lane + 32 * q];
      } else {
        const double* vec = (v < j ? P.U + (size_t)v * ld : P.AU + (size_t)(v - j - 1) * ld) +
                            P.lo + row0 + lane;
        const double* mul = v < j ? an : un;
        if (rows == TILE) {
          double t[TILE / 32];
#pragma unroll
          for (int q = 0; q < TILE / 32; ++q) t[q] = __ldg(vec + 32 * q);
#pragma unroll
          for (int q = 0; q < TILE / 32; ++q) a[q & 3] += t[q] * mul[lane + 32 * q];
        } else {
          for (int q = 0; q < TILE / 32; ++q)
            if (lane + 32 * q < rows) a[q & 3] += __ldg(vec + 32 * q) * mul[lane + 32 * q];
        }
      }
      const double sum = warp_sum((a[0] + a[1]) + (a[2] + a[3]));
      if (lane == 0) bvals[v] = sum;
    }
    pdl_trigger();
    __syncthreads();
    const int G = SEG ? A.ntiles : (int)gridDim.x;
    if (reduce_tail(bvals, nv, P, red, G, tile)) E.finish(P, red);
    return;
  }
  double acc[NVL];
#pragma unroll
  for (int s = 0; s < NVL; ++s) acc[s] = 0.0;
  {
    const int row0 = tile * TILE;
    const int rows = min(TILE, A.n - row0);
    for (int sub = warp * 32; sub < TILE; sub += SPMV_THREADS) {
      const int i = sub + lane;
      const bool ok = i < rows;
      E.chunk(P, row0 + i, ok, ok ? ys[i] : 0.0, tp, acc, small);
    }
  }
  pdl_trigger();
  if (nv == 0) return;
  warps_to_block(acc, nv, wacc, bvals);
  const int G = SEG ? A.ntiles : (int)gridDim.x;
  if (reduce_tail(bvals, nv, P, red, G, tile)) E.finish(P, red);
}

// ---------------------------------------------------------------------------
// Halo planes over peer memory (world > 1, peer transport: CUDA IPC windows
// across processes, plain pointers between in-process ranks).  Every rank's
// window carries two parities x two mailboxes (planes coming from below and
// from above, hmax doubles each) and their flags.  k_halo_push stores this
// rank's boundary planes straight into the neighbours' mailboxes (NVLink P2P
// stores), fences system-wide and — from the last block — raises the
// neighbours' flags to the exchange epoch; k_halo_pull waits for its own two
// flags (bounded spin) and copies the mailboxes into the vector's halo rows.
// Parity reuse is safe: a rank pushes epoch e + 2 only after pulling e + 1,
// which needs its neighbour's push of e + 1, issued after that neighbour
// pulled e.  No NCCL, no host synchronisation.
struct HaloPeerArgs {
  char* const* win;         // [world] window bases as addressable from this rank
  char* mine;               // this rank's window
  size_t off_mb, off_hf;    // byte offsets: mailboxes [2 par][2 dir][hmax], flags [2 par][2 dir]
  size_t hmax;
  int me, world;
  unsigned long long* epoch;  // this rank's halo-exchange counter (in its window)
  unsigned* cnt;              // push completion counter
  GState* g;
};

__device__ __forceinline__ double* halo_mb(char* base, const HaloPeerArgs& A, int par, int dir) {
  return reinterpret_cast<double*>(base + A.off_mb) + ((size_t)par * 2 + dir) * A.hmax;
}
__device__ __forceinline__ unsigned long long* halo_fl(char* base, const HaloPeerArgs& A, int par,
                                                       int dir) {
  return reinterpret_cast<unsigned long long*>(base + A.off_hf) + par * 2 + dir;
}

__global__ void __launch_bounds__(256) k_halo_push(HaloPeerArgs A, const double* own, int n,
                                                   int dn, int up) {
  __shared__ int s_last;
  const unsigned long long e = *A.epoch + 1;
  const int par = (int)(e & 1ull);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t t0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (dn > 0) {  // own rows [0, dn) -> below's "from above" mailbox
    double* dst = halo_mb(A.win[A.me - 1], A, par, 1);
    for (size_t i = t0; i < (size_t)dn; i += stride) dst[i] = own[i];
  }
  if (up > 0) {  // own rows [n - up, n) -> above's "from below" mailbox
    double* dst = halo_mb(A.win[A.me + 1], A, par, 0);
    const double* src = own + n - up;
    for (size_t i = t0; i < (size_t)up; i += stride) dst[i] = src[i];
  }
  __threadfence_system();
  __syncthreads();
#ifdef PGM_PEER_DEBUG
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("push me %d e %llu dn %d up %d n %d own0 %g ownLast %g\n", A.me, e, dn, up, n, own[0],
           up > 0 ? own[n - up] : -1.0);
#endif
  if (threadIdx.x == 0) s_last = (atomicAdd(A.cnt, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence_system();
  *A.cnt = 0;
  *A.epoch = e;
  if (dn > 0) st_release_sys(halo_fl(A.win[A.me - 1], A, par, 1), e);
  if (up > 0) st_release_sys(halo_fl(A.win[A.me + 1], A, par, 0), e);
#ifdef PGM_PEER_DEBUG
  printf("push me %d raised e %llu at %p / %p\n", A.me, e,
         dn > 0 ? (void*)halo_fl(A.win[A.me - 1], A, par, 1) : nullptr,
         up > 0 ? (void*)halo_fl(A.win[A.me + 1], A, par, 0) : nullptr);
#endif
}

__global__ void __launch_bounds__(256) k_halo_pull(HaloPeerArgs A, double* vec, int lo, int n,
                                                   int hi) {
  __shared__ int s_timeout;
  const unsigned long long e = *A.epoch;
  const int par = (int)(e & 1ull);
  if (threadIdx.x == 0) s_timeout = 0;
  __syncthreads();
#ifdef PGM_PEER_DEBUG
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("pull me %d waits e %llu lo %d hi %d at %p / %p\n", A.me, e, lo, hi,
           (void*)halo_fl(A.mine, A, par, 0), (void*)halo_fl(A.mine, A, par, 1));
#endif
  if (threadIdx.x < 2) {
    const int dir = threadIdx.x;
    if ((dir == 0 && lo > 0) || (dir == 1 && hi > 0)) {
      const unsigned long long* f = halo_fl(A.mine, A, par, dir);
      const unsigned long long t_start = peer_clock_ns();
      long long spins = 0;
      while (ld_acquire_sys(f) < e) {
        if ((++spins & 1023) == 0 && peer_clock_ns() - t_start > PEER_WAIT_NS) {
          s_timeout = 1;  // a neighbour never pushed
          break;
        }
      }
    }
  }
  __syncthreads();
  if (s_timeout) {
    if (threadIdx.x == 0) {
      A.g->error = 7;  // PGM_ESTATE
      A.g->active = 0;
      A.g->done = 1;
    }
    return;
  }
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t t0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const double* from_below = halo_mb(A.mine, A, par, 0);
#ifdef PGM_PEER_DEBUG
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("pull me %d e %llu lo %d hi %d fb0 %g fa0 %g flags %llu %llu\n", A.me, e, lo, hi,
           from_below[0], halo_mb(A.mine, A, par, 1)[0], *halo_fl(A.mine, A, par, 0),
           *halo_fl(A.mine, A, par, 1));
#endif
  const double* from_above = halo_mb(A.mine, A, par, 1);
  for (size_t i = t0; i < (size_t)lo; i += stride) vec[i] = __ldcv(from_below + i);
  for (size_t i = t0; i < (size_t)hi; i += stride) vec[(size_t)lo + n + i] = __ldcv(from_above + i);
}

// Newton driver scalars etc. on the peer transport: all-reduce a small device
// buffer through the same windows and epoch as the reduction kernels.
__global__ void k_peer_allreduce_buf(Params P, double* buf, int nv) {
  __shared__ double red[PEER_NV];
  for (int v = threadIdx.x; v < nv; v += blockDim.x) red[v] = buf[v];
  __syncthreads();
  peer_allreduce(red, nv, P);
  for (int v = threadIdx.x; v < nv; v += blockDim.x) buf[v] = red[v];
}

// ---------------------------------------------------------------------------
// x update at the end of a cycle: x += V xc + U cx (gmres.cpp:183-188, with
// M^{-1} of the correction folded into U cx through the cached U^T V; the
// coefficients come from k_end_cycle).  Streaming like the DCGS2 update: a
// warp per 64-row chunk, 2 rows per lane, the basis and U columns read in
// batches of 4 double2 loads per lane.
constexpr int XU_BLOCK = 256;
__global__ void __launch_bounds__(XU_BLOCK) k_xupdate(Params P) {
  __shared__ double cv[MAX_M + MAX_R1 + 8];
  const GState* g = P.g;
  if (g->error != 0) return;
  const int steps = g->steps, r = P.d->r;
  const int nvec = steps + r;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int l = threadIdx.x; l < nvec + 4; l += XU_BLOCK)
    cv[l] = l < steps ? P.xc[l] : (l < nvec ? P.cx[l - steps] : 0.0);
  __syncthreads();
  const int n = P.n;
  const size_t ld = P.ld;
  const double* V0 = P.V + P.lo;
  const double* U0 = P.U + P.lo;
  double* x = P.x + P.lo;
  const int nch = (n + 63) >> 6;
  const int W = gridDim.x * (XU_BLOCK / 32);
  for (int c = blockIdx.x * (XU_BLOCK / 32) + warp; c < nch; c += W) {
    const int row0 = c * 64 + 2 * lane;
    double2 acc = make_double2(0.0, 0.0);
    for (int l0 = 0; l0 < nvec; l0 += 4) {
      double2 t[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int l = l0 + j;
        const double* base = l < steps ? V0 + (size_t)l * ld : U0 + (size_t)(l - steps) * ld;
        t[j] = l < nvec ? __ldg(reinterpret_cast<const double2*>(base + row0))
                        : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc.x += cv[l0 + j] * t[j].x;
        acc.y += cv[l0 + j] * t[j].y;
      }
    }
    if (row0 + 1 < n) {
      double2 xv = *reinterpret_cast<const double2*>(x + row0);
      xv.x += acc.x;
      xv.y += acc.y;
      *reinterpret_cast<double2*>(x + row0) = xv;
    } else if (row0 < n) {
      x[row0] += acc.x;
    }
  }
}

// ---------------------------------------------------------------------------
// DCGS2 cycle close (a cycle that ran all m steps): red = [W_l . u_m (l < m),
// u_m . u_m] completes column m-1 (fin_dcgs2_close).  Same scheme as the step
// SpMV's epilogue: one 512-row tile per block, u_m's rows staged in smem,
// warp w streams W_w, W_{w+8}, ... with all 16 loads per lane in flight.
// (The generic k_sweep<SW_DCLOSE> moved 1.5x the algorithmic bytes at 4.2
// TB/s: its Q set went through the transposed tile.)
__global__ void __launch_bounds__(SPMV_THREADS) k_dclose(Params P, int ntiles) {
  extern __shared__ double sm[];
  pdl_wait();
  if (!P.g->active) return;
  const int m = P.m, nv = m + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int row0 = tile * TILE;
  const int rows = min(TILE, P.n - row0);
  const size_t ld = P.ld;
  double* us = sm;
  double* bvals = us + TILE;
  double* red = bvals + nv;
  const double* um = P.V + (size_t)m * ld + P.lo + row0;
  for (int i = threadIdx.x; i < TILE; i += SPMV_THREADS) us[i] = i < rows ? um[i] : 0.0;
  __syncthreads();
  const double* v0 = P.V + P.lo + row0;
  for (int q = warp; q < nv; q += SPMV_WARPS) {
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    if (q < m) {
      const double* v = v0 + (size_t)q * ld + lane;
      if (rows == TILE) {
        double t[TILE / 32];
#pragma unroll
        for (int i = 0; i < TILE / 32; ++i) t[i] = __ldg(v + 32 * i);
#pragma unroll
        for (int i = 0; i < TILE / 32; ++i) a[i & 3] += t[i] * us[lane + 32 * i];
      } else {
        for (int i = 0; i < TILE / 32; ++i)
          if (lane + 32 * i < rows) a[i & 3] += __ldg(v + 32 * i) * us[lane + 32 * i];
      }
    } else {
      for (int i = 0; i < TILE / 32; ++i) {
        const double u = us[lane + 32 * i];
        a[i & 3] += u * u;
      }
    }
    const double sum = warp_sum((a[0] + a[1]) + (a[2] + a[3]));
    if (lane == 0) bvals[q] = sum;
  }
  pdl_trigger();
  __syncthreads();
  if (reduce_tail(bvals, nv, P, red, ntiles, tile)) fin_dcgs2_close(P, red);
}

// ---------------------------------------------------------------------------
// Streaming sweeps over basis blocks.
enum SweepMode {
  SW_CGS2_B = 0,   // w1 = w - V h1 ; dots V^T w1 (staged)
  SW_CGS2_C = 1,   // w2 = w1 - V h2 (k_cgs2_update; class id for the profile only)
  SW_XUPDATE = 2,  // x += V xc + U cx
  SW_PUSH1 = 3,    // u = V zl (or u given) ; ||u||^2, U^T u
  SW_PUSH2 = 4,    // u -= U proj ; U^T u (staged)
  SW_PUSH3 = 5,    // u -= U proj ; ||u||^2
  SW_DOTS_U = 6,   // U^T u only (apply)
  SW_AXPY_U = 7,   // u += U c only (apply)
  SW_DCLOSE = 8,   // DCGS2 cycle close: W_l . u_m, ||u_m||^2
};

struct SweepSpec {
  const double* in;
  double* out;
  const double* Pv;  // first set base (own region of slot 0)
  int np;
  const double* a;
  const double* P2;
  int np2;
  const double* a2;
  const double* Q;  // dot set (own region of slot 0)
  int nq;
  int qstaged;
  int selfnorm;
  int normlast;  // the self-norm is value nq (after the dots), not value 0
  int skip;
};

template <int MODE>
__device__ __forceinline__ SweepSpec sweep_spec(const Params& P, int k) {
  SweepSpec S{};
  const GState* g = P.g;
  const DState* d = P.d;
  const size_t lo = P.lo;
  if (MODE == SW_CGS2_B) {
    // generic path (np > 112, plain GMRES only: r = 0): W_l . w1 then ||w1||^2
    S.skip = !g->active;
    S.in = S.out = P.V + (size_t)(k + 1) * P.ld + lo;
    S.Pv = P.V + lo;
    S.np = k + 1;
    S.a = P.coefA;
    S.Q = S.Pv;
    S.nq = k + 1;
    S.qstaged = 1;
    S.selfnorm = 1;
    S.normlast = 1;
  } else if (MODE == SW_DCLOSE) {
    S.skip = !g->active;
    S.in = S.out = P.V + (size_t)P.m * P.ld + lo;
    S.Q = P.V + lo;
    S.nq = P.m;
    S.selfnorm = 1;
    S.normlast = 1;
  } else if (MODE == SW_XUPDATE) {
    S.skip = g->error != 0;
    S.in = S.out = P.x + lo;
    S.Pv = P.V + lo;
    S.np = g->steps;
    S.a = P.xc;
    S.P2 = P.U + lo;
    S.np2 = d->r;
    S.a2 = P.cx;
  } else if (MODE == SW_PUSH1) {
    // k == 1: harvest u = V zl ; k == 0: u already holds the candidate
    S.skip = g->error != 0 || !d->push_ok;
    S.out = P.u + lo;
    if (k == 0) {
      S.in = S.out;
    } else {
      S.Pv = P.V + lo;
      S.np = g->steps;
      S.a = P.zl;
    }
    S.Q = P.U + lo;
    S.nq = d->r;
    S.selfnorm = 1;
  } else if (MODE == SW_PUSH2) {
    S.skip = g->error != 0 || !d->push_ok || d->r == 0;
    S.in = S.out = P.u + lo;
    S.Pv = P.U + lo;
    S.np = d->r;
    S.a = P.proj;
    S.Q = S.Pv;
    S.nq = d->r;
    S.qstaged = 1;
  } else if (MODE == SW_PUSH3) {
    S.skip = g->error != 0 || !d->push_ok || d->r == 0;
    S.in = S.out = P.u + lo;
    S.Pv = P.U + lo;
    S.np = d->r;
    S.a = P.proj;
    S.selfnorm = 1;
  } else if (MODE == SW_DOTS_U) {
    S.skip = d->r == 0;
    S.in = S.out = P.u + lo;
    S.Q = P.U + lo;
    S.nq = d->r;
  } else if (MODE == SW_AXPY_U) {
    S.skip = d->r == 0;
    S.in = S.out = P.u + lo;
    S.Pv = P.U + lo;
    S.np = d->r;
    S.a = P.c;
  }
  return S;
}

template <int MODE>
__device__ __forceinline__ void sweep_finish(const Params& P, int k, const double* red) {
  // block-collective (finish.cuh); the push_vector scalars run on thread 0
  if (MODE == SW_CGS2_B) fin_sweep_b(P, k, red);
  if (MODE == SW_PUSH1 && threadIdx.x == 0) fin_push1(P, red);
  if (MODE == SW_PUSH2 && threadIdx.x == 0) fin_push2(P, red);
  if (MODE == SW_PUSH3 && threadIdx.x == 0) fin_push3(P, red);
  if (MODE == SW_DCLOSE) fin_dcgs2_close(P, red);
  if (MODE == SW_DOTS_U) {
    for (int l = threadIdx.x; l < P.d->r; l += blockDim.x) P.proj[l] = red[l];
    __syncthreads();
    defl_coeffs_par(P, P.d->r, P.proj, P.c);
  }
}

// Streaming sweep over basis blocks: each warp owns 32-row chunks (lane =
// row), grid-strided over all warps.  Phase 1 issues every load of the chunk
// first (NP values held in registers), then
//   out[row] = in[row] + sum_l a_l P_l[row] + sum_l a2_l P2_l[row];
// phase 2 forms the dot products of out with the register-resident P set
// (qstaged) or a second set Q through the per-warp transposed tile.
// NP = 0 is the generic path (np > 64): P re-read from L1/L2 for the dots.
constexpr int SW_BLOCK = 128;
constexpr int SW_WARPS = SW_BLOCK / 32;

__host__ __device__ constexpr size_t sweep_smem_doubles(int nv, int np) {
  return (size_t)SW_WARPS * TP_DOUBLES + (size_t)SW_WARPS * NVL * TPR + 2 * (size_t)nv + 2 +
         (size_t)np;
}

template <int MODE, int NP>
__global__ void __launch_bounds__(SW_BLOCK) k_sweep(Params P, int k) {
  extern __shared__ double sm[];
  const SweepSpec S = sweep_spec<MODE>(P, k);
  if (S.skip) return;
  const int nv = S.nq + S.selfnorm;
  const int so = S.selfnorm && !S.normlast;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* tp = sm + warp * TP_DOUBLES;
  double* wacc = sm + SW_WARPS * TP_DOUBLES;
  double* bvals = wacc + SW_WARPS * NVL * TPR;
  double* red = bvals + nv;
  double* as = red + nv;
  double acc[NVL];
#pragma unroll
  for (int s = 0; s < NVL; ++s) acc[s] = 0.0;
  const int n = P.n;
  const size_t ld = P.ld;
  const int nchunks = (n + 31) >> 5;
  const int W = gridDim.x * SW_WARPS;
  for (int l = threadIdx.x; l < S.np; l += blockDim.x) as[l] = S.a[l];
  __syncthreads();
  const int has_in = S.in != nullptr;
  const int qg = S.qstaged ? 0 : S.nq;
  const int nseg = has_in + S.np + S.np2 + qg;
  // L2 prefetch (TMA engine) of every 256-byte row segment of chunk c: one per lane
  auto prefetch = [&](int c) {
    if (c >= nchunks) return;
    const size_t off = (size_t)c * 32;
    for (int q = lane; q < nseg; q += 32) {
      const double* src;
      int l = q - has_in;
      if (l < 0) {
        src = S.in;
      } else if (l < S.np) {
        src = S.Pv + (size_t)l * ld;
      } else if ((l -= S.np) < S.np2) {
        src = S.P2 + (size_t)l * ld;
      } else {
        src = S.Q + (size_t)(l - S.np2) * ld;
      }
      tma_prefetch_l2(src + off, 256);
    }
  };
  prefetch(blockIdx.x * SW_WARPS + warp);
  for (int c = blockIdx.x * SW_WARPS + warp; c < nchunks; c += W) {
    prefetch(c + W);
    const int row = c * 32 + lane;
    const bool ok = row < n;
    double o = (ok && S.in) ? S.in[row] : 0.0;
    double v[NP > 0 ? NP : 1];
    if (NP > 0) {
#pragma unroll
      for (int l = 0; l < NP; ++l)
        v[l] = (l < S.np && ok) ? __ldg(S.Pv + (size_t)l * ld + row) : 0.0;
      __syncwarp();  // scheduling fence: every load is in flight before the first use
      double o4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int l = 0; l < NP; ++l)
        if (l < S.np) o4[l & 3] += as[l] * v[l];
      o += (o4[0] + o4[1]) + (o4[2] + o4[3]);
    } else {
      for (int l0 = 0; l0 < S.np; l0 += 16) {
        double t[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          t[j] = (l0 + j < S.np && ok) ? __ldg(S.Pv + (size_t)(l0 + j) * ld + row) : 0.0;
        __syncwarp();
        double o4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (l0 + j < S.np) o4[j & 3] += as[l0 + j] * t[j];
        o += (o4[0] + o4[1]) + (o4[2] + o4[3]);
      }
    }
    if (S.np2 > 0 && ok) {
      const double* p2 = S.P2 + row;
#pragma unroll 4
      for (int l = 0; l < S.np2; ++l) o += __ldg(S.a2 + l) * __ldg(p2 + (size_t)l * ld);
    }
    if (ok) S.out[row] = o;
    else o = 0.0;
    if (nv == 0) continue;
    if (S.qstaged && NP > 0 && !S.selfnorm) {
      // products with the register-resident P set
#pragma unroll
      for (int sl = 0; sl < (NP + TPR - 1) / TPR; ++sl) {
        if (sl * TPR >= nv) continue;
        const int cnt = min(TPR, nv - sl * TPR);
#pragma unroll
        for (int j = 0; j < TPR; ++j)
          if (j < cnt && sl * TPR + j < NP) tp[j * TPS + lane] = v[sl * TPR + j < NP ? sl * TPR + j : 0] * o;
        __syncwarp();
        const double s = tp_sum16(tp, lane);
        if (lane < cnt) acc[sl] += s;
        __syncwarp();
      }
    } else {
      const double* q = (S.qstaged ? S.Pv : S.Q) + row;
      tp_all(tp, acc, nv, lane, [&](int vv) {
        if (!ok) return 0.0;
        if (S.normlast) return vv == S.nq ? o * o : __ldg(q + (size_t)vv * ld) * o;
        return (so && vv == 0) ? o * o : __ldg(q + (size_t)(vv - so) * ld) * o;
      });
    }
  }
  if (nv == 0) return;
  warps_to_block(acc, nv, wacc, bvals);
  if (reduce_tail(bvals, nv, P, red, (int)gridDim.x, (int)blockIdx.x)) sweep_finish<MODE>(P, k, red);
}

// RPL consecutive rows of one vector (16-byte aligned for RPL >= 2), or zeros.
template <int RPL>
__device__ __forceinline__ void load_rows(const double* p, bool pred, double (&o)[RPL]) {
  if (RPL == 1) {
    o[0] = pred ? __ldg(p) : 0.0;
  } else {
#pragma unroll
    for (int e = 0; e < RPL; e += 2) {
      const double2 t = pred ? __ldg(reinterpret_cast<const double2*>(p + e)) : make_double2(0.0, 0.0);
      o[e] = t.x;
      o[e + 1] = t.y;
    }
  }
}
template <int RPL>
__device__ __forceinline__ void store_rows(double* p, const double (&o)[RPL]) {
  if (RPL == 1) {
    p[0] = o[0];
  } else {
#pragma unroll
    for (int e = 0; e < RPL; e += 2) *reinterpret_cast<double2*>(p + e) = make_double2(o[e], o[e + 1]);
  }
}

// CGS2 pass B, vector set split across the warps of a block (tools/sweepbench.cu):
//   w1 = w + sum_l a_l W_l ; dots W_l . w1, ||w1||^2 and U_j . w1
// (pass C is then a reduction-free update, k_cgs2_update).
// All NW warps of a block work on the same chunk of 32*RPL rows (lane = RPL
// consecutive rows).  Warp q streams the basis vectors l = q + NW*j (j < NPW)
// and, in pass C, the deflation vectors U_j, j = q + NW*i, so every warp keeps
// only a few rows in registers and the SM holds many warps' loads in flight.
// The per-warp partial row sums meet in smem (double-buffered: one barrier
// per chunk); the block sum of the row update is formed in warp order, and
// each warp accumulates its own dot products in lane-private registers across
// all of its chunks (one warp reduction at the end).  The order of every sum
// depends only on the grid size: bitwise reproducible run to run.
// Rows past the owned range (padding / halo memory, always allocated) are read
// and masked before any store or product.
// NUW: deflation vectors per warp (covers the rank r of this cycle; the host
// picks the instantiation), NPW: basis vectors per warp.
template <int MODE, int NW, int RPL, int NUW, int NPW>
__global__ void __launch_bounds__(NW * 32) k_cgs2(Params P, int k) {
  static_assert(MODE == SW_CGS2_B, "pass C is k_cgs2_update");
  constexpr int NA = NPW + NUW + 1;
  constexpr int CR = 32 * RPL;  // rows per chunk
  __shared__ __align__(16) double xs[2][NW][CR];
  __shared__ double bv[NW * NA + 2];
  __shared__ double redv[NW * NA + 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int np = k + 1;
  const int n = P.n;
  const size_t ld = P.ld;
  const int nch = (n + CR - 1) / CR;
  const double* V0 = P.V + P.lo;
  // Ahead of the PDL wait: L2 prefetch of this warp's W_0..W_k segments of its
  // first two chunks (W_l, l <= k, were written >= 2 kernels back).
  for (int c = blockIdx.x; c < nch && c < (int)(blockIdx.x + 2 * gridDim.x); c += gridDim.x) {
    const size_t off = (size_t)c * CR;
    for (int q = lane; q < NPW; q += 32) {
      const int l = warp + NW * q;
      if (l < np) tma_prefetch_l2(V0 + (size_t)l * ld + off, CR * 8);
    }
  }
  pdl_wait();
  if (!P.g->active) return;
  const int r = P.d->r;
  double* w = P.V + (size_t)(k + 1) * ld + P.lo;
  const double* U0 = P.U + P.lo;
  const double* coef = P.coefA;
  double aw[NPW];
#pragma unroll
  for (int j = 0; j < NPW; ++j) {
    const int l = warp + NW * j;
    aw[j] = l < np ? coef[l] : 0.0;
  }
  double acc[NA];
#pragma unroll
  for (int j = 0; j < NA; ++j) acc[j] = 0.0;
  // L2 prefetch (TMA engine) of this warp's segments of chunk c
  auto prefetch = [&](int c) {
    if (c >= nch) return;
    const size_t off = (size_t)c * CR;
    for (int q = lane; q < NPW + NUW + 1; q += 32) {
      const double* src = nullptr;
      if (q < NPW) {
        const int l = warp + NW * q;
        if (l < np) src = V0 + (size_t)l * ld;
      } else if (q < NPW + NUW) {
        const int lu = warp + NW * (q - NPW);
        if (lu < r) src = U0 + (size_t)lu * ld;
      } else if (warp == 0) {
        src = w;
      }
      if (src) tma_prefetch_l2(src + off, CR * 8);
    }
  };
  int buf = 0;
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    prefetch(c + 2 * gridDim.x);
    const int row0 = c * CR + lane * RPL;
    double v[NPW][RPL];
    double u[NUW > 0 ? NUW : 1][RPL];
    double win[RPL];
#pragma unroll
    for (int j = 0; j < NPW; ++j) {
      const int l = warp + NW * j;
      load_rows<RPL>(V0 + (size_t)l * ld + row0, l < np, v[j]);
    }
#pragma unroll
    for (int j = 0; j < NUW; ++j) {
      const int lu = warp + NW * j;
      load_rows<RPL>(U0 + (size_t)lu * ld + row0, lu < r, u[j]);
    }
    load_rows<RPL>(w + row0, warp == 0, win);
    __syncwarp();  // scheduling fence: every load of the chunk in flight before the first use
#pragma unroll
    for (int e = 0; e < RPL; ++e) {
      double p0 = win[e], p1 = 0.0;
#pragma unroll
      for (int j = 0; j < NPW; ++j) {
        if (j & 1) p1 += aw[j] * v[j][e];
        else p0 += aw[j] * v[j][e];
      }
      xs[buf][warp][lane * RPL + e] = p0 + p1;
    }
    __syncthreads();
    double o[RPL];
#pragma unroll
    for (int e = 0; e < RPL; ++e) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < NW; ++q) s += xs[buf][q][lane * RPL + e];
      o[e] = (row0 + e < n) ? s : 0.0;
    }
    if (warp == 0) {
      if (row0 + RPL <= n) {
        store_rows<RPL>(w + row0, o);
      } else {
#pragma unroll
        for (int e = 0; e < RPL; ++e)
          if (row0 + e < n) w[row0 + e] = o[e];
      }
    }
#pragma unroll
    for (int e = 0; e < RPL; ++e) {
#pragma unroll
      for (int j = 0; j < NPW; ++j) acc[j] += v[j][e] * o[e];
#pragma unroll
      for (int j = 0; j < NUW; ++j) acc[NPW + j] += u[j][e] * o[e];
      if (warp == 0) acc[NPW + NUW] += o[e] * o[e];
    }
    buf ^= 1;
  }
  pdl_trigger();
  // block values: bv[l] = W_l . w1 (l < np), bv[np] = ||w1||^2, bv[np + 1 + j] = U_j . w1
  const int nv = np + 1 + r;
#pragma unroll
  for (int j = 0; j < NA; ++j) {
    const double sum = warp_sum(acc[j]);
    if (lane == 0) {
      if (j < NPW) {
        const int l = warp + NW * j;
        if (l < np) bv[l] = sum;
      } else if (j < NPW + NUW) {
        const int lu = warp + NW * (j - NPW);
        if (lu < r) bv[np + 1 + lu] = sum;
      } else if (warp == 0) {
        bv[np] = sum;
      }
    }
  }
  __syncthreads();
  if (reduce_tail(bv, nv, P, redv, (int)gridDim.x, (int)blockIdx.x)) sweep_finish<MODE>(P, k, redv);
}

// CGS2 pass C: W_{k+1} = w1 + sum_l b_l W_l (b_l = -h2_l s_l).  No reduction:
// ||w2||^2 and U^T w2 were formed from pass B's dots (fin_sweep_b), so this is
// a pure stream: each warp owns 64-row chunks (2 rows per lane), the basis is
// read in batches of 8 vectors with all loads of a batch in flight.
constexpr int UPD_BLOCK = 256;
__global__ void __launch_bounds__(UPD_BLOCK) k_cgs2_update(Params P, int k) {
  __shared__ double as[MAX_M + 8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int np = k + 1;
  const int n = P.n;
  const size_t ld = P.ld;
  const int nch = (n + 63) >> 6;
  const int W = gridDim.x * (UPD_BLOCK / 32);
  const double* V0 = P.V + P.lo;
  {
    // ahead of the PDL wait: this warp's first chunk of W_0..W_k into L2
    const int c = blockIdx.x * (UPD_BLOCK / 32) + warp;
    if (c < nch)
      for (int l = lane; l < np; l += 32) tma_prefetch_l2(V0 + (size_t)l * ld + (size_t)c * 64, 512);
  }
  pdl_wait();
  if (!P.g->active) return;
  for (int l = threadIdx.x; l < np + 8; l += UPD_BLOCK) as[l] = l < np ? P.coefB[l] : 0.0;
  __syncthreads();
  double* w = P.V + (size_t)(k + 1) * ld + P.lo;
  for (int c = blockIdx.x * (UPD_BLOCK / 32) + warp; c < nch; c += W) {
    const int row0 = c * 64 + 2 * lane;
    double2 o = *reinterpret_cast<const double2*>(w + row0);
    for (int l0 = 0; l0 < np; l0 += 8) {
      double2 t[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        t[j] = (l0 + j < np) ? __ldg(reinterpret_cast<const double2*>(V0 + (size_t)(l0 + j) * ld + row0))
                             : make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        o.x += as[l0 + j] * t[j].x;
        o.y += as[l0 + j] * t[j].y;
      }
    }
    if (row0 + 1 < n) {
      *reinterpret_cast<double2*>(w + row0) = o;
    } else if (row0 < n) {
      w[row0] = o.x;
    }
  }
  pdl_trigger();
}

#ifndef PGM_DUPD_PF
#define PGM_DUPD_PF 0
#endif
#ifndef PGM_DUPD_BATCH
#define PGM_DUPD_BATCH 4  // basis vectors per load batch (measured: 4 and 16 beat 8)
#endif
// DCGS2 update pass (one stream over W_0..W_{k-1}, u_k = W_k, y = W_{k+1}):
//   q_k (unnormalised)  W_k     = u + sum_{l<k} coefA_l W_l          (k >= 1)
//   u_{k+1}             W_{k+1} = coefA_k y + sum_{l<k} coefB_l W_l + coefB_k W_k'
#ifndef PGM_UPD_MINB
#define PGM_UPD_MINB 4  // min resident blocks per SM: 64 registers, 4 x 256 threads (3 at the natural 78 registers: update pass 3.4 % slower at config 3)
#endif
__global__ void __launch_bounds__(UPD_BLOCK, PGM_UPD_MINB) k_dcgs2_update(Params P, int k) {
  __shared__ double ca[MAX_M + 32], cb[MAX_M + 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = P.n;
  const size_t ld = P.ld;
  const int nch = (n + 63) >> 6;
  const int W = gridDim.x * (UPD_BLOCK / 32);
  const double* V0 = P.V + P.lo;
  pdl_wait();
  if (!P.g->active) return;
  for (int l = threadIdx.x; l < k + PGM_DUPD_BATCH; l += UPD_BLOCK) {
    ca[l] = l <= k ? P.coefA[l] : 0.0;
    cb[l] = l <= k ? P.coefB[l] : 0.0;
  }
  __syncthreads();
  double* wk = P.V + (size_t)k * ld + P.lo;
  double* wn = P.V + (size_t)(k + 1) * ld + P.lo;
  for (int c = blockIdx.x * (UPD_BLOCK / 32) + warp; c < nch; c += W) {
#if PGM_DUPD_PF
    // L2 prefetch of this warp's next chunk: W_0..W_{k+1}, one 512 B segment per lane
    if (c + W < nch)
      for (int l = lane; l < k + 2; l += 32)
        tma_prefetch_l2(V0 + (size_t)l * ld + (size_t)(c + W) * 64, 512);
#endif
    const int row0 = c * 64 + 2 * lane;
    double2 q = *reinterpret_cast<const double2*>(wk + row0);
    const double2 y = *reinterpret_cast<const double2*>(wn + row0);
    double2 un = make_double2(0.0, 0.0);
    for (int l0 = 0; l0 < k; l0 += PGM_DUPD_BATCH) {
      double2 t[PGM_DUPD_BATCH];
#pragma unroll
      for (int j = 0; j < PGM_DUPD_BATCH; ++j)
        t[j] = (l0 + j < k) ? __ldg(reinterpret_cast<const double2*>(V0 + (size_t)(l0 + j) * ld + row0))
                            : make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < PGM_DUPD_BATCH; ++j) {
        q.x += ca[l0 + j] * t[j].x;
        q.y += ca[l0 + j] * t[j].y;
        un.x += cb[l0 + j] * t[j].x;
        un.y += cb[l0 + j] * t[j].y;
      }
    }
    const double2 o = make_double2(ca[k] * y.x + un.x + cb[k] * q.x, ca[k] * y.y + un.y + cb[k] * q.y);
    if (row0 + 1 < n) {
      if (k > 0) *reinterpret_cast<double2*>(wk + row0) = q;
      *reinterpret_cast<double2*>(wn + row0) = o;
    } else if (row0 < n) {
      if (k > 0) wk[row0] = q.x;
      wn[row0] = o.x;
    }
  }
  pdl_trigger();
}

// Cross-GPU path: finisher after the allreduce of P.red_out.
template <int KIND>
__global__ void k_finish(Params P, int k) {
  // KIND: 0..7 sweep modes, 100 step spmv, 101 residual (k = initial), 102 push spmv.
  // All threads of the block take part (the finishers are block-collective).
  const double* red = P.red_out;
  if (KIND == 100) {
    if (P.g->active) fin_step_spmv(P, k, red);
  } else if (KIND == 101) {
    if (!(P.g->error != 0 || (!k && P.g->done))) fin_residual(P, red, k != 0);
  } else if (KIND == 102) {
    if (P.d->push_ok && threadIdx.x == 0) fin_push_spmv(P, red);
  } else if (KIND == 103) {
    if (P.g->active) fin_dcgs2(P, k, red);
  } else {
    const SweepSpec S = sweep_spec<KIND>(P, k);
    if (!S.skip) sweep_finish<KIND>(P, k, red);
  }
}

// ---------------------------------------------------------------------------
// Deterministic mode: every reduction value is dot(a_v, b_v) over the owned
// rows of two vectors that the reduction kernel left in memory.  k_det_dots
// forms, per node plane, the sequential sum  acc += a_i * b_i  over the
// plane's rows in ascending order (the reference's deterministic
// Executor::dot_kernel with block = n_axis^2, parallel.cpp:120-131), then
// combines the planes with the reference's pairwise fold (parallel.cpp:33-46)
// — for one rank in the kernel's last block, for world > 1 after the plane
// partials of all ranks were gathered (k_det_finish).  The result depends
// only on the vectors, never on the partition: bit-identical for any rank
// count, and bit-identical to the reference executor's dot of the same
// vectors.  The finishers then run unchanged (same dispatch as k_finish).
struct DetPair {
  const double* a;
  const double* b;
};

template <int KIND>
__device__ __forceinline__ bool det_skip(const Params& P, int k) {
  if (KIND == 100 || KIND == 103) return !P.g->active;
  if (KIND == 101) return P.g->error != 0 || (!k && P.g->done);
  if (KIND == 102) return !P.d->push_ok;
  if (KIND == SW_CGS2_B) return !P.g->active;
  return sweep_spec<KIND>(P, k).skip != 0;
}

template <int KIND>
__device__ __forceinline__ int det_nv(const Params& P, int k) {
  const int r = P.d->r;
  if (KIND == 100) return k + 1;
  if (KIND == 101) return 1 + r;
  if (KIND == 102) return 2 * r + 1;
  if (KIND == 103) return (k > 0 ? k : 1) + k + 2 + r;
  if (KIND == SW_CGS2_B) return k + 2 + r;
  const SweepSpec S = sweep_spec<KIND>(P, k);
  return S.nq + (S.selfnorm ? 1 : 0);
}

template <int KIND>
__device__ __forceinline__ DetPair det_pair(const Params& P, int k, int v) {
  const size_t ld = P.ld, lo = P.lo;
  const double* V = P.V + lo;
  const double* U = P.U + lo;
  const double* AU = P.AU + lo;
  if (KIND == 100) return {V + (size_t)v * ld, V + (size_t)(k + 1) * ld};
  if (KIND == 101) return v == 0 ? DetPair{V, V} : DetPair{U + (size_t)(v - 1) * ld, V};
  if (KIND == 102) {
    const int j = P.d->r;
    if (v < j) return {U + (size_t)v * ld, AU + (size_t)j * ld};
    if (v == j) return {U + (size_t)j * ld, AU + (size_t)j * ld};
    return {U + (size_t)j * ld, AU + (size_t)(v - j - 1) * ld};
  }
  if (KIND == 103) {
    const int nb = k > 0 ? k : 1;
    const double* y = V + (size_t)(k + 1) * ld;
    const double* u = V + (size_t)k * ld;
    if (v < nb) return {V + (size_t)v * ld, y};
    if (v < nb + k) return {V + (size_t)(v - nb) * ld, u};
    if (v == nb + k) return {u, u};
    if (v == nb + k + 1) return {u, y};
    return {U + (size_t)(v - nb - k - 2) * ld, y};
  }
  if (KIND == SW_CGS2_B) {
    const double* w = V + (size_t)(k + 1) * ld;
    if (v <= k) return {V + (size_t)v * ld, w};
    if (v == k + 1) return {w, w};
    return {U + (size_t)(v - k - 2) * ld, w};
  }
  const SweepSpec S = sweep_spec<KIND>(P, k);
  const double* o = S.out;
  if (S.selfnorm) {
    const int self = S.normlast ? S.nq : 0;
    if (v == self) return {o, o};
    const int q = S.normlast ? v : v - 1;
    return {S.Q + (size_t)q * ld, o};
  }
  return {S.Q + (size_t)v * ld, o};
}

// the reference's pairwise fold over s[0..n) (destroys s)
__device__ __forceinline__ double det_fold(double* s, int n) {
  if (n == 0) return 0.0;
  while (n > 1) {
    const int m = n / 2;
    for (int i = 0; i < m; ++i) s[i] = __dadd_rn(s[2 * i], s[2 * i + 1]);
    int nm = m;
    if (n % 2) s[nm++] = s[n - 1];
    n = nm;
  }
  return s[0];
}

template <int KIND>
__device__ __forceinline__ void det_finish_dispatch(const Params& P, int k, const double* red) {
  if (KIND == 100) {
    fin_step_spmv(P, k, red);
  } else if (KIND == 101) {
    fin_residual(P, red, k != 0);
  } else if (KIND == 102) {
    if (threadIdx.x == 0) fin_push_spmv(P, red);
  } else if (KIND == 103) {
    fin_dcgs2(P, k, red);
  } else {
    sweep_finish<KIND>(P, k, red);
  }
}

constexpr int DET_THREADS = 128;
constexpr int DET_MAXNV = 2 * MAX_M + 2 + MAX_R1;

// One thread per (plane, value): the sequential plane sum.  Launched after
// the reduction kernel (stream order), grid = ceil(nplanes * nv / 128).
template <int KIND>
__global__ void __launch_bounds__(DET_THREADS) k_det_dots(Params P, int k) {
  __shared__ double red[DET_MAXNV];
  __shared__ int s_last;
  if (det_skip<KIND>(P, k)) return;
  const int nv = det_nv<KIND>(P, k);
  const int np = P.nplanes;
  const long t = (long)blockIdx.x * DET_THREADS + threadIdx.x;
  if (t < (long)np * nv) {
    const int q = (int)(t / nv), v = (int)(t % nv);
    const DetPair pr = det_pair<KIND>(P, k, v);
    const long r0 = (long)q * P.plane;
    const int rows = (int)min((long)P.plane, (long)P.n - r0);
    const double* a = pr.a + r0;
    const double* b = pr.b + r0;
    double acc = 0.0;
    int i = 0;
    for (; i + 4 <= rows; i += 4) {  // loads run ahead of the (sequential) sum
      const double a0 = a[i], a1 = a[i + 1], a2 = a[i + 2], a3 = a[i + 3];
      const double b0 = b[i], b1 = b[i + 1], b2 = b[i + 2], b3 = b[i + 3];
      acc = __dadd_rn(acc, __dmul_rn(a0, b0));
      acc = __dadd_rn(acc, __dmul_rn(a1, b1));
      acc = __dadd_rn(acc, __dmul_rn(a2, b2));
      acc = __dadd_rn(acc, __dmul_rn(a3, b3));
    }
    for (; i < rows; ++i) acc = __dadd_rn(acc, __dmul_rn(a[i], b[i]));
    P.det_pp[(size_t)v * np + q] = acc;
  }
  if (P.world > 1) return;  // gathered on the host side, folded by k_det_finish
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(P.det_cnt, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int v = threadIdx.x; v < nv; v += DET_THREADS)
    red[v] = det_fold(P.det_pp + (size_t)v * np, np);
  if (threadIdx.x == 0) *P.det_cnt = 0;
  __syncthreads();
  det_finish_dispatch<KIND>(P, k, red);
}

// world > 1: fold the gathered plane partials of all ranks (global plane
// order) and run the finisher, identically on every rank.
template <int KIND>
__global__ void __launch_bounds__(DET_THREADS) k_det_finish(Params P, int k) {
  __shared__ double red[DET_MAXNV];
  if (det_skip<KIND>(P, k)) return;
  const int nv = det_nv<KIND>(P, k);
  const int npg = P.nplanes_global;
  double* all = const_cast<double*>(P.det_all);
  for (int v = threadIdx.x; v < nv; v += DET_THREADS) red[v] = det_fold(all + (size_t)v * npg, npg);
  __syncthreads();
  det_finish_dispatch<KIND>(P, k, red);
}

// End of an Arnoldi cycle (the inner loop stopped in fin_sweep_c): back-
// substitution of the rotated Hessenberg system (solve_least_squares,
// gmres.cpp:92-107; same row-oriented summation order, from a shared-memory
// copy of the triangle) and the x-update coefficients
//   x += M^{-1} V y = V y + U (|mu| T^{-1} U^T V y - U^T V y).
// One block; dynamic smem: k*k triangle + y + tz.
__global__ void __launch_bounds__(256) k_end_cycle(Params P) {
  extern __shared__ double sm[];
  __shared__ int s_ok;
  GState* g = P.g;
  if (g->error) return;
  const int k = g->steps, m = P.m;
  double* R = sm;             // k x k, column-major (upper triangle used)
  double* y = R + k * k;      // k
  double* tz = y + k;         // MAX_R1
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int i = e % k, j = e / k;
    R[e] = i <= j ? P.h_rot[(size_t)j * (m + 1) + i] : 0.0;
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) y[i] = P.gv[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    s_ok = 1;
    for (int i = k - 1; i >= 0; --i) {
      const double d = R[i + i * k];
      if (d == 0.0) {
        set_error(P, 3 /*ESINGULAR*/, g->restart, i);
        s_ok = 0;
        break;
      }
      double s = y[i];
      for (int j = i + 1; j < k; ++j) s -= R[i + j * k] * y[j];
      y[i] = s / d;
    }
  }
  __syncthreads();
  if (!s_ok) return;
  const int r = P.d->r;
  for (int l = threadIdx.x; l < r; l += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += y[j] * P.tU[(size_t)j * P.R1 + l];
    tz[l] = s;
  }
  __syncthreads();
  if (r > 0) defl_coeffs_par(P, r, tz, P.cx);
  for (int j = threadIdx.x; j < k; j += blockDim.x) P.xc[j] = y[j] * P.s[j];
}

// ---------------------------------------------------------------------------
// Restart harvest, dense part (deflation.cpp:15-82, 232-248): power iteration
// for the running |mu|, inverse power iteration (explicit H^-1 by
// Gauss-Jordan) for the smallest Ritz pair, lift coefficients for u = V z.
__device__ __forceinline__ void hmatvec(const double* M, int k, const double* z, double* out) {
  // two threads per row, halves of the column range combined by a shuffle
  const int t = threadIdx.x, i = t >> 1, half = t & 1;
  double s = 0.0;
  if (i < k) {
    const int j0 = half ? (k >> 1) : 0, j1 = half ? k : (k >> 1);
    for (int j = j0; j < j1; ++j) s += M[i + j * k] * z[j];
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  if (i < k && !half) out[i] = s;
}

// Row sums of an 8-row x 32-lane tile: a[r] = this lane's partial of row r.
// Transposing butterfly: lane l ends with the sum over all lanes of row
// r(l) = 4 b4 + 2 b3 + b2 (b = the bits of l); 9 shuffles for 8 sums, fixed order.
__device__ __forceinline__ double rowsum8(const double (&a)[8], int lane) {
  double b[4], c[2];
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    b[q] = (h16 ? a[q + 4] : a[q]) + __shfl_xor_sync(0xffffffffu, h16 ? a[q] : a[q + 4], 16);
#pragma unroll
  for (int q = 0; q < 2; ++q)
    c[q] = (h8 ? b[q + 2] : b[q]) + __shfl_xor_sync(0xffffffffu, h8 ? b[q] : b[q + 2], 8);
  double d = (h4 ? c[1] : c[0]) + __shfl_xor_sync(0xffffffffu, h4 ? c[0] : c[1], 4);
  d += __shfl_xor_sync(0xffffffffu, d, 2);
  d += __shfl_xor_sync(0xffffffffu, d, 1);
  return d;
}
__device__ __forceinline__ int rowsum8_row(int lane) {
  return ((lane >> 2) & 1) | (((lane >> 3) & 1) << 1) | (((lane >> 4) & 1) << 2);
}
// sum over the 8 row-owner lanes (lane % 4 == 0) of a warp; result in lane 0
__device__ __forceinline__ double owners_sum(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 16);
  return v;
}

// largest_ritz_value (deflation.cpp:57-82) for k <= 64 with the whole CTA:
// warp w owns rows 8w..8w+7, lane the columns lane and lane + 32, the H
// entries live in registers (16 per lane); one matvec = 16 FMAs + one
// transposing butterfly per warp, the three sums y.y, y.Hy, Hy.Hy one smem
// combine over the 8 warps; two CTA barriers per iteration.  Same iteration
// as the one-warp version below: y = H z unnormalised, theta = y.Hy / y.y,
// residual |Hy - theta y| / |y| (exact pass only near convergence).
__device__ void ritz_power8(const Params& P, int k, int m, double tol, double scale,
                            double skip_above) {
  __shared__ double sy[2][64];
  __shared__ double spart[RITZ_THREADS / 32][4];
  DState* d = P.d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t hld = (size_t)m + 1;
  double h[8][2];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int i = 8 * warp + r, j = lane + 32 * c;
      h[r][c] = (i < k && j < k && j + 1 >= i) ? __ldcg(P.h_orig + (size_t)j * hld + i) : 0.0;
    }
  const int row = 8 * warp + rowsum8_row(lane);
  const bool owner = (lane & 3) == 0 && row < k;
  for (int i = threadIdx.x; i < 128; i += blockDim.x) (&sy[0][0])[i] = 0.0;
  __syncthreads();
  // y_1 = H z_0, z_0 = 1 / sqrt(k)
  {
    const double z0 = 1.0 / sqrt((double)k);
    double a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = h[r][0] * (lane < k ? z0 : 0.0) + h[r][1] * (lane + 32 < k ? z0 : 0.0);
    const double hy = rowsum8(a, lane);
    if (owner) sy[0][row] = hy;
  }
  __syncthreads();
  bool have = false, conv = false, broke = false;
  double val = 0.0;
  int cur = 0;
  for (int it = 0; it < d->pow_maxit; ++it) {
    const double y0 = sy[cur][lane], y1 = sy[cur][lane + 32];
    double a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = h[r][0] * y0 + h[r][1] * y1;
    const double hy = rowsum8(a, lane);
    const double yi = owner ? sy[cur][row] : 0.0;
    double p = owner ? yi * yi : 0.0, q = owner ? yi * hy : 0.0, hh = owner ? hy * hy : 0.0;
    p = owners_sum(p);
    q = owners_sum(q);
    hh = owners_sum(hh);
    if (lane == 0) {
      spart[warp][0] = p;
      spart[warp][1] = q;
      spart[warp][2] = hh;
    }
    __syncthreads();
    double yy = 0.0, yhy = 0.0, hsq = 0.0;
#pragma unroll
    for (int w = 0; w < RITZ_THREADS / 32; ++w) {
      yy += spart[w][0];
      yhy += spart[w][1];
      hsq += spart[w][2];
    }
    const double nz = sqrt(yy);
    if (!isfinite(nz) || nz == 0.0) {
      broke = true;
      break;
    }
    const double theta = yhy / yy;
    const bool exact = !(hsq / yy - theta * theta > skip_above);
    if (owner) sy[cur ^ 1][row] = hy / nz;  // H z_i for the next iteration
    if (exact) {
      const double t = hy - theta * yi;
      const double e = owners_sum(owner ? t * t : 0.0);
      if (lane == 0) spart[warp][3] = e;
    }
    __syncthreads();
    double resid = INFINITY;
    if (exact) {
      double e = 0.0;
#pragma unroll
      for (int w = 0; w < RITZ_THREADS / 32; ++w) e += spart[w][3];
      resid = sqrt(e / yy);
    }
    val = theta;
    have = true;
#if PGM_TAIL_TIMING
    if (threadIdx.x == 0) atomicAdd(&g_tail_ns[13], 1ull);
#endif
    if (resid <= tol * scale) {
      conv = true;
      break;
    }
    cur ^= 1;
  }
  const bool ok = conv || (!broke && have);
  if (threadIdx.x == 0 && ok && isfinite(val) && fabs(val) > fabs(d->mu)) d->mu = val;  // observe_ritz
}

__global__ void __launch_bounds__(RITZ_THREADS) k_ritz(Params P, int hcopy) {
  extern __shared__ double sm[];
  GState* g = P.g;
  DState* d = P.d;
  if (g->error || !g->harvest) return;
  const int k = g->steps;
  const int tid = threadIdx.x;
  __shared__ double s_red[32];
  // a new harvest: the previous truncation's rotation has been applied; a
  // rejected push this time must not re-apply it (k_rotate runs regardless)
  // two CTAs: CTA 1 runs the power iteration (running |mu|), CTA 0 the
  // Gauss-Jordan inverse and the inverse iteration (smallest Ritz pair)
  const bool main_cta = blockIdx.x == 0;
  if (tid == 0 && main_cta) d->rotate = 0;
  if (k == 0) {
    if (tid == 0 && main_cta) {
      d->skipped++;
      d->push_ok = 0;
      d->theta = __longlong_as_double(0x7ff8000000000000LL);
    }
    return;
  }
  const int m = g->m;
  double* H = sm;               // k*k
  double* B = H + k * k;        // k*k (inverse)
  double* z = B + k * k;        // k
  double* nx = z + k;           // k
  double* hz = nx + k;          // k
  double* colc = hz + k;        // k
  __shared__ int s_piv;
  // hcopy: a third k*k smem block keeps H for warp 0's matvecs while the
  // Gauss-Jordan inverse consumes the first one (host: when 3 m^2 fits)
  double* H2 = colc + k;
  auto load_h = [&]() {
    for (int e = tid; e < k * k; e += blockDim.x) {
      const int i = e % k, j = e / k;
      const int top = min(k - 1, j + 1);
      const double h = (i <= top) ? P.h_orig[(size_t)j * (m + 1) + i] : 0.0;
      H[e] = h;
      if (hcopy) H2[e] = h;
    }
  };
  load_h();
  __syncthreads();
  double fr = 0.0;
  for (int e = tid; e < k * k; e += blockDim.x) fr += H[e] * H[e];
  const double scale = sqrt(block_sum(fr, s_red));
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  if (!(scale > 0.0) || !isfinite(scale)) {
    if (tid == 0 && main_cta) {
      d->skipped++;
      d->push_ok = 0;
      d->theta = nan;
    }
    return;
  }
  const double tol = d->inv_tol;
  const int warp = tid >> 5, lane = tid & 31;
#if PGM_TAIL_TIMING
  const unsigned long long rt0 = gtimer();
  int n_pow = 0, n_inv = 0;
#endif
  // H (Hessenberg block, column-major i + j (m+1)) read by lane-per-row
  // matvecs straight from P.h_orig (L1-resident after the first sweep): the
  // smem copy is consumed by the Gauss-Jordan inverse that runs meanwhile.
  const double* hg = P.h_orig;
  const size_t hld = (size_t)m + 1;
  constexpr int RQ = (MAX_M + 31) / 32;  // rows per lane
  // y = H v, lane per row (Hessenberg: H(i, j) = 0 for j < i - 1), four
  // independent accumulators so the loads of consecutive columns overlap
  auto hmv_global = [&](const double* v, double (&out)[RQ]) {
#pragma unroll
    for (int q = 0; q < RQ; ++q) {
      const int i = lane + 32 * q;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      if (i < k) {
        int j = i > 0 ? i - 1 : 0;
        if (hcopy) {
          const double* hr = H2 + i;
          double a4 = 0.0, a5 = 0.0, a6 = 0.0, a7 = 0.0;
          for (; j + 8 <= k; j += 8) {
            a0 += hr[j * k] * v[j];
            a1 += hr[(j + 1) * k] * v[j + 1];
            a2 += hr[(j + 2) * k] * v[j + 2];
            a3 += hr[(j + 3) * k] * v[j + 3];
            a4 += hr[(j + 4) * k] * v[j + 4];
            a5 += hr[(j + 5) * k] * v[j + 5];
            a6 += hr[(j + 6) * k] * v[j + 6];
            a7 += hr[(j + 7) * k] * v[j + 7];
          }
          for (; j < k; ++j) a0 += hr[j * k] * v[j];
          a0 += a4;
          a1 += a5;
          a2 += a6;
          a3 += a7;
        } else {
          for (; j + 4 <= k; j += 4) {
            a0 += __ldg(hg + (size_t)j * hld + i) * v[j];
            a1 += __ldg(hg + (size_t)(j + 1) * hld + i) * v[j + 1];
            a2 += __ldg(hg + (size_t)(j + 2) * hld + i) * v[j + 2];
            a3 += __ldg(hg + (size_t)(j + 3) * hld + i) * v[j + 3];
          }
          for (; j < k; ++j) a0 += __ldg(hg + (size_t)j * hld + i) * v[j];
        }
      }
      out[q] = (a0 + a1) + (a2 + a3);
    }
  };
  auto wsum0 = [&](double v) { return __shfl_sync(0xffffffffu, warp_sum(v), 0); };
  // three warp sums with interleaved shuffle chains (lane 0's values broadcast)
  auto wsum3 = [&](double& a, double& b, double& c) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    a = __shfl_sync(0xffffffffu, a, 0);
    b = __shfl_sync(0xffffffffu, b, 0);
    c = __shfl_sync(0xffffffffu, c, 0);
  };
  // |Hz - theta z|^2 = |Hy|^2/|y|^2 - theta^2 (Rayleigh quotient theta): from
  // the same sums, with rounding error <= ~8 eps scale^2.  Far from
  // convergence this proves resid > tol * scale and the exact residual pass
  // (a second dependent warp reduction) is skipped; near it, the exact
  // formula decides, exactly as deflation.cpp:48-52 / 74-78.
  const double skip_above = fmax(64.0 * 2.220446049250313e-16 * scale * scale,
                                 4.0 * (tol * scale) * (tol * scale));
  if (!main_cta) {
#if PGM_TAIL_TIMING
    const unsigned long long pt0 = gtimer();
#endif
    if (k <= 64) ritz_power8(P, k, m, tol, scale, skip_above);
#if PGM_TAIL_TIMING
    if (tid == 0) atomicAdd(&g_tail_ns[4], gtimer() - pt0);
#endif
    if (k <= 64 || warp != 0) return;
  }
  if (!main_cta) {
    // ---- largest_ritz_value: power iteration (deflation.cpp:57-82), one warp,
    // shuffles only.  y = H z_{i-1} unnormalised; theta = y.Hy / y.y = z.Hz;
    // residual |Hy - theta y| / |y| = |Hz - theta z|.
    double* yv = nx;  // smem broadcast copy of y (warp 0 only)
    double y[RQ], hy[RQ];
    for (int i = lane; i < k; i += 32) z[i] = 1.0 / sqrt((double)k);
    __syncwarp();
    hmv_global(z, y);
#pragma unroll
    for (int q = 0; q < RQ; ++q)
      if (lane + 32 * q < k) yv[lane + 32 * q] = y[q];
    __syncwarp();
    bool have = false, conv = false, broke = false;
    double val = 0.0;
    for (int it = 0; it < d->pow_maxit; ++it) {
#if PGM_TAIL_TIMING
      ++n_pow;
#endif
      hmv_global(yv, hy);
      double p = 0.0, qq = 0.0, hh = 0.0;
#pragma unroll
      for (int q = 0; q < RQ; ++q)
        if (lane + 32 * q < k) {
          p += y[q] * y[q];
          qq += y[q] * hy[q];
          hh += hy[q] * hy[q];
        }
      wsum3(p, qq, hh);
      const double yy = p, yhy = qq;
      const double nz = sqrt(yy);
      if (!isfinite(nz) || nz == 0.0) {
        broke = true;
        break;
      }
      const double theta = yhy / yy;
      const bool exact = !(hh / yy - theta * theta > skip_above);
      double e = 0.0;
      __syncwarp();
#pragma unroll
      for (int q = 0; q < RQ; ++q)
        if (lane + 32 * q < k) {
          const double t = hy[q] - theta * y[q];
          e += t * t;
          y[q] = hy[q] / nz;  // H z_i for the next iteration
          yv[lane + 32 * q] = y[q];
        }
      const double resid = exact ? sqrt(wsum0(e) / yy) : INFINITY;
      __syncwarp();
      val = theta;
      have = true;
      if (resid <= tol * scale) {
        conv = true;
        break;
      }
    }
    const bool ok = conv || (!broke && have);
    if (lane == 0 && ok && isfinite(val) && fabs(val) > fabs(d->mu)) d->mu = val;  // observe_ritz
#if PGM_TAIL_TIMING
    if (lane == 0) {
      atomicAdd(&g_tail_ns[4], gtimer() - rt0);
      atomicAdd(&g_tail_ns[13], (unsigned long long)n_pow);
    }
#endif
    return;
  } else if (warp != 0) {
    // ---- meanwhile warps 1..7: H^-1 by Gauss-Jordan with partial pivoting,
    // [H | I] -> [I | H^-1] in smem (named barrier 1 over these 224 threads)
    const int t7 = tid - 32, n7 = RITZ_THREADS - 32;
    auto gsync = [] { asm volatile("bar.sync 1, %0;" ::"n"(RITZ_THREADS - 32)); };
    for (int e = t7; e < k * k; e += n7) B[e] = ((e % k) == (e / k)) ? 1.0 : 0.0;
    const int i0 = t7 % k, a0 = t7 / k, di = n7 % k, da = n7 / k;
    gsync();
    for (int c = 0; c < k; ++c) {
      if (warp == 1) {
        double best = -1.0;
        int bi = c;
        for (int i = c + lane; i < k; i += 32) {
          const double a = fabs(H[i + c * k]);
          if (a > best) {
            best = a;
            bi = i;
          }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
          }
        }
        if (lane == 0) s_piv = bi;
      }
      gsync();
      const int pv = s_piv;
      if (pv != c) {
        for (int j = t7; j < 2 * k; j += n7) {
          double* M = j < k ? H : B;
          const int jj = j < k ? j : j - k;
          const double t = M[c + jj * k];
          M[c + jj * k] = M[pv + jj * k];
          M[pv + jj * k] = t;
        }
      }
      gsync();
      const double piv = H[c + c * k];
      gsync();
      for (int j = t7; j < 2 * k; j += n7) {
        double* M = j < k ? H : B;
        const int jj = j < k ? j : j - k;
        M[c + jj * k] /= piv;
      }
      for (int i = t7; i < k; i += n7) colc[i] = H[i + c * k];
      gsync();
      // H columns <= c are unit vectors by now (and H itself is not read
      // after the inverse): only H columns c+1..k-1 and all of B change
      // (row swaps move B's unit entries, so any B column can have a
      // nonzero in row c); (row, column) stepped incrementally, no integer
      // division per element
      {
        const int nh = k - 1 - c;
        int i = i0, a = a0;
        for (int e = t7; e < k * (nh + k); e += n7) {
          if (i != c) {
            double* M = a < nh ? H + (size_t)(c + 1 + a) * k : B + (size_t)(a - nh) * k;
            M[i] -= colc[i] * M[c];
          }
          i += di;
          a += da;
          if (i >= k) {
            i -= k;
            ++a;
          }
        }
      }
      gsync();
    }
  }
  __syncthreads();
#if PGM_TAIL_TIMING
  const unsigned long long rt2 = gtimer();
#endif
  // ---- smallest_ritz_pair: inverse power iteration (deflation.cpp:31-54),
  // warp 0: y = H^-1 z (smem, lane per row), hy = H y (global); y.y and y.hy
  // in one pass, then the residual while z <- y / |y| is written.
  if (warp != 0) return;
  bool conv = false;
  double val = 0.0;
  {
    for (int i = lane; i < k; i += 32) z[i] = 1.0 / sqrt((double)k);
    __syncwarp();
    double y[RQ], hy[RQ];
    for (int it = 0; it < d->inv_maxit; ++it) {
#pragma unroll
      for (int q = 0; q < RQ; ++q) {
        const int i = lane + 32 * q;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if (i < k) {
          int j = 0;
          for (; j + 4 <= k; j += 4) {
            a0 += B[i + j * k] * z[j];
            a1 += B[i + (j + 1) * k] * z[j + 1];
            a2 += B[i + (j + 2) * k] * z[j + 2];
            a3 += B[i + (j + 3) * k] * z[j + 3];
          }
          for (; j < k; ++j) a0 += B[i + j * k] * z[j];
          nx[i] = (a0 + a1) + (a2 + a3);
        }
        y[q] = (a0 + a1) + (a2 + a3);
      }
      __syncwarp();
      hmv_global(nx, hy);
      double p = 0.0, qq = 0.0, hh = 0.0;
#pragma unroll
      for (int q = 0; q < RQ; ++q)
        if (lane + 32 * q < k) {
          p += y[q] * y[q];
          qq += y[q] * hy[q];
          hh += hy[q] * hy[q];
        }
      wsum3(p, qq, hh);
      const double yy = p, yhy = qq;
      const double nz = sqrt(yy);
      if (!isfinite(nz) || nz == 0.0) break;
      const double theta = yhy / yy;
      const bool exact = !(hh / yy - theta * theta > skip_above);
      double e = 0.0;
#pragma unroll
      for (int q = 0; q < RQ; ++q)
        if (lane + 32 * q < k) {
          const double t = hy[q] - theta * y[q];
          e += t * t;
          z[lane + 32 * q] = y[q] / nz;
        }
      const double resid = exact ? sqrt(wsum0(e) / yy) : INFINITY;
      __syncwarp();
      val = theta;
#if PGM_TAIL_TIMING
      ++n_inv;
#endif
      if (resid <= tol * scale) {
        conv = true;
        break;
      }
    }
  }
#if PGM_TAIL_TIMING
  if (lane == 0) {
    const unsigned long long rt3 = gtimer();
    atomicAdd(&g_tail_ns[5], rt2 - rt0);   // until Gauss-Jordan done
    atomicAdd(&g_tail_ns[6], rt3 - rt2);   // inverse iteration
    atomicAdd(&g_tail_ns[7], (unsigned long long)n_inv);
    atomicAdd(&g_tail_ns[8], 1ull);
    atomicAdd(&g_tail_ns[13], (unsigned long long)n_pow);
  }
#endif
  if (conv) {
    for (int l = lane; l < k; l += 32) P.zl[l] = z[l] * P.s[l];
    if (lane == 0) {
      d->theta = val;
      if (d->r >= P.R1) {  // a failed truncation left the basis full (deflation.cpp:132-135)
        d->skipped++;
        d->push_ok = 0;
      } else {
        d->push_ok = 1;
      }
    }
  } else if (tid == 0) {
    d->skipped++;
    d->push_ok = 0;
    d->theta = nan;
  }
}

// U <- U Q, AU <- AU Q after truncation (deflation.cpp:216-221); block 0 also
// appends the DeflationRecord of this restart (deflation.cpp:262).
template <bool RECORD>
__global__ void __launch_bounds__(256) k_rotate(Params P) {
  GState* g = P.g;
  DState* d = P.d;
  if (RECORD) {
    if (g->error || !g->harvest) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const int h = d->n_hist;
      if (h < d->hist_cap) {
        P.hist_restart[h] = (uint32_t)g->restart;
        P.hist_r[h] = (uint32_t)d->r;
        P.hist_mu[h] = d->mu;
        P.hist_theta[h] = d->theta;
      }
      d->n_hist = h + 1;
    }
  }
  if (!d->rotate) return;
  const int r0 = d->r0, r = d->r, R1 = P.R1;
  // q stored l-major with the output index j contiguous (padded to even):
  // one LDS.128 gives two coefficients; each thread rotates a PAIR of rows
  // (double2 loads), so every coefficient load feeds four FMAs
  constexpr int QP = MAX_R1 + 1 + (MAX_R1 + 1) % 2;
  __shared__ __align__(16) double q[MAX_R1 * QP];
  for (int e = threadIdx.x; e < r0 * QP; e += blockDim.x) {
    const int l = e / QP, j = e % QP;
    q[e] = (j < r) ? P.Q[l + (size_t)j * R1] : 0.0;
  }
  __syncthreads();
  const size_t npair = ((size_t)P.n + 1) / 2;
  for (size_t pr = blockIdx.x * (size_t)blockDim.x + threadIdx.x; pr < npair;
       pr += (size_t)gridDim.x * blockDim.x) {
    const size_t row = 2 * pr;
    const bool pair = row + 1 < (size_t)P.n;
#pragma unroll 1
    for (int which = 0; which < 2; ++which) {
      double* base = (which == 0 ? P.U : P.AU) + P.lo + row;
      double2 in[MAX_R1];
#pragma unroll
      for (int l = 0; l < MAX_R1; ++l)
        if (l < r0) {
          const double* src = base + (size_t)l * P.ld;
          in[l] = pair ? *reinterpret_cast<const double2*>(src) : make_double2(src[0], 0.0);
        }
      // output columns j, j+1 at a time: one LDS.128 of coefficients feeds
      // four FMAs (two rows x two outputs); the j loop stays a runtime loop
      // so the only register array is in[] (compile-time indices)
      for (int j = 0; j < r; j += 2) {
        double x0 = 0.0, y0 = 0.0, x1 = 0.0, y1 = 0.0;
#pragma unroll
        for (int l = 0; l < MAX_R1; ++l)
          if (l < r0) {
            const double2 qq = *reinterpret_cast<const double2*>(q + l * QP + j);
            x0 += in[l].x * qq.x;
            y0 += in[l].y * qq.x;
            x1 += in[l].x * qq.y;
            y1 += in[l].y * qq.y;
          }
        double* d0 = base + (size_t)j * P.ld;
        if (pair) *reinterpret_cast<double2*>(d0) = make_double2(x0, y0);
        else d0[0] = x0;
        if (j + 1 < r) {
          double* d1 = d0 + P.ld;
          if (pair) *reinterpret_cast<double2*>(d1) = make_double2(x1, y1);
          else d1[0] = x1;
        }
      }
    }
  }
}

__global__ void k_clear_rotate(DState* d) { d->rotate = 0; }

// Standalone Deflator::truncate() (deflation.cpp:186-225) then refresh.
__global__ void k_truncate_once(Params P) {
  if (threadIdx.x != 0) return;
  DState* d = P.d;
  const int r0 = d->r;
  q_identity(P, r0);
  d->trunc_fail = 0;
  const int r = truncate_drop(P, r0, r0);
  d->r0 = r0;
  d->rotate = (r != r0);
  d->r = r;
  refresh_tinv(P);
}

__global__ void k_observe(DState* d, double v) {
  if (isfinite(v) && fabs(v) > fabs(d->mu)) d->mu = v;
}

// ---------------------------------------------------------------------------
// CSR -> SELL conversion: one warp per slice.
// SELL layout of one 512-row tile (one block): stable sort of the rows by
// length, descending (cub::BlockRadixSort is stable; padding rows past n sort
// after every real row), 32 rows per slice.  Writes lane_len / lane_row and
// the slice sizes into sptr[s] (32 * length rounded up to a multiple of 4;
// exclusive-scanned afterwards).  bad: bit 0 = row_ptr[0] != 0 or
// row_ptr[n] != nnz, bit 1 = row_ptr decreasing.
__global__ void __launch_bounds__(256) k_sell_layout(const unsigned* rp, int n,
                                                     unsigned long long nnz, unsigned* lane_len,
                                                     unsigned short* lane_row,
                                                     unsigned long long* sptr, int* bad) {
  constexpr int IPT = TILE / 256;  // rows per thread
  using Sort = cub::BlockRadixSort<unsigned, 256, IPT, int>;
  __shared__ typename Sort::TempStorage tmp;
  __shared__ unsigned s_len[TILE];
  const int tile = blockIdx.x;
  const int r0 = tile * TILE;
  unsigned key[IPT];
  int val[IPT];
  for (int q = 0; q < IPT; ++q) {
    const int i = threadIdx.x * IPT + q;  // blocked arrangement: keeps the original order
    const int row = r0 + i;
    unsigned len = 0;
    if (row < n) {
      const unsigned a = rp[row], b = rp[row + 1];
      if (b < a) atomicOr(bad, 2);
      len = b - a;
    }
    // descending by length; padding rows get the lowest key (after empty rows)
    key[q] = row < n ? len + 1u : 0u;
    val[q] = i;
  }
  if (tile == 0 && threadIdx.x == 0 && (rp[0] != 0u || (unsigned long long)rp[n] != nnz))
    atomicOr(bad, 1);
  Sort(tmp).SortDescending(key, val);
  for (int q = 0; q < IPT; ++q) {
    const int j = threadIdx.x * IPT + q;  // sorted position = slice * 32 + lane
    const int row = r0 + val[q];
    const bool real = key[q] != 0u;
    const unsigned len = real ? key[q] - 1u : 0u;
    lane_len[(size_t)tile * TILE + j] = len;
    lane_row[(size_t)tile * TILE + j] = real ? (unsigned short)val[q] : (unsigned short)0xFFFF;
    s_len[j] = len;
    (void)row;
  }
  __syncthreads();
  if (threadIdx.x < SPT) {
    unsigned m = 0;
    for (int l = 0; l < 32; ++l) m = max(m, s_len[threadIdx.x * 32 + l]);
    sptr[(size_t)tile * SPT + threadIdx.x] = 32ull * ((m + 3u) / 4u * 4u);
  }
}

// 16-bit column-delta compression of a SELL matrix (see spmv_tile<true>).
// k_sell_delta_max: largest delta between consecutive entries of a row
// (unsigned: a descending pair counts as huge and disables compression).
__global__ void k_sell_delta_max(Sell A, int nslices, unsigned* out) {
  const int lane = threadIdx.x & 31;
  const size_t s = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  if (s >= (size_t)nslices) return;
  const unsigned long long base = A.sptr[s];
  const int len = (int)A.lane_len[s * 32 + lane];
  unsigned m = 0, prev = 0;
  for (int t = 0; t < len; ++t) {
    const unsigned c = A.col[base + (size_t)(t >> 2) * 128 + lane * 4 + (t & 3)];
    if (t > 0) m = max(m, c - prev);
    prev = c;
  }
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 16));
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 8));
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 4));
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 2));
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 1));
  if (lane == 0) atomicMax(out, m);
}

__global__ void k_sell_compress(Sell A, int nslices, unsigned short* col16, unsigned* lane_base) {
  const int lane = threadIdx.x & 31;
  const size_t s = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  if (s >= (size_t)nslices) return;
  const unsigned long long base = A.sptr[s];
  const int L = (int)((A.sptr[s + 1] - base) >> 5);
  const int len = (int)A.lane_len[s * 32 + lane];
  unsigned prev = len > 0 ? A.col[base + lane * 4] : 0u;
  lane_base[s * 32 + lane] = prev;
  for (int t = 0; t < L; ++t) {
    const size_t idx = base + (size_t)(t >> 2) * 128 + lane * 4 + (t & 3);
    unsigned d = 0;
    if (t < len) {
      const unsigned c = A.col[idx];
      d = c - prev;
      prev = c;
    }
    col16[idx] = (unsigned short)d;
  }
}

// Rows that read halo columns (global column < rb or >= re; columns ascending
// per row): out[0] = last such row below, out[1] = first such row above.
// Halo tiles (world > 1): the last row whose first column lies below the own
// block and the first row whose last column lies above it, from the SELL
// layout (32-bit local column ids, rows sorted ascending: entry t = 0 is the
// row's first column, t = len - 1 its last).  Own local columns: [lo, hi).
__global__ void k_halo_rows_sell(Sell A, int nslices, unsigned lo, unsigned hi, int* out) {
  const int lane = threadIdx.x & 31;
  const size_t s = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  if (s >= (size_t)nslices) return;
  const int len = (int)A.lane_len[s * 32 + lane];
  const unsigned short ro = A.lane_row[s * 32 + lane];
  if (ro == 0xFFFF || len == 0) return;
  const unsigned long long base = A.sptr[s];
  const int row = (int)((s / SPT) * TILE + ro);
  const int tl = len - 1;
  const unsigned c0 = A.col[base + lane * 4];
  const unsigned c1 = A.col[base + (size_t)(tl >> 2) * 128 + lane * 4 + (tl & 3)];
  if (c0 < lo) atomicMax(&out[0], row);
  if (c1 >= hi) atomicMin(&out[1], row);
}

// CSR -> SELL gather for slices [s0, s0 + count): entry t of the lane that
// holds row `row` is CSR entry rp[row] + t, read from ci / v at offset
// (rp[row] + t - csr_base) — the caller's arrays (csr_base = 0) or a staged
// chunk of them.  Padding entries get value 0 and column 0.
__global__ void k_csr_to_sell(Sell A, double* val, unsigned* col, const unsigned* rp,
                              const unsigned* ci, const double* v, unsigned col_shift,
                              int s0, int count, unsigned long long csr_base, int write_cols) {
  const int lane = threadIdx.x & 31;
  const size_t sl = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  if (sl >= (size_t)count) return;
  const size_t s = s0 + sl;
  const unsigned long long base = A.sptr[s];
  const int L = (int)((A.sptr[s + 1] - base) >> 5);
  const int len = (int)A.lane_len[s * 32 + lane];
  const unsigned short ro = A.lane_row[s * 32 + lane];
  const size_t tile = s / SPT;
  const size_t row = tile * TILE + ro;
  const size_t start = (ro != 0xFFFF) ? (size_t)rp[row] - csr_base : 0;
  for (int t = 0; t < L; ++t) {
    const size_t idx = base + (size_t)(t >> 2) * 128 + lane * 4 + (t & 3);
    if (t < len) {
      val[idx] = v[start + t];
      if (write_cols) col[idx] = ci[start + t] - col_shift;
    } else {
      val[idx] = 0.0;
      if (write_cols) col[idx] = 0u;
    }
  }
}

// out[i] = in[i] (own rows) — halo-free copy helper
__global__ void k_copy(double* __restrict__ out, const double* __restrict__ in, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}


// ---------------------------------------------------------------------------
// Newton driver scalars (newton.cpp:54,72-73): per-block partials of
// sum rhs^2 (rhs = -R(u)) and of max|delta| with u += delta fused in; a
// one-block kernel combines the partials in block order (deterministic).
__global__ void __launch_bounds__(256) k_newton_partials(const double* __restrict__ rhs,
                                                         const double* __restrict__ delta,
                                                         double* __restrict__ u, int n,
                                                         double* part) {
  __shared__ double s_sum[8], s_max[8];
  double sq = 0.0, mx = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (rhs) sq += rhs[i] * rhs[i];
    if (delta) {
      const double d = delta[i];
      u[i] = u[i] + d;  // ex.axpy(1.0, delta, u)
      mx = fmax(mx, fabs(d));
    }
  }
  sq = warp_sum(sq);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_sum[warp] = sq;
    s_max[warp] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += s_sum[w];
      b = fmax(b, s_max[w]);
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

__global__ void k_newton_final(const double* part, int G, double* out, int nv, int rank) {
  if (threadIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int q = 0; q < G; ++q) {
    a += part[2 * q];
    b = fmax(b, part[2 * q + 1]);
  }
  for (int v = 0; v < nv; ++v) out[v] = 0.0;
  out[0] = a;
  out[1 + rank] = b;
}

}  // namespace pgm
