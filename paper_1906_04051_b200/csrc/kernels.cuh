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

#include "common.cuh"
#include "finish.cuh"

namespace pgm {

// ---------------------------------------------------------------------------
// SELL-32 with a per-tile length sort (sigma = TILE).
struct Sell {
  const unsigned long long* sptr;  // [nslices + 1] entry offsets (multiples of 32)
  const unsigned* lane_len;        // [nslices * 32] true row length
  const unsigned short* lane_row;  // [nslices * 32] row within tile, 0xFFFF = empty lane
  const double* val;
  const unsigned* col;             // local column (index into the padded x buffer)
  int ntiles;
  int n;
};

__device__ __forceinline__ void spmv_tile(const Sell& A, const double* __restrict__ x, int tile,
                                          double* ys) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int sl = warp; sl < SPT; sl += nw) {
    const size_t s = (size_t)tile * SPT + sl;
    const unsigned long long base = A.sptr[s];
    const int L = (int)((A.sptr[s + 1] - base) >> 5);
    if (L == 0) continue;
    const int len = (int)A.lane_len[s * 32 + lane];
    const unsigned short ro = A.lane_row[s * 32 + lane];
    const double* vp = A.val + base + lane;
    const unsigned* cp = A.col + base + lane;
    double acc = 0.0;
    for (int t = 0; t < L; t += SPMV_UNROLL) {
      double v[SPMV_UNROLL];
      unsigned c[SPMV_UNROLL];
#pragma unroll
      for (int u = 0; u < SPMV_UNROLL; ++u) {
        if (t + u < L) {
          v[u] = __ldcs(vp + (size_t)(t + u) * 32);
          c[u] = __ldcs(cp + (size_t)(t + u) * 32);
        }
      }
      double xv[SPMV_UNROLL];
#pragma unroll
      for (int u = 0; u < SPMV_UNROLL; ++u) xv[u] = (t + u < len) ? __ldg(x + c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < SPMV_UNROLL; ++u)
        if (t + u < len) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
    }
    if (ro != 0xFFFF) ys[ro] = acc;
  }
}

// ---- SpMV epilogues ---------------------------------------------------------------
// y = A x, nothing else (pgm_spmv).
struct PlainEpi {
  const double* xin;
  double* y;  // own region
  __device__ bool skip(const Params&) const { return false; }
  __device__ int nvals(const Params&) const { return 0; }
  __device__ void prologue(const Params&, double*) const {}
  __device__ void tile(const Params&, int row0, int rows, double* ys, double*, double*) const {
    for (int i = threadIdx.x; i < rows; i += blockDim.x) y[row0 + i] = ys[i];
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
  __device__ void tile(const Params& P, int row0, int rows, double* ys, double* acc,
                       double* sm) const {
    const int r = P.d->r;
    const double sk = sm[0];
    double* w = P.V + (size_t)(k + 1) * P.ld + P.lo + row0;
    const double* au = P.AU + P.lo + row0;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) {
      double y = sk * ys[i];
      for (int l = 0; l < r; ++l) y += sm[1 + l] * au[(size_t)l * P.ld + i];
      w[i] = y;
      ys[i] = y;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int l = warp; l <= k; l += nw) {
      const double* vl = P.V + (size_t)l * P.ld + P.lo + row0;
      double a = 0.0;
      for (int i = lane; i < rows; i += 32) a += vl[i] * ys[i];
      acc[l * 32 + lane] += a;
    }
  }
  __device__ void finish(const Params& P, const double* red) const { fin_step_spmv(P, k, red); }
};

// Explicit residual r = b - A x into W_0; dots ||r||^2 and U_l . r.
struct ResidualEpi {
  int initial;
  __device__ bool skip(const Params& P) const { return P.g->error != 0 || (!initial && P.g->done); }
  __device__ int nvals(const Params& P) const { return 1 + P.d->r; }
  __device__ void prologue(const Params&, double*) const {}
  __device__ void tile(const Params& P, int row0, int rows, double* ys, double* acc,
                       double*) const {
    double* w = P.V + P.lo + row0;
    const double* b = P.b + P.lo + row0;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) {
      const double rv = b[i] + (-ys[i]);  // r = b; r += -1 * (A x)   (gmres.cpp:143-145)
      w[i] = rv;
      ys[i] = rv;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int nv = 1 + P.d->r;
    for (int v = warp; v < nv; v += nw) {
      double a = 0.0;
      if (v == 0) {
        for (int i = lane; i < rows; i += 32) a += ys[i] * ys[i];
      } else {
        const double* ul = P.U + (size_t)(v - 1) * P.ld + P.lo + row0;
        for (int i = lane; i < rows; i += 32) a += ul[i] * ys[i];
      }
      acc[v * 32 + lane] += a;
    }
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
  __device__ void tile(const Params& P, int row0, int rows, double* ys, double* acc,
                       double* sm) const {
    const int j = P.d->r;
    const double ps = sm[0];
    double* us = sm + 8;  // TILE doubles
    double* uj = P.U + (size_t)j * P.ld + P.lo + row0;
    double* auj = P.AU + (size_t)j * P.ld + P.lo + row0;
    const double* u = P.u + P.lo + row0;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) {
      const double un = u[i] * ps;
      const double an = ys[i] * ps;
      uj[i] = un;
      auj[i] = an;
      us[i] = un;
      ys[i] = an;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int nv = 2 * j + 1;
    for (int v = warp; v < nv; v += nw) {
      double a = 0.0;
      if (v < j) {  // U_l . AU_j
        const double* ul = P.U + (size_t)v * P.ld + P.lo + row0;
        for (int i = lane; i < rows; i += 32) a += ul[i] * ys[i];
      } else if (v == j) {  // U_j . AU_j
        for (int i = lane; i < rows; i += 32) a += us[i] * ys[i];
      } else {  // U_j . AU_l
        const double* al = P.AU + (size_t)(v - j - 1) * P.ld + P.lo + row0;
        for (int i = lane; i < rows; i += 32) a += us[i] * al[i];
      }
      acc[v * 32 + lane] += a;
    }
  }
  __device__ void finish(const Params& P, const double* red) const { fin_push_spmv(P, red); }
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
__device__ __forceinline__ const double* epi_input(const Params& P, const ResidualEpi&) {
  return P.x;
}
template <>
__device__ __forceinline__ const double* epi_input(const Params& P, const PushEpi&) {
  return P.u;
}

constexpr int EPI_SMALL = 8 + 64;  // prologue scratch (doubles) before the tile buffers

// dynamic smem: [small EPI_SMALL | us TILE (push only) | ys TILE | acc nv*32 | red nv]
template <class Epi>
__global__ void __launch_bounds__(SPMV_THREADS) k_spmv(Sell A, Params P, Epi E) {
  extern __shared__ double sm[];
  if (E.skip(P)) return;
  const int nv = E.nvals(P);
  double* small = sm;
  double* ys = sm + EPI_SMALL + TILE;
  double* acc = ys + TILE;
  double* red = acc + nv * 32;
  E.prologue(P, small);
  for (int i = threadIdx.x; i < nv * 32; i += blockDim.x) acc[i] = 0.0;
  __syncthreads();
  const double* x = epi_input(P, E);
  for (int tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x) {
    spmv_tile(A, x, tile, ys);
    __syncthreads();
    const int row0 = tile * TILE;
    const int rows = min(TILE, A.n - row0);
    E.tile(P, row0, rows, ys, acc, small);
    __syncthreads();
  }
  if (nv == 0) return;
  if (P.world > 1) {
    if (grid_reduce(acc, nv, P, red)) {
      for (int v = threadIdx.x; v < nv; v += blockDim.x) P.red_out[v] = red[v];
    }
    return;
  }
  if (grid_reduce(acc, nv, P, red)) {
    if (threadIdx.x == 0) E.finish(P, red);
  }
}

// ---------------------------------------------------------------------------
// Streaming sweeps over basis blocks.
enum SweepMode {
  SW_CGS2_B = 0,   // w1 = w - V h1 ; dots V^T w1 (staged)
  SW_CGS2_C = 1,   // w2 = w1 - V h2 ; ||w2||^2, U^T w2
  SW_XUPDATE = 2,  // x += V xc + U cx
  SW_PUSH1 = 3,    // u = V zl (or u given) ; ||u||^2, U^T u
  SW_PUSH2 = 4,    // u -= U proj ; U^T u (staged)
  SW_PUSH3 = 5,    // u -= U proj ; ||u||^2
  SW_DOTS_U = 6,   // U^T u only (apply)
  SW_AXPY_U = 7,   // u += U c only (apply)
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
  int skip;
};

template <int MODE>
__device__ __forceinline__ SweepSpec sweep_spec(const Params& P, int k) {
  SweepSpec S{};
  const GState* g = P.g;
  const DState* d = P.d;
  const size_t lo = P.lo;
  if (MODE == SW_CGS2_B) {
    S.skip = !g->active;
    S.in = S.out = P.V + (size_t)(k + 1) * P.ld + lo;
    S.Pv = P.V + lo;
    S.np = k + 1;
    S.a = P.coefA;
    S.Q = S.Pv;
    S.nq = k + 1;
    S.qstaged = 1;
  } else if (MODE == SW_CGS2_C) {
    S.skip = !g->active;
    S.in = S.out = P.V + (size_t)(k + 1) * P.ld + lo;
    S.Pv = P.V + lo;
    S.np = k + 1;
    S.a = P.coefB;
    S.Q = P.U + lo;
    S.nq = d->r;
    S.selfnorm = 1;
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
  if (MODE == SW_CGS2_B) fin_sweep_b(P, k, red);
  if (MODE == SW_CGS2_C) fin_sweep_c(P, k, red);
  if (MODE == SW_PUSH1) fin_push1(P, red);
  if (MODE == SW_PUSH2) fin_push2(P, red);
  if (MODE == SW_PUSH3) fin_push3(P, red);
  if (MODE == SW_DOTS_U) {
    for (int l = 0; l < P.d->r; ++l) P.proj[l] = red[l];
    defl_coeffs(P, P.d->r, P.proj, P.c);
  }
}

// dynamic smem: [a np | a2 np2 | os CH | acc nv*32 | red nv | stage np*CH]
template <int MODE>
__global__ void __launch_bounds__(SW_THREADS) k_sweep(Params P, int k) {
  extern __shared__ double sm[];
  const SweepSpec S = sweep_spec<MODE>(P, k);
  if (S.skip) return;
  const int nv = S.nq + S.selfnorm;
  const int so = S.selfnorm;
  double* as = sm;
  double* a2s = as + S.np;
  double* os = a2s + S.np2;
  double* acc = os + CH;
  double* red = acc + nv * 32;
  double* st = red + nv;
  for (int l = threadIdx.x; l < S.np; l += blockDim.x) as[l] = S.a[l];
  for (int l = threadIdx.x; l < S.np2; l += blockDim.x) a2s[l] = S.a2[l];
  for (int i = threadIdx.x; i < nv * 32; i += blockDim.x) acc[i] = 0.0;
  __syncthreads();
  const int n = P.n;
  const size_t ld = P.ld;
  const int nchunks = (n + CH - 1) / CH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int row = chunk * CH + threadIdx.x;
    const bool ok = row < n;
    double o = 0.0;
    if (ok) {
      o = S.in ? S.in[row] : 0.0;
      const double* pv = S.Pv + row;
#pragma unroll 8
      for (int l = 0; l < S.np; ++l) {
        const double v = pv[(size_t)l * ld];
        if (S.qstaged) st[l * CH + threadIdx.x] = v;
        o += as[l] * v;
      }
      const double* p2 = S.P2 + row;
#pragma unroll 4
      for (int l = 0; l < S.np2; ++l) o += a2s[l] * p2[(size_t)l * ld];
      S.out[row] = o;
    } else if (S.qstaged) {
      for (int l = 0; l < S.np; ++l) st[l * CH + threadIdx.x] = 0.0;
    }
    if (nv == 0) continue;
    os[threadIdx.x] = o;
    __syncthreads();
    for (int v = warp; v < nv; v += nw) {
      double a = 0.0;
      if (so && v == 0) {
#pragma unroll
        for (int q = 0; q < CH / 32; ++q) {
          const double t = os[lane + 32 * q];
          a += t * t;
        }
      } else if (S.qstaged) {
        const double* sl = st + (v - so) * CH;
#pragma unroll
        for (int q = 0; q < CH / 32; ++q) a += sl[lane + 32 * q] * os[lane + 32 * q];
      } else {
        const double* ql = S.Q + (size_t)(v - so) * ld + chunk * CH;
#pragma unroll
        for (int q = 0; q < CH / 32; ++q) {
          const int rr = lane + 32 * q;
          if (chunk * CH + rr < n) a += ql[rr] * os[rr];
        }
      }
      acc[v * 32 + lane] += a;
    }
    __syncthreads();
  }
  if (nv == 0) return;
  if (P.world > 1) {
    if (grid_reduce(acc, nv, P, red))
      for (int v = threadIdx.x; v < nv; v += blockDim.x) P.red_out[v] = red[v];
    return;
  }
  if (grid_reduce(acc, nv, P, red)) {
    if (threadIdx.x == 0) sweep_finish<MODE>(P, k, red);
  }
}

// Cross-GPU path: finisher after the allreduce of P.red_out.
template <int KIND>
__global__ void k_finish(Params P, int k) {
  // KIND: 0..7 sweep modes, 100 step spmv, 101 residual (k = initial), 102 push spmv
  if (threadIdx.x != 0) return;
  const double* red = P.red_out;
  if (KIND == 100) {
    if (P.g->active) fin_step_spmv(P, k, red);
  } else if (KIND == 101) {
    if (!(P.g->error != 0 || (!k && P.g->done))) fin_residual(P, red, k != 0);
  } else if (KIND == 102) {
    if (P.d->push_ok) fin_push_spmv(P, red);
  } else {
    const SweepSpec S = sweep_spec<KIND>(P, k);
    if (!S.skip) sweep_finish<KIND>(P, k, red);
  }
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

__global__ void __launch_bounds__(RITZ_THREADS) k_ritz(Params P) {
  extern __shared__ double sm[];
  GState* g = P.g;
  DState* d = P.d;
  if (g->error || !g->harvest) return;
  const int k = g->steps;
  const int tid = threadIdx.x;
  __shared__ double s_red[32];
  if (k == 0) {
    if (tid == 0) {
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
  auto load_h = [&]() {
    for (int e = tid; e < k * k; e += blockDim.x) {
      const int i = e % k, j = e / k;
      const int top = min(k - 1, j + 1);
      H[e] = (i <= top) ? P.h_orig[(size_t)j * (m + 1) + i] : 0.0;
    }
  };
  load_h();
  __syncthreads();
  double fr = 0.0;
  for (int e = tid; e < k * k; e += blockDim.x) fr += H[e] * H[e];
  const double scale = sqrt(block_sum(fr, s_red));
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  if (!(scale > 0.0) || !isfinite(scale)) {
    if (tid == 0) {
      d->skipped++;
      d->push_ok = 0;
      d->theta = nan;
    }
    return;
  }
  const double tol = d->inv_tol;
  // ---- largest_ritz_value: power iteration (deflation.cpp:57-82)
  {
    for (int i = tid; i < k; i += blockDim.x) z[i] = 1.0 / sqrt((double)k);
    __syncthreads();
    hmatvec(H, k, z, nx);
    __syncthreads();
    bool have = false, conv = false, broke = false;
    double val = 0.0;
    for (int it = 0; it < d->pow_maxit; ++it) {
      double p = 0.0;
      for (int i = tid; i < k; i += blockDim.x) p += nx[i] * nx[i];
      const double nz = sqrt(block_sum(p, s_red));
      if (!isfinite(nz) || nz == 0.0) {
        broke = true;
        break;
      }
      for (int i = tid; i < k; i += blockDim.x) z[i] = nx[i] / nz;
      __syncthreads();
      hmatvec(H, k, z, hz);
      __syncthreads();
      double q = 0.0;
      for (int i = tid; i < k; i += blockDim.x) q += z[i] * hz[i];
      const double theta = block_sum(q, s_red);
      double e = 0.0;
      for (int i = tid; i < k; i += blockDim.x) {
        const double t = hz[i] - theta * z[i];
        e += t * t;
      }
      const double resid = sqrt(block_sum(e, s_red));
      val = theta;
      have = true;
      if (resid <= tol * scale) {
        conv = true;
        break;
      }
      for (int i = tid; i < k; i += blockDim.x) nx[i] = hz[i];  // H z of the new z
      __syncthreads();
    }
    const bool ok = conv || (!broke && have);
    if (tid == 0 && ok && isfinite(val) && fabs(val) > fabs(d->mu)) d->mu = val;  // observe_ritz
  }
  __syncthreads();
  // ---- H^-1 by Gauss-Jordan with partial pivoting: [H | I] -> [I | H^-1]
  for (int e = tid; e < k * k; e += blockDim.x) B[e] = ((e % k) == (e / k)) ? 1.0 : 0.0;
  __syncthreads();
  for (int c = 0; c < k; ++c) {
    if (tid < 32) {
      double best = -1.0;
      int bi = c;
      for (int i = c + tid; i < k; i += 32) {
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
      if (tid == 0) s_piv = bi;
    }
    __syncthreads();
    const int p = s_piv;
    if (p != c) {
      for (int j = tid; j < 2 * k; j += blockDim.x) {
        double* M = j < k ? H : B;
        const int jj = j < k ? j : j - k;
        const double t = M[c + jj * k];
        M[c + jj * k] = M[p + jj * k];
        M[p + jj * k] = t;
      }
    }
    __syncthreads();
    const double piv = H[c + c * k];
    __syncthreads();
    for (int j = tid; j < 2 * k; j += blockDim.x) {
      double* M = j < k ? H : B;
      const int jj = j < k ? j : j - k;
      M[c + jj * k] /= piv;
    }
    for (int i = tid; i < k; i += blockDim.x) colc[i] = H[i + c * k];
    __syncthreads();
    for (int e = tid; e < 2 * k * k; e += blockDim.x) {
      const int i = e % k, j = e / k;
      if (i == c) continue;
      double* M = j < k ? H : B;
      const int jj = j < k ? j : j - k;
      M[i + jj * k] -= colc[i] * M[c + jj * k];
    }
    __syncthreads();
  }
  load_h();  // H again for theta / residuals
  __syncthreads();
  // ---- smallest_ritz_pair: inverse power iteration (deflation.cpp:31-54)
  for (int i = tid; i < k; i += blockDim.x) z[i] = 1.0 / sqrt((double)k);
  __syncthreads();
  bool conv = false;
  double val = 0.0;
  for (int it = 0; it < d->inv_maxit; ++it) {
    hmatvec(B, k, z, nx);
    __syncthreads();
    double p = 0.0;
    for (int i = tid; i < k; i += blockDim.x) p += nx[i] * nx[i];
    const double nz = sqrt(block_sum(p, s_red));
    if (!isfinite(nz) || nz == 0.0) break;
    for (int i = tid; i < k; i += blockDim.x) z[i] = nx[i] / nz;
    __syncthreads();
    hmatvec(H, k, z, hz);
    __syncthreads();
    double q = 0.0;
    for (int i = tid; i < k; i += blockDim.x) q += z[i] * hz[i];
    const double theta = block_sum(q, s_red);
    double e = 0.0;
    for (int i = tid; i < k; i += blockDim.x) {
      const double t = hz[i] - theta * z[i];
      e += t * t;
    }
    const double resid = sqrt(block_sum(e, s_red));
    val = theta;
    if (resid <= tol * scale) {
      conv = true;
      break;
    }
  }
  if (conv) {
    for (int l = tid; l < k; l += blockDim.x) P.zl[l] = z[l] * P.s[l];
    if (tid == 0) {
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
  __shared__ double q[MAX_R1 * MAX_R1];
  for (int e = threadIdx.x; e < r0 * r; e += blockDim.x) q[e] = P.Q[(e % r0) + (e / r0) * R1];
  __syncthreads();
  for (size_t row = blockIdx.x * (size_t)blockDim.x + threadIdx.x; row < (size_t)P.n;
       row += (size_t)gridDim.x * blockDim.x) {
#pragma unroll 1
    for (int which = 0; which < 2; ++which) {
      double* base = (which == 0 ? P.U : P.AU) + P.lo + row;
      double in[MAX_R1];
#pragma unroll
      for (int l = 0; l < MAX_R1; ++l)
        if (l < r0) in[l] = base[(size_t)l * P.ld];
      for (int j = 0; j < r; ++j) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < MAX_R1; ++l)
          if (l < r0) s += in[l] * q[l + j * r0];
        base[(size_t)j * P.ld] = s;
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
__global__ void k_csr_to_sell(Sell A, double* val, unsigned* col, const unsigned* rp,
                              const unsigned* ci, const double* v, unsigned col_shift,
                              int nslices, int write_cols) {
  const int lane = threadIdx.x & 31;
  const size_t s = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  if (s >= (size_t)nslices) return;
  const unsigned long long base = A.sptr[s];
  const int L = (int)((A.sptr[s + 1] - base) >> 5);
  const int len = (int)A.lane_len[s * 32 + lane];
  const unsigned short ro = A.lane_row[s * 32 + lane];
  const size_t tile = s / SPT;
  const size_t row = tile * TILE + ro;
  const size_t start = (ro != 0xFFFF) ? rp[row] : 0;
  for (int t = 0; t < L; ++t) {
    const size_t idx = base + (size_t)t * 32 + lane;
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

}  // namespace pgm
