// Scalar "finisher" logic run once per reduction by the last block of a
// kernel (or by k_finish after a cross-GPU allreduce).  Every fin_* function is
// block-collective: all threads of that block call it; loops over independent
// entries run across the threads, the inherently serial parts (Givens chain,
// control decisions) run on thread 0 from shared-memory copies.  Each function is the
// restatement of the reference's host-side scalar work at that point of the
// restart cycle; citations into /root/reference/proj.
#pragma once

#include <math.h>

#include "common.cuh"
#include "dense.cuh"

namespace pgm {

// coeff = |mu| T^{-1} t - t  (Deflator::apply, deflation.cpp:110-115)
__device__ __forceinline__ void defl_coeffs(const Params& P, int r, const double* t,
                                            double* c) {
  const double amu = fabs(P.d->mu);
  for (int i = 0; i < r; ++i) {
    double s = 0.0;
    for (int j = 0; j < r; ++j) s += P.Tinv[i + j * P.R1] * t[j];
    c[i] = amu * s - t[i];
  }
}

// Block-collective version (t must be visible to every thread of the block).
__device__ __forceinline__ void defl_coeffs_par(const Params& P, int r,
                                                const double* __restrict__ t,
                                                double* __restrict__ c) {
  const double amu = fabs(P.d->mu);
  const double* __restrict__ ti = P.Tinv;
  const int R1 = P.R1;
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    double s = 0.0;
    // independent loads batched (the finisher is on the step's critical path)
#pragma unroll 8
    for (int j = 0; j < r; ++j) s += ti[i + j * R1] * t[j];
    c[i] = amu * s - t[i];
  }
}

__device__ __forceinline__ void set_error(const Params& P, int code, int restart, int step) {
  GState* g = P.g;
  if (!g->error) {
    g->error = code;
    g->err_restart = restart;
    g->err_step = step;
  }
  g->active = 0;
  g->done = 1;
}

// Begin cycle `restart` from the explicit residual r = W_0 (unnormalised):
// GmresWorkspace::begin_cycle (gmres.cpp:21-26) with the scale folded lazily,
// plus U^T v_0 for the first deflation apply.
__device__ __forceinline__ void begin_cycle(const Params& P, int restart, double beta,
                                            const double* Ur) {
  GState* g = P.g;
  const int m = P.m;
  const double sc = 1.0 / beta;
  if (threadIdx.x == 0) {
    g->restart = restart;
    g->beta_cycle = beta;
    g->steps = 0;
    g->lucky = 0;
    g->active = 1;
    P.s[0] = sc;
  }
  for (int i = threadIdx.x; i <= m; i += blockDim.x) P.gv[i] = i == 0 ? beta : 0.0;
  const int r = P.d->r;
  for (int l = threadIdx.x; l < r; l += blockDim.x) P.tU[l] = Ur[l] * sc;
  __syncthreads();
  defl_coeffs_par(P, r, P.tU, P.c);
}

// After the explicit residual (gmres.cpp:142-147 + :149-157 / :191-212).
// red[0] = ||r||^2, red[1+l] = U_l . r
__device__ void fin_residual(const Params& P, const double* red, bool initial) {
  __shared__ int s_begin, s_restart;
  __shared__ double s_beta;
  if (threadIdx.x == 0) {
    s_begin = 0;
    GState* g = P.g;
    const double beta = sqrt(red[0]);
    s_beta = beta;
    g->beta = beta;
    bool exit_loop = false;
    if (initial) {
      g->beta0 = beta;
      if (!isfinite(beta)) {
        set_error(P, 2 /*ENONFINITE*/, -1, -1);
      } else if (beta == 0.0) {
        g->converged = 1;
        g->final_relative = 0.0;
        g->done = 1;
      } else if (g->max_restarts == 0) {
        g->done = 1;
        exit_loop = true;
      } else {
        s_begin = 1;
        s_restart = 0;
      }
    } else {
      const int restart = g->restart;
      P.expl[restart] = beta;
      g->restarts = restart + 1;
      g->total_inner += (unsigned long long)g->steps;
      exit_loop = true;
      if (!isfinite(beta)) {
        set_error(P, 2, restart, -1);
        exit_loop = false;
      } else if (g->lucky) {
        g->breakdown = 1;
        g->converged = 1;
        g->done = 1;
      } else if (!g->fixed && beta <= g->rel_tol * g->beta0) {
        g->converged = 1;
        g->done = 1;
      } else if (beta == 0.0) {
        g->converged = 1;
        g->done = 1;
      } else if (restart + 1 >= g->max_restarts) {
        g->done = 1;
      } else {
        s_begin = 1;
        s_restart = restart + 1;
        exit_loop = false;
      }
    }
    if (exit_loop) {
      // loop exit bookkeeping (gmres.cpp:213-216)
      g->final_relative = g->beta0 > 0.0 ? beta / g->beta0 : 0.0;
      if (!g->converged && !g->fixed) g->converged = beta <= g->rel_tol * g->beta0;
      g->active = 0;
    }
  }
  __syncthreads();
  if (s_begin) begin_cycle(P, s_restart, s_beta, red + 1);
}

// After sweep A (fused into the step SpMV): red[l] = W_l . w, l <= k.
__device__ __forceinline__ void fin_step_spmv(const Params& P, int k, const double* red) {
  for (int l = threadIdx.x; l <= k; l += blockDim.x) {
    const double h = P.s[l] * red[l];
    P.h1[l] = h;
    P.coefA[l] = -h * P.s[l];
  }
}

// After CGS2 pass 2 (update w1 and its dots), gmres.cpp:50-65 + 67-90:
//   red[l] = W_l . w1 (l <= k), red[k+1] = ||w1||^2, red[k+2+j] = U_j . w1.
// h = h1 + h2; pass C (w2 = w1 - V h2, k_cgs2_update) needs no reduction:
//   ||w2||^2 = ||w1||^2 - ||h2||^2                 (V orthonormal)
//   U^T W_{k+1} = U^T w1 - sum_l h2_l U^T v_l      (U^T v_l kept in tU)
// then h_{k+1,k}, the Givens update, the records and the inner-loop exits
// (gmres.cpp:163-180), and the deflation coefficients of the next apply.
__device__ void fin_sweep_b(const Params& P, int k, const double* red) {
  __shared__ double sH[MAX_M + 2], sC[MAX_M], sS[MAX_M], sh2[MAX_M + 1];
  __shared__ int s_go;
  GState* g = P.g;
  const int m = P.m;
  const size_t col = (size_t)k * (m + 1);
  for (int l = threadIdx.x; l <= k; l += blockDim.x) {
    const double sl = P.s[l];
    const double h2 = sl * red[l];
    sh2[l] = h2;
    P.coefB[l] = -h2 * sl;
    const double h = P.h1[l] + h2;
    P.h_orig[col + l] = h;
    sH[l] = h;
    if (l < k) {
      sC[l] = P.cs[l];
      sS[l] = P.sn[l];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s_go = 0;
    double nh2 = 0.0;
    for (int l = 0; l <= k; ++l) nh2 += sh2[l] * sh2[l];
    const double hnext = sqrt(fmax(red[k + 1] - nh2, 0.0));
    sH[k + 1] = hnext;
    P.h_orig[col + k + 1] = hnext;
    if (!isfinite(hnext) || !isfinite(red[k + 1])) {
      set_error(P, 2, g->restart, k);
    } else {
      P.s[k + 1] = hnext > 0.0 ? 1.0 / hnext : 0.0;
      // apply_rotations_and_update(k)
      for (int i = 0; i < k; ++i) {
        const double hi = sH[i], hj = sH[i + 1];
        sH[i] = sC[i] * hi + sS[i] * hj;
        sH[i + 1] = -sS[i] * hi + sC[i] * hj;
      }
      const double a = sH[k], b = sH[k + 1];
      const double rr = hypot(a, b);
      double ck, sk;
      if (rr == 0.0) {
        ck = 1.0;
        sk = 0.0;
      } else {
        ck = a / rr;
        sk = b / rr;
      }
      P.cs[k] = ck;
      P.sn[k] = sk;
      sH[k] = rr;
      sH[k + 1] = 0.0;
      const double gk = P.gv[k];
      P.gv[k + 1] = -sk * gk;
      P.gv[k] = ck * gk;
      const double monitored = fabs(-sk * gk);
      const int idx = g->n_inner++;
      P.rec_restart[idx] = (uint32_t)g->restart;
      P.rec_step[idx] = (uint32_t)k;
      P.rec_mon[idx] = monitored;
      g->steps = k + 1;
      bool stop = false;
      if (hnext < g->breakdown_scale * g->beta_cycle) {
        g->lucky = 1;
        stop = true;
      } else if (!g->fixed && monitored <= g->rel_tol * g->beta0) {
        stop = true;
      }
      if (k + 1 >= m) stop = true;
      if (stop) g->active = 0;  // back-substitution: k_end_cycle
      s_go = !stop;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= k + 1; i += blockDim.x) P.h_rot[col + i] = sH[i];
  if (s_go) {
    const int r = P.d->r, R1 = P.R1;
    double* t = P.tU + (size_t)(k + 1) * R1;
    const double sk1 = P.s[k + 1];
    for (int j = threadIdx.x; j < r; j += blockDim.x) {
      double uw = red[k + 2 + j];
      for (int l = 0; l <= k; ++l) uw -= sh2[l] * P.tU[(size_t)l * R1 + j];
      t[j] = uw * sk1;
    }
    __syncthreads();
    defl_coeffs_par(P, r, t, P.c);
  }
}


// ---- DCGS2 (delayed CGS2, one reduction per Arnoldi step) ---------------------
// Step k runs the operator on the lagged vector u_k = W_k (orthogonalised once
// against v_0..v_{k-1}); the SpMV epilogue's ONE reduction delivers
//   red = [W_l . y (nb), W_l . u (k), u.u, u.y, U_j . y (r)],  nb = max(k, 1).
// The finisher completes column k-1 of H (second-pass coefficients a, the
// subdiagonal beta = |u - Q a|), applies its Givens rotation and the exits,
// then forms the first pass of column k through A M^-1 Q = Q H and the
// coefficients of the single update pass (k_dcgs2_update).  Restatement:
// oracle/pgmres_oracle.py::_dcgs2_cycle (reference parity measured there).
// Coefficient slots: coefA[l] = -a_l s_l (l < k), coefA[k] = 1/beta;
// coefB[l] = -(Ha_l/beta + h1_l) s_l (l < k), coefB[k] = -(Ha_k/beta + h1_k) s_k.
// tU[k] holds U^T u_k (raw) until the step finalises it.

// Column k-1 completion, called by EVERY thread of the finishing block (sa = a
// in smem).  The global reads (column k-1 of H, the previous rotations) are
// issued block-parallel into smem first; thread 0 then runs the short serial
// part (Givens chain, records, exits) on smem only — the finisher sits on
// the critical path between two kernels, so its latency chain matters.
// Returns 1 (in every thread) to continue.
__device__ int dcgs2_column(const Params& P, int k, const double* sa, double alpha, bool close,
                            double* sH, double* s_beta) {
  __shared__ double sC[MAX_M], sS[MAX_M], s_na2;
  __shared__ int s_ret;
  GState* g = P.g;
  const int m = P.m;
  const size_t col = (size_t)(k - 1) * (m + 1);
  const int kk = k - 1;  // the column being completed
  // thread 0's scalars, loaded up front (they land during the parallel phase)
  double bscale = 0.0, bcyc = 0.0, gk = 0.0, rtol = 0.0, b0 = 0.0;
  int fixed = 0, restart = 0, ninner = 0;
  if (threadIdx.x == 0) {
    bscale = g->breakdown_scale;
    bcyc = g->beta_cycle;
    gk = P.gv[kk];
    rtol = g->rel_tol;
    b0 = g->beta0;
    fixed = g->fixed;
    restart = g->restart;
    ninner = g->n_inner;
  }
  for (int l = threadIdx.x; l < k; l += blockDim.x) {
    const double h = P.h_orig[col + l] + sa[l];
    P.h_orig[col + l] = h;
    sH[l] = h;
    if (l < kk) {
      sC[l] = P.cs[l];
      sS[l] = P.sn[l];
    }
  }
  if (threadIdx.x < 32) {
    double v = 0.0;
    for (int l = threadIdx.x; l < k; l += 32) v += sa[l] * sa[l];
    v = warp_sum(v);
    if (threadIdx.x == 0) s_na2 = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s_ret = 0;
    const double na2 = s_na2;
    // Pythagorean remainder ||u_k - Q a||^2 = alpha - ||a||^2.  When it sits at
    // rounding level of alpha the value carries no digits (it can even clamp
    // to 0).  If the bound sqrt(floor) is itself below the breakdown
    // threshold the Krylov space is exhausted (gmres.cpp:173 fires for any
    // true value); otherwise the step is ambiguous: the cycle closes here (not
    // a lucky breakdown) and later cycles run the CGS2 step, whose remainder
    // norm is formed explicitly (pass B) — no false breakdown at the rounding
    // floor.
    const double diff = alpha - na2;
    const double floor2 = 4.0 * (k + 1) * 2.220446049250313e-16 * alpha;
    bool ambiguous = false;
    double beta = sqrt(fmax(diff, 0.0));
    if (diff <= floor2 && alpha > 0.0 && sqrt(floor2) >= bscale * bcyc) {
      ambiguous = true;
      beta = sqrt(floor2);
    }
    *s_beta = beta;
    sH[k] = beta;
    P.h_orig[col + k] = beta;
    if (!isfinite(beta) || !isfinite(alpha)) {
      set_error(P, 2, restart, k - 1);
    } else {
      for (int i = 0; i < kk; ++i) {
        const double hi = sH[i], hj = sH[i + 1];
        sH[i] = sC[i] * hi + sS[i] * hj;
        sH[i + 1] = -sS[i] * hi + sC[i] * hj;
      }
      const double a = sH[kk], b = sH[kk + 1];
      const double rr = hypot(a, b);
      double ck, sk;
      if (rr == 0.0) {
        ck = 1.0;
        sk = 0.0;
      } else {
        ck = a / rr;
        sk = b / rr;
      }
      P.cs[kk] = ck;
      P.sn[kk] = sk;
      sH[kk] = rr;
      sH[kk + 1] = 0.0;
      P.gv[kk + 1] = -sk * gk;
      P.gv[kk] = ck * gk;
      const double monitored = fabs(-sk * gk);
      const int idx = ninner;
      g->n_inner = ninner + 1;
      P.rec_restart[idx] = (uint32_t)restart;
      P.rec_step[idx] = (uint32_t)kk;
      P.rec_mon[idx] = monitored;
      g->steps = kk + 1;
      bool stop = close || kk + 1 >= m;
      if (ambiguous) {
        g->dc_fallback = 1;
        stop = true;
      } else if (beta < bscale * bcyc) {
        g->lucky = 1;
        stop = true;
      } else if (!fixed && monitored <= rtol * b0) {
        stop = true;
      }
      if (stop) {
        g->active = 0;
      } else {
        // beta == 0 without the breakdown exit (breakdown_scale = 0 or
        // beta_cycle = 0, fixed iterations): continue with finite
        // coefficients, as the reference's arnoldi_step does for hnext == 0
        // (gmres.cpp:60-63)
        P.s[k] = beta > 0.0 ? 1.0 / beta : 0.0;
        s_ret = 1;
      }
    }
  }
  __syncthreads();
  // the rotated column (h_rot, gmres.cpp:67-90), written block-parallel
  if (isfinite(*s_beta))
    for (int i = threadIdx.x; i <= kk + 1; i += blockDim.x) P.h_rot[col + i] = sH[i];
  return s_ret;
}

__device__ void fin_dcgs2(const Params& P, int k, const double* red) {
  __shared__ double sa[MAX_M + 1], sb[MAX_M + 1], sHa[MAX_M + 2], sh1[MAX_M + 2];
  __shared__ double sH[MAX_M + 2];
  __shared__ double s_beta, s_qw;
  __shared__ int s_go;
  const int m = P.m, R1 = P.R1, r = P.d->r;
  const int nb = k > 0 ? k : 1;
  const double alpha = red[nb + k], gamma = red[nb + k + 1];
  const double* Uy = red + nb + k + 2;
  for (int l = threadIdx.x; l < nb; l += blockDim.x) {
    const double sl = P.s[l];
    sb[l] = sl * red[l];
    if (l < k) sa[l] = sl * red[nb + l];
  }
  __syncthreads();
  if (k == 0) {
    if (threadIdx.x == 0) {
      s_go = 1;
      s_beta = 1.0;
    }
  } else {
    const int go = dcgs2_column(P, k, sa, alpha, false, sH, (double*)&s_beta);
    if (threadIdx.x == 0) s_go = go;
  }
  __syncthreads();
  if (!s_go) return;
  const double beta = s_beta;
  const double ib = beta > 0.0 ? 1.0 / beta : 0.0;
  if (k == 0) {
    // q_0 is final: column 0's first pass h1_0 = v_0 . y; u_1 = y - h1_0 v_0
    if (threadIdx.x == 0) {
      const double h1 = sb[0];
      P.h_orig[0] = h1;
      P.coefA[0] = 1.0;                 // 1/beta (y is not rescaled)
      P.coefB[0] = -h1 * P.s[0];
      P.s[1] = 1.0;
      sh1[0] = h1;
    }
    __syncthreads();
    double* tn = P.tU + (size_t)1 * R1;
    for (int j = threadIdx.x; j < r; j += blockDim.x) tn[j] = Uy[j] - sh1[0] * P.tU[j];
    __syncthreads();
    defl_coeffs_par(P, r, tn, P.c);
    return;
  }
  // H[:k+1, :k] a (Hessenberg: row l has columns >= l-1)
  for (int l = threadIdx.x; l <= k; l += blockDim.x) {
    // independent loads batched 8 deep (no stores in the loop)
    const double* __restrict__ hrow = P.h_orig + l;
    double s = 0.0;
#pragma unroll 8
    for (int j = (l > 0 ? l - 1 : 0); j < k; ++j) s += __ldcg(hrow + (size_t)j * (m + 1)) * sa[j];
    sHa[l] = s;
  }
  if (threadIdx.x == 0) {
    double ab = 0.0;
    for (int l = 0; l < k; ++l) ab += sa[l] * sb[l];
    s_qw = (gamma - ab) * ib;  // q_k . y
  }
  __syncthreads();
  const double sk = P.s[k];
  const size_t colk = (size_t)k * (m + 1);
  for (int l = threadIdx.x; l <= k; l += blockDim.x) {
    const double h1 = l < k ? (sb[l] - sHa[l]) * ib : (s_qw - sHa[k]) * ib;
    sh1[l] = h1;
    P.h_orig[colk + l] = h1;  // first pass of column k (second pass added at step k+1)
    if (l < k) {
      const double sl = P.s[l];
      P.coefA[l] = -sa[l] * sl;
      P.coefB[l] = -(sHa[l] * ib + h1) * sl;
    } else {
      P.coefA[k] = ib;
      P.coefB[k] = -(sHa[k] * ib + h1) * sk;
    }
  }
  __syncthreads();
  // U^T v_k = s_k (U^T u_k - sum_l a_l U^T v_l); U^T u_{k+1} (raw) for the next apply
  double* tk = P.tU + (size_t)k * R1;
  double* tn = P.tU + (size_t)(k + 1) * R1;
  for (int j = threadIdx.x; j < r; j += blockDim.x) {
    // one pass over U^T v_l (global, loads batched 8 deep) for both sums
    const double* __restrict__ tcol = P.tU + j;
    double t = tk[j], u = Uy[j] * ib;
#pragma unroll 8
    for (int l = 0; l < k; ++l) {
      const double tl = __ldcg(tcol + (size_t)l * R1);
      t -= sa[l] * tl;
      u -= (sHa[l] * ib + sh1[l]) * tl;
    }
    const double tq = sk * t;
    tk[j] = tq;
    u -= (sHa[k] * ib + sh1[k]) * tq;
    tn[j] = u;
  }
  if (threadIdx.x == 0) P.s[k + 1] = 1.0;
  __syncthreads();
  defl_coeffs_par(P, r, tn, P.c);
}

// Cycle end without an early exit: red = [W_l . u_m (m), u_m . u_m] completes column m-1.
__device__ void fin_dcgs2_close(const Params& P, const double* red) {
  __shared__ double sa[MAX_M + 1], sH[MAX_M + 2];
  __shared__ double s_beta;
  const int m = P.m;
  for (int l = threadIdx.x; l < m; l += blockDim.x) sa[l] = P.s[l] * red[l];
  __syncthreads();
  dcgs2_column(P, m, sa, red[m], true, sH, (double*)&s_beta);
}

// ---- restart harvest: push_vector (deflation.cpp:123-184) ----------------------

// red[0] = ||u||^2, red[1+l] = U_l . u
__device__ __forceinline__ void fin_push1(const Params& P, const double* red) {
  DState* d = P.d;
  const double norm_in = sqrt(red[0]);
  d->norm_in = norm_in;
  if (!(norm_in > 0.0) || !isfinite(norm_in)) {
    d->skipped++;
    d->push_ok = 0;
    return;
  }
  const int r = d->r;
  for (int l = 0; l < r; ++l) P.proj[l] = -red[1 + l];
  if (r == 0) {  // no Gram-Schmidt passes: norm_left == norm_in
    d->pscale = 1.0 / norm_in;
  }
}

// second Gram-Schmidt pass projections: red[l] = U_l . u
__device__ __forceinline__ void fin_push2(const Params& P, const double* red) {
  for (int l = 0; l < P.d->r; ++l) P.proj[l] = -red[l];
}

// red[0] = ||u||^2 after both passes: acceptance test (deflation.cpp:174-179)
__device__ __forceinline__ void fin_push3(const Params& P, const double* red) {
  DState* d = P.d;
  const double norm_left = sqrt(red[0]);
  if (!(norm_left >= d->accept_tol * d->norm_in)) {
    d->skipped++;
    d->push_ok = 0;
    return;
  }
  d->pscale = 1.0 / norm_left;
}

// One Deflator::truncate() call (deflation.cpp:186-225): drop up to `drop`
// dominant-|lambda| directions of T, accumulating the rotation into Q
// (r0 x r, ld R1; Q must hold the identity on the first call).  Returns the
// new rank.
__device__ int truncate_drop(const Params& P, int r0, int r) {
  DState* d = P.d;
  const int R1 = P.R1;
  double* Q = P.Q;
  double* w = P.dwork;                       // eigen workspace
  double* v = w + 4 * R1 * R1 + 8 * R1;      // R1
  double* hv = v + R1;                       // R1
  double* pm = hv + R1;                      // R1 x R1 reflector
  double* tmp = pm + R1 * R1;                // R1 x R1
  double* qn = tmp + R1 * R1;                // R1 x R1
  for (int dropped = 0; dropped < d->drop && r > 1; ++dropped) {
    if (dense::dominant_eigvec(P.T, r, R1, v, w, P.iwork) != 0) {
      d->trunc_fail = 1;
      return r;
    }
    double vn = 0.0;
    for (int i = 0; i < r; ++i) vn += v[i] * v[i];
    vn = sqrt(vn);
    if (!(vn > 0.0) || !isfinite(vn)) {
      d->trunc_fail = 1;
      return r;
    }
    for (int i = 0; i < r; ++i) v[i] /= vn;
    // Householder reflection mapping v onto the last axis (deflation.cpp:206-214)
    for (int i = 0; i < r; ++i) hv[i] = v[i];
    const double sigma = v[r - 1] >= 0.0 ? 1.0 : -1.0;
    hv[r - 1] += sigma;
    double denom = 0.0;
    for (int i = 0; i < r; ++i) denom += hv[i] * hv[i];
    for (int j = 0; j < r; ++j)
      for (int i = 0; i < r; ++i) {
        double p = (i == j) ? 1.0 : 0.0;
        if (denom > 0.0) p -= (2.0 / denom) * (hv[i] * hv[j]);
        pm[i + j * R1] = p;
      }
    // T <- q^T T q with q = pm[:, :r-1]
    for (int j = 0; j < r - 1; ++j)  // tmp = q^T T  ((r-1) x r)
      for (int i = 0; i < r; ++i) {
        double s = 0.0;
        for (int l = 0; l < r; ++l) s += pm[l + j * R1] * P.T[l + i * R1];
        tmp[j + i * R1] = s;
      }
    for (int j = 0; j < r - 1; ++j)
      for (int i = 0; i < r - 1; ++i) {
        double s = 0.0;
        for (int l = 0; l < r; ++l) s += tmp[i + l * R1] * pm[l + j * R1];
        P.T[i + j * R1] = s;
      }
    // Q <- Q q  (r0 x (r-1))
    for (int j = 0; j < r - 1; ++j)
      for (int i = 0; i < r0; ++i) {
        double s = 0.0;
        for (int l = 0; l < r; ++l) s += Q[i + l * R1] * pm[l + j * R1];
        qn[i + j * R1] = s;
      }
    for (int j = 0; j < r - 1; ++j)
      for (int i = 0; i < r0; ++i) Q[i + j * R1] = qn[i + j * R1];
    r = r - 1;
  }
  return r;
}

__device__ __forceinline__ void q_identity(const Params& P, int r0) {
  for (int j = 0; j < r0; ++j)
    for (int i = 0; i < r0; ++i) P.Q[i + j * P.R1] = (i == j) ? 1.0 : 0.0;
}

// push_vector's overflow loop (deflation.cpp:177-181).
__device__ void truncate_all(const Params& P) {
  DState* d = P.d;
  const int r0 = d->r;
  q_identity(P, r0);
  d->trunc_fail = 0;
  int r = r0;
  while (r > d->r_max) {
    const int before = r;
    r = truncate_drop(P, r0, r);
    if (r == before || d->trunc_fail) break;
  }
  d->r0 = r0;
  d->rotate = (r != r0);
  d->r = r;
}

// T^{-1} of the active block (refresh_lu, deflation.cpp:227-230).
__device__ void refresh_tinv(const Params& P) {
  const int r = P.d->r, R1 = P.R1;
  if (r == 0) return;
  double* a = P.dwork;  // R1 x R1 copy
  for (int j = 0; j < r; ++j)
    for (int i = 0; i < r; ++i) a[i + j * R1] = P.T[i + j * R1];
  dense::invert(a, r, R1, P.Tinv, R1, P.iwork, a + R1 * R1);
}

// After A u: red[l] = U_l . AU_j (l <= j), red[j+1+l] = U_j . AU_l (l < j).
__device__ void fin_push_spmv(const Params& P, const double* red) {
  DState* d = P.d;
  const int j = d->r, R1 = P.R1;
  for (int l = 0; l < j; ++l) {
    P.T[l + j * R1] = red[l];
    P.T[j + l * R1] = red[j + 1 + l];
  }
  P.T[j + j * R1] = red[j];
  d->r = j + 1;
  d->rotate = 0;
  if (d->r > d->r_max) truncate_all(P);
  refresh_tinv(P);
}

}  // namespace pgm
