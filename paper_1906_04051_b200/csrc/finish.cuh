// Scalar "finisher" logic run once per reduction by the last block of a
// kernel (or by k_finish after a cross-GPU allreduce).  Each function is the
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
  const int m = g->m;
  g->restart = restart;
  g->beta_cycle = beta;
  g->steps = 0;
  g->lucky = 0;
  g->active = 1;
  P.s[0] = 1.0 / beta;
  for (int i = 0; i <= m; ++i) P.gv[i] = 0.0;
  P.gv[0] = beta;
  const int r = P.d->r;
  for (int l = 0; l < r; ++l) P.tU[l] = Ur[l] * P.s[0];
  defl_coeffs(P, r, P.tU, P.c);
}

// After the explicit residual (gmres.cpp:142-147 + :149-157 / :191-212).
// red[0] = ||r||^2, red[1+l] = U_l . r
__device__ void fin_residual(const Params& P, const double* red, bool initial) {
  GState* g = P.g;
  const double beta = sqrt(red[0]);
  g->beta = beta;
  if (initial) {
    g->beta0 = beta;
    if (!isfinite(beta)) {
      set_error(P, 2 /*ENONFINITE*/, -1, -1);
      return;
    }
    if (beta == 0.0) {
      g->converged = 1;
      g->final_relative = 0.0;
      g->done = 1;
      return;
    }
    if (g->max_restarts == 0) {
      g->done = 1;
    } else {
      begin_cycle(P, 0, beta, red + 1);
      return;
    }
  } else {
    const int restart = g->restart;
    P.expl[restart] = beta;
    g->restarts = restart + 1;
    g->total_inner += (unsigned long long)g->steps;
    if (!isfinite(beta)) {
      set_error(P, 2, restart, -1);
      return;
    }
    if (g->lucky) {
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
      begin_cycle(P, restart + 1, beta, red + 1);
      return;
    }
  }
  // loop exit bookkeeping (gmres.cpp:213-216)
  g->final_relative = g->beta0 > 0.0 ? beta / g->beta0 : 0.0;
  if (!g->converged && !g->fixed) g->converged = beta <= g->rel_tol * g->beta0;
  g->active = 0;
}

// After sweep A (fused into the step SpMV): red[l] = W_l . w, l <= k.
__device__ __forceinline__ void fin_step_spmv(const Params& P, int k, const double* red) {
  for (int l = 0; l <= k; ++l) {
    const double h = P.s[l] * red[l];
    P.h1[l] = h;
    P.coefA[l] = -h * P.s[l];
  }
}

// After CGS2 pass 2 dots: red[l] = W_l . w1.  h = h1 + h2 (gmres.cpp:50-53).
__device__ __forceinline__ void fin_sweep_b(const Params& P, int k, const double* red) {
  const size_t col = (size_t)k * (P.m + 1);
  for (int l = 0; l <= k; ++l) {
    const double h2 = P.s[l] * red[l];
    P.coefB[l] = -h2 * P.s[l];
    const double h = P.h1[l] + h2;
    P.h_orig[col + l] = h;
    P.h_rot[col + l] = h;
  }
}

// Back-substitution (gmres.cpp:92-107) and the x-update coefficients
// x += M^{-1} V y = V y + U (|mu| T^{-1} U^T V y - U^T V y).
__device__ void end_cycle(const Params& P) {
  GState* g = P.g;
  g->active = 0;
  const int k = g->steps, m = g->m;
  double* y = P.xc;  // y first, scaled in place below
  for (int i = 0; i < k; ++i) y[i] = P.gv[i];
  for (int i = k - 1; i >= 0; --i) {
    const double d = P.h_rot[(size_t)i * (m + 1) + i];
    if (d == 0.0) {
      set_error(P, 3 /*ESINGULAR*/, g->restart, i);
      return;
    }
    double s = y[i];
    for (int j = i + 1; j < k; ++j) s -= P.h_rot[(size_t)j * (m + 1) + i] * y[j];
    y[i] = s / d;
  }
  const int r = P.d->r;
  if (r > 0) {
    double tz[MAX_R1 * 2];
    for (int l = 0; l < r; ++l) {
      double s = 0.0;
      for (int j = 0; j < k; ++j) s += y[j] * P.tU[(size_t)j * P.R1 + l];
      tz[l] = s;
    }
    defl_coeffs(P, r, tz, P.cx);
  }
  for (int j = 0; j < k; ++j) y[j] *= P.s[j];
}

// After CGS2 pass 2 update: red[0] = ||w2||^2, red[1+l] = U_l . w2.
// h_{k+1,k}, Givens update, records and the inner-loop exits
// (gmres.cpp:58-90, 163-180).
__device__ void fin_sweep_c(const Params& P, int k, const double* red) {
  GState* g = P.g;
  const int m = g->m;
  const double hnext = sqrt(red[0]);
  const size_t col = (size_t)k * (m + 1);
  P.h_orig[col + k + 1] = hnext;
  P.h_rot[col + k + 1] = hnext;
  if (!isfinite(hnext)) {
    set_error(P, 2, g->restart, k);
    return;
  }
  P.s[k + 1] = hnext > 0.0 ? 1.0 / hnext : 0.0;
  // apply_rotations_and_update(k)
  double* H = P.h_rot + col;
  for (int i = 0; i < k; ++i) {
    const double hi = H[i], hj = H[i + 1];
    H[i] = P.cs[i] * hi + P.sn[i] * hj;
    H[i + 1] = -P.sn[i] * hi + P.cs[i] * hj;
  }
  const double a = H[k], b = H[k + 1];
  const double rr = hypot(a, b);
  if (rr == 0.0) {
    P.cs[k] = 1.0;
    P.sn[k] = 0.0;
  } else {
    P.cs[k] = a / rr;
    P.sn[k] = b / rr;
  }
  H[k] = rr;
  H[k + 1] = 0.0;
  P.gv[k + 1] = -P.sn[k] * P.gv[k];
  P.gv[k] = P.cs[k] * P.gv[k];
  const double monitored = fabs(P.gv[k + 1]);
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
  if (stop) {
    end_cycle(P);
    return;
  }
  const int r = P.d->r;
  double* t = P.tU + (size_t)(k + 1) * P.R1;
  for (int l = 0; l < r; ++l) t[l] = red[1 + l] * P.s[k + 1];
  defl_coeffs(P, r, t, P.c);
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
