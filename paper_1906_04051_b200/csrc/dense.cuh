// Small dense fp64 linear algebra for the restart-time deflation work
// (T^{-1}, the truncation eigensolve).  Single-thread routines, compiled for
// both host (unit tests via tests/dense_harness.cpp) and device (run inside
// the last block of the push kernel, deflation.cpp:186-230 equivalents).
// Column-major storage: A(i, j) = a[i + j * ld].
#pragma once

#include <math.h>

#if defined(__CUDACC__)
#define PGM_HD __host__ __device__ __forceinline__
#else
#define PGM_HD inline
#endif

namespace pgm {
namespace dense {

// In-place LU with partial pivoting (row interchanges recorded in perm:
// row i of the factor is row perm[i] of the input).  Mirrors the unblocked
// Doolittle scheme of a PartialPivLU: a zero pivot column is skipped.
PGM_HD void lu_factor(double* a, int n, int ld, int* perm) {
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double big = fabs(a[k + k * ld]);
    for (int i = k + 1; i < n; ++i) {
      const double v = fabs(a[i + k * ld]);
      if (v > big) {
        big = v;
        piv = i;
      }
    }
    if (big != 0.0) {
      if (piv != k) {
        for (int j = 0; j < n; ++j) {
          const double t = a[k + j * ld];
          a[k + j * ld] = a[piv + j * ld];
          a[piv + j * ld] = t;
        }
        const int t = perm[k];
        perm[k] = perm[piv];
        perm[piv] = t;
      }
      const double d = a[k + k * ld];
      for (int i = k + 1; i < n; ++i) a[i + k * ld] /= d;
    }
    for (int j = k + 1; j < n; ++j) {
      const double ukj = a[k + j * ld];
      for (int i = k + 1; i < n; ++i) a[i + j * ld] -= a[i + k * ld] * ukj;
    }
  }
}

// x = A^{-1} b from lu_factor output; b and x may alias only if perm is identity,
// so x is always a separate array.
PGM_HD void lu_solve(const double* lu, int n, int ld, const int* perm, const double* b,
                     double* x) {
  for (int i = 0; i < n; ++i) x[i] = b[perm[i]];
  for (int i = 0; i < n; ++i) {
    double s = x[i];
    for (int j = 0; j < i; ++j) s -= lu[i + j * ld] * x[j];
    x[i] = s;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (int j = i + 1; j < n; ++j) s -= lu[i + j * ld] * x[j];
    x[i] = s / lu[i + i * ld];
  }
}

// inv (ld_inv) = A^{-1}; `a` is destroyed (holds the LU), work needs n doubles,
// perm n ints.
PGM_HD void invert(double* a, int n, int ld, double* inv, int ld_inv, int* perm, double* work) {
  lu_factor(a, n, ld, perm);
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < n; ++i) work[i] = (i == j) ? 1.0 : 0.0;
    lu_solve(a, n, ld, perm, work, inv + j * ld_inv);
  }
}

// Orthogonal reduction to upper Hessenberg form, A <- P^T A P with one
// Householder reflector per column (P = P_0 ... P_{n-3}); entries below the
// first subdiagonal are zeroed on return.
PGM_HD void hessenberg_reduce(double* a, int n, int ld) {
#define A_(i, j) a[(i) + (j) * ld]
  for (int c = 0; c + 2 < n; ++c) {
    // reflector v (stored over A(c+1:n, c)) with (I - 2 v v^T / v^T v) x = alpha e_1
    double sq = 0.0;
    for (int i = c + 1; i < n; ++i) sq += A_(i, c) * A_(i, c);
    const double xnorm = sqrt(sq);
    if (xnorm == 0.0) continue;
    const double x0 = A_(c + 1, c);
    const double alpha = x0 > 0.0 ? -xnorm : xnorm;
    A_(c + 1, c) = x0 - alpha;
    const double vtv = sq - x0 * x0 + A_(c + 1, c) * A_(c + 1, c);
    if (vtv == 0.0) {
      A_(c + 1, c) = x0;
      continue;
    }
    const double tau = 2.0 / vtv;
    // left: rows c+1..n-1 of columns c+1..n-1
    for (int j = c + 1; j < n; ++j) {
      double d = 0.0;
      for (int i = c + 1; i < n; ++i) d += A_(i, c) * A_(i, j);
      d *= tau;
      for (int i = c + 1; i < n; ++i) A_(i, j) -= d * A_(i, c);
    }
    // right: columns c+1..n-1 of every row
    for (int i = 0; i < n; ++i) {
      double d = 0.0;
      for (int j = c + 1; j < n; ++j) d += A_(i, j) * A_(j, c);
      d *= tau;
      for (int j = c + 1; j < n; ++j) A_(i, j) -= d * A_(j, c);
    }
    A_(c + 1, c) = alpha;
    for (int i = c + 2; i < n; ++i) A_(i, c) = 0.0;
  }
#undef A_
}

// Minimal complex arithmetic for the shifted QR below.
struct cplx {
  double re, im;
};
PGM_HD cplx c_make(double re, double im) { return cplx{re, im}; }
PGM_HD cplx c_add(cplx a, cplx b) { return cplx{a.re + b.re, a.im + b.im}; }
PGM_HD cplx c_sub(cplx a, cplx b) { return cplx{a.re - b.re, a.im - b.im}; }
PGM_HD cplx c_mul(cplx a, cplx b) {
  return cplx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
PGM_HD cplx c_conj(cplx a) { return cplx{a.re, -a.im}; }
PGM_HD cplx c_scale(cplx a, double s) { return cplx{a.re * s, a.im * s}; }
PGM_HD double c_abs(cplx a) { return hypot(a.re, a.im); }
PGM_HD cplx c_sqrt(cplx a) {  // principal branch
  const double r = c_abs(a);
  if (r == 0.0) return cplx{0.0, 0.0};
  const double t = sqrt(0.5 * (r + fabs(a.re)));
  if (a.re >= 0.0) return cplx{t, 0.5 * a.im / t};
  return cplx{0.5 * fabs(a.im) / t, a.im >= 0.0 ? t : -t};
}

// Eigenvalues of a real upper Hessenberg matrix `h` (not modified) by the
// explicitly shifted QR iteration in complex arithmetic: each sweep factors
// H - mu I = QR over the active window with complex Givens rotations
// G = [c s; -conj(s) c] (c real) and forms RQ + mu I; mu is the eigenvalue
// of the trailing 2x2 nearest its last diagonal entry (Wilkinson), with an
// ad-hoc shift every 10th sweep of a window.  A subdiagonal entry below
// eps * (|h_{i-1,i-1}| + |h_ii|) splits the window.  zwork: >= 2*n*n + n
// doubles.  Returns false if a window needs more than 90 sweeps.
PGM_HD bool hessenberg_eigvals(const double* h, int n, int ld, double* wr, double* wi,
                               double* zwork) {
  cplx* z = reinterpret_cast<cplx*>(zwork);  // n x n, column-major
  double* gc = zwork + 2 * n * n;            // n rotation cosines
#define Z_(i, j) z[(i) + (j) * n]
  double fro = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double v = (i <= j + 1) ? h[i + j * ld] : 0.0;
      Z_(i, j) = c_make(v, 0.0);
      fro += v * v;
    }
  fro = sqrt(fro);
  const double eps = 2.220446049250313e-16;
  int hi = n - 1, sweeps = 0;
  while (hi >= 0) {
    int lo = hi;
    while (lo > 0) {
      double s = c_abs(Z_(lo - 1, lo - 1)) + c_abs(Z_(lo, lo));
      if (s == 0.0) s = fro;
      if (c_abs(Z_(lo, lo - 1)) <= eps * s) {
        Z_(lo, lo - 1) = c_make(0.0, 0.0);
        break;
      }
      --lo;
    }
    if (lo == hi) {
      wr[hi] = Z_(hi, hi).re;
      wi[hi] = Z_(hi, hi).im;
      --hi;
      sweeps = 0;
      continue;
    }
    if (++sweeps > 90) return false;
    cplx mu;
    if (sweeps % 10 == 0) {
      const double t = c_abs(Z_(hi, hi - 1)) + (hi >= 2 ? c_abs(Z_(hi - 1, hi - 2)) : 0.0);
      mu = c_add(Z_(hi, hi), c_make(0.75 * t, 0.25 * t));
    } else {
      const cplx p = Z_(hi - 1, hi - 1), q = Z_(hi - 1, hi), r = Z_(hi, hi - 1), d = Z_(hi, hi);
      const cplx half = c_scale(c_sub(p, d), 0.5);
      const cplx disc = c_sqrt(c_add(c_mul(half, half), c_mul(q, r)));
      const cplx mid = c_scale(c_add(p, d), 0.5);
      const cplx m1 = c_add(mid, disc), m2 = c_sub(mid, disc);
      mu = c_abs(c_sub(m1, d)) <= c_abs(c_sub(m2, d)) ? m1 : m2;
    }
    for (int i = lo; i <= hi; ++i) Z_(i, i) = c_sub(Z_(i, i), mu);
    // QR: rotations k = lo..hi-1 zero Z(k+1, k); the sine of rotation k is
    // parked in Z(k+1, k), which it zeroes
    for (int k = lo; k < hi; ++k) {
      const cplx x = Z_(k, k), y = Z_(k + 1, k);
      const double ax = c_abs(x), ay = c_abs(y);
      const double rr = hypot(ax, ay);
      double c;
      cplx sn;
      if (rr == 0.0) {
        c = 1.0;
        sn = c_make(0.0, 0.0);
      } else if (ax == 0.0) {
        c = 0.0;
        sn = c_scale(c_conj(y), 1.0 / ay);
      } else {
        c = ax / rr;
        sn = c_scale(c_mul(c_scale(x, 1.0 / ax), c_conj(y)), 1.0 / rr);
      }
      for (int j = k; j <= hi; ++j) {
        const cplx a1 = Z_(k, j), a2 = Z_(k + 1, j);
        Z_(k, j) = c_add(c_scale(a1, c), c_mul(sn, a2));
        Z_(k + 1, j) = c_sub(c_scale(a2, c), c_mul(c_conj(sn), a1));
      }
      gc[k] = c;
      Z_(k + 1, k) = sn;
    }
    // RQ: apply G_k^H from the right, k = lo..hi-1
    for (int k = lo; k < hi; ++k) {
      const double c = gc[k];
      const cplx sn = Z_(k + 1, k);
      Z_(k + 1, k) = c_make(0.0, 0.0);
      for (int i = lo; i <= k + 1; ++i) {
        const cplx a1 = Z_(i, k), a2 = Z_(i, k + 1);
        Z_(i, k) = c_add(c_scale(a1, c), c_mul(a2, c_conj(sn)));
        Z_(i, k + 1) = c_sub(c_scale(a2, c), c_mul(a1, sn));
      }
    }
    for (int i = lo; i <= hi; ++i) Z_(i, i) = c_add(Z_(i, i), mu);
  }
  return true;
#undef Z_
}

// Unit-norm eigenvector of the eigenvalue of largest modulus (first one on
// ties, like a maxCoeff over |lambda|), by inverse iteration on (T - lambda I)
// — the quantity Deflator::truncate asks Eigen's EigenSolver for
// (deflation.cpp:189-203).  For a complex dominant pair the complex
// eigenvector is phase-normalised (largest-modulus component real) and its
// real part is returned, or its imaginary part when the real part vanishes.
// work: >= 4*n*n + 6*n doubles; iwork: >= n ints.  Returns 0 on success.
PGM_HD int dominant_eigvec(const double* T, int n, int ld, double* v, double* work, int* iwork) {
  double* h = work;             // n*n
  double* wr = h + n * n;       // n
  double* wi = wr + n;          // n
  double* m = wi + n;           // 2n*2n real embedding of the complex shift
  double* b = m + 4 * n * n;    // 2n
  double* xs = b + 2 * n;       // 2n
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) h[i + j * n] = T[i + j * ld];
  hessenberg_reduce(h, n, n);
  if (!hessenberg_eigvals(h, n, n, wr, wi, m)) return 1;
  // complex arithmetic leaves real eigenvalues with rounding-level imaginary
  // parts once a complex shift was used
  for (int i = 0; i < n; ++i)
    if (fabs(wi[i]) <= 1e-13 * hypot(wr[i], wi[i])) wi[i] = 0.0;
  int dom = 0;
  double best = -1.0;
  for (int i = 0; i < n; ++i) {
    const double mag = hypot(wr[i], wi[i]);
    if (mag > best) {
      best = mag;
      dom = i;
    }
  }
  const double lr = wr[dom], li = wi[dom];
  double tn = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) tn = fmax(tn, fabs(T[i + j * ld]));
  const double tiny = 1e-300 + 2.220446049250313e-16 * tn;
  if (li == 0.0) {
    // real inverse iteration
    for (int i = 0; i < n; ++i) b[i] = 1.0 / sqrt((double)n) * (1.0 + 0.01 * i);
    for (int it = 0; it < 3; ++it) {
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) m[i + j * n] = T[i + j * ld] - (i == j ? lr : 0.0);
      lu_factor(m, n, n, iwork);
      for (int i = 0; i < n; ++i)
        if (m[i + i * n] == 0.0) m[i + i * n] = tiny;
      lu_solve(m, n, n, iwork, b, xs);
      double nrm = 0.0;
      for (int i = 0; i < n; ++i) nrm += xs[i] * xs[i];
      nrm = sqrt(nrm);
      if (!(nrm > 0.0) || !isfinite(nrm)) return 2;
      for (int i = 0; i < n; ++i) b[i] = xs[i] / nrm;
    }
    for (int i = 0; i < n; ++i) v[i] = b[i];
    return 0;
  }
  // complex: (T - (lr + i li) I)(x + i y) = (c + i d) as a 2n x 2n real system
  const int n2 = 2 * n;
  for (int i = 0; i < n2; ++i) b[i] = (i < n) ? 1.0 / sqrt((double)n) * (1.0 + 0.01 * i) : 0.0;
  for (int it = 0; it < 3; ++it) {
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const double t = T[i + j * ld] - (i == j ? lr : 0.0);
        const double s = (i == j) ? li : 0.0;
        m[i + j * n2] = t;             // [ T-lr   li ]
        m[i + (j + n) * n2] = s;       // [ -li  T-lr ]
        m[(i + n) + j * n2] = -s;
        m[(i + n) + (j + n) * n2] = t;
      }
    lu_factor(m, n2, n2, iwork);
    for (int i = 0; i < n2; ++i)
      if (m[i + i * n2] == 0.0) m[i + i * n2] = tiny;
    lu_solve(m, n2, n2, iwork, b, xs);
    double nrm = 0.0;
    for (int i = 0; i < n2; ++i) nrm += xs[i] * xs[i];
    nrm = sqrt(nrm);
    if (!(nrm > 0.0) || !isfinite(nrm)) return 2;
    for (int i = 0; i < n2; ++i) b[i] = xs[i] / nrm;
  }
  // phase-normalise: largest-modulus component made real positive
  int big = 0;
  double bm = -1.0;
  for (int i = 0; i < n; ++i) {
    const double mg = hypot(b[i], b[i + n]);
    if (mg > bm) {
      bm = mg;
      big = i;
    }
  }
  const double cr = b[big] / bm, ci = -b[big + n] / bm;  // multiply by conj phase
  double rn = 0.0;
  for (int i = 0; i < n; ++i) {
    v[i] = b[i] * cr - b[i + n] * ci;
    rn += v[i] * v[i];
  }
  if (sqrt(rn) <= 1e-12)
    for (int i = 0; i < n; ++i) v[i] = b[i] * ci + b[i + n] * cr;
  return 0;
}

}  // namespace dense
}  // namespace pgm
