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

PGM_HD double sgn_of(double a, double b) { return b >= 0.0 ? fabs(a) : -fabs(a); }

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

// Reduce a general matrix to upper Hessenberg form by stabilised elementary
// similarity transformations (Gaussian elimination with pivoting); entries
// below the first subdiagonal are zeroed on return.
PGM_HD void hessenberg(double* a, int n, int ld) {
#define A_(i, j) a[(i) + (j) * ld]
  for (int m = 1; m < n - 1; ++m) {
    double x = 0.0;
    int piv = m;
    for (int j = m; j < n; ++j)
      if (fabs(A_(j, m - 1)) > fabs(x)) {
        x = A_(j, m - 1);
        piv = j;
      }
    if (piv != m) {
      for (int j = m - 1; j < n; ++j) {
        const double t = A_(piv, j);
        A_(piv, j) = A_(m, j);
        A_(m, j) = t;
      }
      for (int j = 0; j < n; ++j) {
        const double t = A_(j, piv);
        A_(j, piv) = A_(j, m);
        A_(j, m) = t;
      }
    }
    if (x != 0.0) {
      for (int i = m + 1; i < n; ++i) {
        double y = A_(i, m - 1);
        if (y != 0.0) {
          y /= x;
          A_(i, m - 1) = y;
          for (int j = m; j < n; ++j) A_(i, j) -= y * A_(m, j);
          for (int j = 0; j < n; ++j) A_(j, m) += y * A_(j, i);
        }
      }
    }
  }
  for (int j = 0; j < n; ++j)
    for (int i = j + 2; i < n; ++i) A_(i, j) = 0.0;
#undef A_
}

// Eigenvalues of an upper Hessenberg matrix by the Francis double-shift QR
// iteration (destroys a).  Returns false if an eigenvalue fails to converge
// in 30 iterations.
PGM_HD bool hqr(double* a, int n, int ld, double* wr, double* wi) {
#define A_(i, j) a[(i) + (j) * ld]
  double anorm = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = (i > 0 ? i - 1 : 0); j < n; ++j) anorm += fabs(A_(i, j));
  int nn = n - 1;
  double t = 0.0;
  double p = 0.0, q = 0.0, r = 0.0, s, w, x, y, z = 0.0;
  while (nn >= 0) {
    int its = 0, l;
    do {
      for (l = nn; l >= 1; --l) {
        s = fabs(A_(l - 1, l - 1)) + fabs(A_(l, l));
        if (s == 0.0) s = anorm;
        if (fabs(A_(l, l - 1)) + s == s) {
          A_(l, l - 1) = 0.0;
          break;
        }
      }
      x = A_(nn, nn);
      if (l == nn) {
        wr[nn] = x + t;
        wi[nn] = 0.0;
        --nn;
      } else {
        y = A_(nn - 1, nn - 1);
        w = A_(nn, nn - 1) * A_(nn - 1, nn);
        if (l == nn - 1) {
          p = 0.5 * (y - x);
          q = p * p + w;
          z = sqrt(fabs(q));
          x += t;
          if (q >= 0.0) {
            z = p + sgn_of(z, p);
            wr[nn - 1] = wr[nn] = x + z;
            if (z != 0.0) wr[nn] = x - w / z;
            wi[nn - 1] = wi[nn] = 0.0;
          } else {
            wr[nn - 1] = wr[nn] = x + p;
            wi[nn - 1] = z;
            wi[nn] = -z;
          }
          nn -= 2;
        } else {
          if (its == 30) return false;
          if (its == 10 || its == 20) {
            t += x;
            for (int i = 0; i <= nn; ++i) A_(i, i) -= x;
            s = fabs(A_(nn, nn - 1)) + fabs(A_(nn - 1, nn - 2));
            y = x = 0.75 * s;
            w = -0.4375 * s * s;
          }
          ++its;
          int m;
          for (m = nn - 2; m >= l; --m) {
            z = A_(m, m);
            r = x - z;
            s = y - z;
            p = (r * s - w) / A_(m + 1, m) + A_(m, m + 1);
            q = A_(m + 1, m + 1) - z - r - s;
            r = A_(m + 2, m + 1);
            s = fabs(p) + fabs(q) + fabs(r);
            p /= s;
            q /= s;
            r /= s;
            if (m == l) break;
            const double u = fabs(A_(m, m - 1)) * (fabs(q) + fabs(r));
            const double v = fabs(p) * (fabs(A_(m - 1, m - 1)) + fabs(z) + fabs(A_(m + 1, m + 1)));
            if (u + v == v) break;
          }
          for (int i = m + 2; i <= nn; ++i) {
            A_(i, i - 2) = 0.0;
            if (i != m + 2) A_(i, i - 3) = 0.0;
          }
          for (int k = m; k <= nn - 1; ++k) {
            if (k != m) {
              p = A_(k, k - 1);
              q = A_(k + 1, k - 1);
              r = 0.0;
              if (k != nn - 1) r = A_(k + 2, k - 1);
              if ((x = fabs(p) + fabs(q) + fabs(r)) != 0.0) {
                p /= x;
                q /= x;
                r /= x;
              }
            }
            if ((s = sgn_of(sqrt(p * p + q * q + r * r), p)) != 0.0) {
              if (k == m) {
                if (l != m) A_(k, k - 1) = -A_(k, k - 1);
              } else {
                A_(k, k - 1) = -s * x;
              }
              p += s;
              x = p / s;
              y = q / s;
              z = r / s;
              q /= p;
              r /= p;
              for (int j = k; j <= nn; ++j) {
                p = A_(k, j) + q * A_(k + 1, j);
                if (k != nn - 1) {
                  p += r * A_(k + 2, j);
                  A_(k + 2, j) -= p * z;
                }
                A_(k + 1, j) -= p * y;
                A_(k, j) -= p * x;
              }
              const int mmin = nn < k + 3 ? nn : k + 3;
              for (int i = l; i <= mmin; ++i) {
                p = x * A_(i, k) + y * A_(i, k + 1);
                if (k != nn - 1) {
                  p += z * A_(i, k + 2);
                  A_(i, k + 2) -= p * r;
                }
                A_(i, k + 1) -= p * q;
                A_(i, k) -= p;
              }
            }
          }
        }
      }
    } while (l < nn - 1);
  }
  return true;
#undef A_
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
  hessenberg(h, n, n);
  if (!hqr(h, n, n, wr, wi)) return 1;
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
