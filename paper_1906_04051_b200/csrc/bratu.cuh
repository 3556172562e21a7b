// Device FEM assembly of the Bratu system (the caller side of the hot path,
// SURVEY §8(f) row 1): closed-form CSR pattern (assembly.cpp:139-194), the
// Jacobian values (assembly.cpp:248-314) and the residual (assembly.cpp:196-246)
// for tri-quadratic 27-node hexahedra on the unit cube.
//
// Every entry accumulates its element contributions in ascending element order
// with the reference's operation order and no FMA contraction, so at u = 0
// (the first Newton system, exp(0) = 1 exactly) the matrix and right-hand side
// are bit-identical to the reference assembly.  For u != 0 the only difference
// is the last-ulp behaviour of exp().
#pragma once

#include <math.h>
#include <stdint.h>

#include <cmath>

namespace pgm {
namespace bratu {

struct Table {
  double phi[27][27];   // [quadrature point][local node]
  double sref[27][27];  // reference stiffness sum_q w grad_a . grad_b
  double w[27];         // quadrature weights
};

__constant__ Table c_tab;

// ---- host table (same expression order as the reference's build_table) ----
inline void lag3(double x, double* v) {
  v[0] = 0.5 * x * (x - 1.0);
  v[1] = 1.0 - x * x;
  v[2] = 0.5 * x * (x + 1.0);
}
inline void dlag3(double x, double* v) {
  v[0] = x - 0.5;
  v[1] = -2.0 * x;
  v[2] = x + 0.5;
}

#if defined(__GNUC__) && !defined(__clang__)
__attribute__((optimize("fp-contract=off")))
#endif
inline void build_table(Table& t) {
  const double g = std::sqrt(0.6);
  const double pts[3] = {-g, 0.0, g};
  const double wts[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
  double grad[27][27][3];
  int q = 0;
  for (int qz = 0; qz < 3; ++qz)
    for (int qy = 0; qy < 3; ++qy)
      for (int qx = 0; qx < 3; ++qx) {
        t.w[q] = wts[qx] * wts[qy] * wts[qz];
        double lx[3], ly[3], lz[3], dx[3], dy[3], dz[3];
        lag3(pts[qx], lx);
        lag3(pts[qy], ly);
        lag3(pts[qz], lz);
        dlag3(pts[qx], dx);
        dlag3(pts[qy], dy);
        dlag3(pts[qz], dz);
        int a = 0;
        for (int az = 0; az < 3; ++az)
          for (int ay = 0; ay < 3; ++ay)
            for (int ax = 0; ax < 3; ++ax) {
              t.phi[q][a] = lx[ax] * ly[ay] * lz[az];
              grad[q][a][0] = dx[ax] * ly[ay] * lz[az];
              grad[q][a][1] = lx[ax] * dy[ay] * lz[az];
              grad[q][a][2] = lx[ax] * ly[ay] * dz[az];
              ++a;
            }
        ++q;
      }
  for (int a = 0; a < 27; ++a)
    for (int b = 0; b < 27; ++b) {
      double s = 0.0;
      for (int k = 0; k < 27; ++k)
        s += t.w[k] * (grad[k][a][0] * grad[k][b][0] + grad[k][a][1] * grad[k][b][1] +
                       grad[k][a][2] * grad[k][b][2]);
      t.sref[a][b] = s;
    }
}

// ---- per-axis stencil reach (assembly.cpp:67-79) ----
__host__ __device__ __forceinline__ uint32_t reach(uint32_t i, uint32_t last, uint32_t* lo) {
  uint32_t a, b;
  if (i % 2 == 1) {
    a = i - 1;
    b = i + 1;
  } else {
    a = i >= 2 ? i - 2 : 0;
    b = (i + 2 < last) ? i + 2 : last;
  }
  *lo = a;
  return b - a + 1;
}

struct Mesh {
  uint32_t n_e, na;       // elements / node lines per axis
  uint64_t plane;         // na^2
  uint32_t row_begin;     // first assembled row (partitioned assembly)
  uint32_t nrows;
  double lambda, vol, stiff_sc;
};

__device__ __forceinline__ bool dirichlet(uint32_t ix, uint32_t iy, uint32_t last) {
  return ix == 0 || ix == last || iy == 0 || iy == last;
}

// row lengths into rp[1 + i] (rp[0] = 0), later scanned
__global__ void k_row_len(Mesh M, unsigned* rp) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= M.nrows) return;
  const uint64_t v = M.row_begin + i;
  const uint32_t ix = (uint32_t)(v % M.na), iy = (uint32_t)((v / M.na) % M.na),
                 iz = (uint32_t)(v / M.plane);
  const uint32_t last = M.na - 1;
  uint32_t lo;
  unsigned len = 1;
  if (!dirichlet(ix, iy, last)) len = reach(ix, last, &lo) * reach(iy, last, &lo) * reach(iz, last, &lo);
  rp[i + 1] = len;
  if (i == 0) rp[0] = 0;
}

// column ids, ascending (x fastest)
__global__ void k_cols(Mesh M, const unsigned* rp, unsigned* ci, double* va) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= M.nrows) return;
  const uint64_t v = M.row_begin + i;
  const uint32_t ix = (uint32_t)(v % M.na), iy = (uint32_t)((v / M.na) % M.na),
                 iz = (uint32_t)(v / M.plane);
  const uint32_t last = M.na - 1;
  unsigned k = rp[i];
  if (dirichlet(ix, iy, last)) {
    ci[k] = (unsigned)v;
    va[k] = 1.0;
    return;
  }
  uint32_t xl, yl, zl;
  const uint32_t xn = reach(ix, last, &xl), yn = reach(iy, last, &yl), zn = reach(iz, last, &zl);
  for (uint32_t cz = zl; cz < zl + zn; ++cz)
    for (uint32_t cy = yl; cy < yl + yn; ++cy)
      for (uint32_t cx = xl; cx < xl + xn; ++cx)
        ci[k++] = (unsigned)(cx + M.na * (cy + (uint64_t)M.na * cz));
}

// f[e][q] = ((lambda * vol) * w_q) * exp(sum_a ue[a] phi[q][a])   (assembly.cpp:99-110)
__global__ void k_elem_f(Mesh M, const double* __restrict__ u, double* f, uint64_t e0,
                         uint64_t ne_count) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= ne_count * 27) return;
  const uint64_t e = e0 + t / 27;
  const int q = (int)(t % 27);
  const uint32_t ex = (uint32_t)(e % M.n_e), ey = (uint32_t)((e / M.n_e) % M.n_e),
                 ez = (uint32_t)(e / ((uint64_t)M.n_e * M.n_e));
  double uq = 0.0;
  if (u) {
    int a = 0;
    for (uint32_t az = 0; az < 3; ++az)
      for (uint32_t ay = 0; ay < 3; ++ay)
        for (uint32_t ax = 0; ax < 3; ++ax) {
          const uint64_t gid = (2 * ex + ax) + M.na * ((2 * ey + ay) + (uint64_t)M.na * (2 * ez + az));
          uq = __dadd_rn(uq, __dmul_rn(u[gid], c_tab.phi[q][a]));
          ++a;
        }
  }
  f[t] = __dmul_rn(__dmul_rn(__dmul_rn(M.lambda, M.vol), c_tab.w[q]), exp(uq));
}

// element range along one axis containing node index i: [lo, hi]
__device__ __forceinline__ void elem_range(uint32_t i, uint32_t n_e, int* lo, int* hi) {
  if (i & 1) {
    *lo = *hi = (int)(i >> 1);
  } else {
    *lo = (int)(i >> 1) - 1;
    *hi = (int)(i >> 1);
    if (*lo < 0) *lo = 0;
    if (*hi > (int)n_e - 1) *hi = (int)n_e - 1;
  }
}

// Jacobian values: one warp per free row, lane b < 27 computes the element
// block entry eb[a][b] and adds it to the row slot of column gid[b]
// (assembly.cpp:258-283: eb = -stiff*sref, then += (f_q phi_qa) phi_qb over q).
__global__ void k_jac_values(Mesh M, const unsigned* rp, const double* __restrict__ f,
                             uint64_t e0, double* va) {
  __shared__ double rows_s[8][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  if (i >= M.nrows) return;
  const uint64_t v = M.row_begin + i;
  const uint32_t ix = (uint32_t)(v % M.na), iy = (uint32_t)((v / M.na) % M.na),
                 iz = (uint32_t)(v / M.plane);
  const uint32_t last = M.na - 1;
  if (dirichlet(ix, iy, last)) {
    if (lane == 0) va[rp[i]] = 1.0;
    return;
  }
  uint32_t xl, yl, zl;
  const uint32_t xn = reach(ix, last, &xl), yn = reach(iy, last, &yl);
  reach(iz, last, &zl);
  const unsigned len = rp[i + 1] - rp[i];
  double* rs = rows_s[warp];
  for (unsigned p = lane; p < len; p += 32) rs[p] = 0.0;
  __syncwarp();
  int xlo, xhi, ylo, yhi, zlo, zhi;
  elem_range(ix, M.n_e, &xlo, &xhi);
  elem_range(iy, M.n_e, &ylo, &yhi);
  elem_range(iz, M.n_e, &zlo, &zhi);
  for (int ez = zlo; ez <= zhi; ++ez)
    for (int ey = ylo; ey <= yhi; ++ey)
      for (int ex = xlo; ex <= xhi; ++ex) {
        const uint64_t e = (uint64_t)ex + M.n_e * ((uint64_t)ey + (uint64_t)M.n_e * ez);
        const int a = (int)(ix - 2 * ex) + 3 * (int)(iy - 2 * ey) + 9 * (int)(iz - 2 * ez);
        if (lane < 27) {
          const int b = lane;
          const int bx = b % 3, by = (b / 3) % 3, bz = b / 9;
          const double* fe = f + (e - e0) * 27;
          double eb = __dmul_rn(-M.stiff_sc, c_tab.sref[a][b]);
          for (int q = 0; q < 27; ++q) {
            const double fa = __dmul_rn(fe[q], c_tab.phi[q][a]);
            eb = __dadd_rn(eb, __dmul_rn(fa, c_tab.phi[q][b]));
          }
          const uint32_t cx = 2 * ex + bx, cy = 2 * ey + by, cz = 2 * ez + bz;
          const unsigned pos = ((cz - zl) * yn + (cy - yl)) * xn + (cx - xl);
          rs[pos] = __dadd_rn(rs[pos], eb);
        }
        __syncwarp();
      }
  double* out = va + rp[i];
  for (unsigned p = lane; p < len; p += 32) out[p] = rs[p];
}

// rhs = -R(u): free rows sum the element residuals in ascending element order
// (re[a] = -stiff * sum_b sref[a][b] ue[b] + sum_q f_q phi_qa); Dirichlet rows
// carry R_i = u_i (assembly.cpp:206-244).
__global__ void k_residual_rhs(Mesh M, const double* __restrict__ u, const double* __restrict__ f,
                               uint64_t e0, double* rhs) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= M.nrows) return;
  const uint64_t v = M.row_begin + i;
  const uint32_t ix = (uint32_t)(v % M.na), iy = (uint32_t)((v / M.na) % M.na),
                 iz = (uint32_t)(v / M.plane);
  const uint32_t last = M.na - 1;
  if (dirichlet(ix, iy, last)) {
    rhs[i] = u ? -u[v] : -0.0;
    return;
  }
  int xlo, xhi, ylo, yhi, zlo, zhi;
  elem_range(ix, M.n_e, &xlo, &xhi);
  elem_range(iy, M.n_e, &ylo, &yhi);
  elem_range(iz, M.n_e, &zlo, &zhi);
  double R = 0.0;
  for (int ez = zlo; ez <= zhi; ++ez)
    for (int ey = ylo; ey <= yhi; ++ey)
      for (int ex = xlo; ex <= xhi; ++ex) {
        const uint64_t e = (uint64_t)ex + M.n_e * ((uint64_t)ey + (uint64_t)M.n_e * ez);
        const int a = (int)(ix - 2 * ex) + 3 * (int)(iy - 2 * ey) + 9 * (int)(iz - 2 * ez);
        double s = 0.0;
        if (u) {
          int b = 0;
          for (uint32_t bz = 0; bz < 3; ++bz)
            for (uint32_t by = 0; by < 3; ++by)
              for (uint32_t bx = 0; bx < 3; ++bx) {
                const uint64_t gid =
                    (2 * ex + bx) + M.na * ((2 * ey + by) + (uint64_t)M.na * (2 * ez + bz));
                s = __dadd_rn(s, __dmul_rn(c_tab.sref[a][b], u[gid]));
                ++b;
              }
        } else {
          for (int b = 0; b < 27; ++b) s = __dadd_rn(s, __dmul_rn(c_tab.sref[a][b], 0.0));
        }
        const double* fe = f + (e - e0) * 27;
        double load = 0.0;
        for (int q = 0; q < 27; ++q) load = __dadd_rn(load, __dmul_rn(fe[q], c_tab.phi[q][a]));
        const double re = __dadd_rn(__dmul_rn(-M.stiff_sc, s), load);
        R = __dadd_rn(R, re);
      }
  rhs[i] = -R;
}

}  // namespace bratu
}  // namespace pgm
