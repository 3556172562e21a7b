// pgmres/dgmres.hpp — header-only C++ drop-in for the reference's linear-solve
// API (/root/reference/proj/include/dgmres/{gmres,deflation,sparse}.hpp) on top
// of the C ABI in pgmres.h.  A caller such as newton.cpp:60-70 keeps its code:
//
//   reference                                   drop-in (this header)
//   dgmres::CsrMatrix          sparse.hpp:17    pgmres::CsrMatrix (same fields)
//   dgmres::GmresConfig        gmres.hpp:17     pgmres::GmresConfig (same fields)
//   dgmres::GmresReport        gmres.hpp:31     pgmres::GmresReport (+ write_csv)
//   dgmres::DeflationConfig    deflation.hpp:15 pgmres::DeflationConfig
//   dgmres::Deflator           deflation.hpp:35 pgmres::Deflator (state on the GPU)
//   dgmres::Executor           parallel.hpp:86  pgmres::DeviceExecutor
//   dgmres::deflated_gmres     deflation.hpp:97 pgmres::deflated_gmres
//   dgmres::gmres_restarted    gmres.hpp:110    pgmres::gmres_restarted (opA = CSR,
//                                               opM = nullptr; no std::function ops)
//
// Errors keep the reference's exception types and messages:
// std::invalid_argument (m = 0, r_max = 0, ...) and std::runtime_error
// ("gmres: initial residual is not finite", "gmres: non-finite Arnoldi
// coefficient at restart X, step Y", "gmres: singular projection in least
// squares", ...).  Link with -lpgmres (paper_1906_04051_b200/_lib).
#pragma once

#include <cstdint>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../pgmres.h"
#include "pattern_hash.hpp"

namespace pgmres {

using index_t = std::uint32_t;
using DenseVector = std::vector<double>;

struct CsrMatrix {
  index_t n = 0;
  std::vector<index_t> row_ptr;
  std::vector<index_t> col_idx;
  std::vector<double> values;
  std::uint64_t nnz() const { return col_idx.size(); }
};

struct GmresConfig {
  std::uint32_t m = 50;
  std::uint32_t max_restarts = 100;
  double rel_tol = 1e-8;
  bool fixed_iterations = false;
  double breakdown_scale = 1e-14;
};

struct DeflationConfig {
  std::uint32_t r_max = 20;
  std::uint32_t drop = 1;
  double accept_tol = 1e-8;
  std::uint32_t inv_power_maxit = 500;
  double inv_power_tol = 1e-10;
  std::uint32_t power_maxit = 200;
};

struct InnerRecord {
  std::uint32_t restart;
  std::uint32_t inner;
  double monitored;
};

struct DeflationRecord {
  std::uint32_t restart;
  std::uint32_t r;
  double mu;
  double smallest_ritz;
};

struct GmresReport {
  double beta0 = 0.0;
  std::vector<InnerRecord> inner;
  std::vector<double> explicit_residual;
  std::uint32_t restarts = 0;
  std::uint64_t total_inner = 0;
  bool converged = false;
  bool breakdown = false;
  double final_relative = 0.0;
  double solve_seconds = 0.0;  // device time of the solve

  // restart,inner_step,monitored_residual,explicit_residual (gmres.cpp:117-130)
  void write_csv(std::ostream& os) const {
    os << "restart,inner_step,monitored_residual,explicit_residual\n";
    const auto prec = os.precision(17);
    for (std::size_t i = 0; i < inner.size(); ++i) {
      const InnerRecord& rec = inner[i];
      const bool closes = i + 1 == inner.size() || inner[i + 1].restart != rec.restart;
      os << rec.restart << ',' << rec.inner << ',' << rec.monitored << ',';
      if (closes && rec.restart < explicit_residual.size()) os << explicit_residual[rec.restart];
      os << '\n';
    }
    os.precision(prec);
  }
};

namespace detail {
inline void check(pgm_status s, const pgm_context* ctx) {
  if (s == PGM_OK) return;
  const std::string msg = pgm_last_error(ctx);
  if (s == PGM_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
}  // namespace detail

// One GPU (one rank of the z-slab partition when world > 1).
class DeviceExecutor {
 public:
  explicit DeviceExecutor(int device = 0) : device_(device) {}
  DeviceExecutor(int device, std::uint32_t n_axis, int rank, int world, const void* nccl_id)
      : device_(device), n_axis_(n_axis), rank_(rank), world_(world), nccl_id_(nccl_id) {}
  ~DeviceExecutor() {
    release();
    if (ctx_) pgm_context_destroy(ctx_);
  }
  DeviceExecutor(const DeviceExecutor&) = delete;
  DeviceExecutor& operator=(const DeviceExecutor&) = delete;

  pgm_context* context(index_t n_global) {
    if (!ctx_) {
      pgm_context_config cfg{device_, rank_, world_, nccl_id_, nullptr, n_axis_, n_global, 1};
      detail::check(pgm_context_create(&cfg, &ctx_), nullptr);
      n_global_ = n_global;
    } else if (n_global != n_global_) {
      throw std::invalid_argument("DeviceExecutor: matrix size changed");
    }
    return ctx_;
  }
  pgm_context* handle() const { return ctx_; }

  // Upload (or refresh the values of) a host CSR matrix.  ONE device matrix
  // stays resident, keyed on the pattern's identity (n, nnz, hash of row_ptr
  // and col_idx — content, not the host object's address): the same pattern
  // only moves the values (Newton re-assembles values on a fixed pattern,
  // assembly.cpp:253); a new pattern releases the previous device copy.
  pgm_matrix* matrix(const CsrMatrix& A) {
    pgm_context* ctx = context(world_ == 1 ? A.n : n_global_);
    if (A.row_ptr.size() != std::size_t(A.n) + 1)
      throw std::invalid_argument("CsrMatrix: row_ptr must have n + 1 entries");
    const std::uint64_t h =
        detail::pattern_hash(A.row_ptr.data(), A.n, A.col_idx.data(), A.col_idx.size());
    if (cur_.mat && cur_.n == A.n && cur_.nnz == A.nnz() && cur_.hash == h) {
      detail::check(pgm_matrix_update_values(cur_.mat, A.values.data(), 0), ctx);
      return cur_.mat;
    }
    release();
    pgm_csr_view v{A.n, A.nnz(), A.row_ptr.data(), A.col_idx.data(), A.values.data()};
    pgm_matrix* m = nullptr;
    detail::check(pgm_matrix_upload(ctx, &v, 0, &m), ctx);
    cur_ = Entry{A.n, A.nnz(), h, m};
    return m;
  }
  // Drop the resident device matrix (the next solve uploads again).
  void release() {
    if (cur_.mat) pgm_matrix_destroy(cur_.mat);
    cur_ = Entry{};
  }

  void spmv(const CsrMatrix& A, const DenseVector& x, DenseVector& y) {
    pgm_matrix* m = matrix(A);
    y.resize(x.size());
    detail::check(pgm_spmv(m, x.data(), y.data(), 0), ctx_);
  }

 private:
  struct Entry {
    index_t n = 0;
    std::uint64_t nnz = 0, hash = 0;
    pgm_matrix* mat = nullptr;
  };
  int device_ = 0;
  std::uint32_t n_axis_ = 0;
  int rank_ = 0, world_ = 1;
  const void* nccl_id_ = nullptr;
  index_t n_global_ = 0;
  pgm_context* ctx_ = nullptr;
  Entry cur_;
};

class Deflator {
 public:
  explicit Deflator(DeflationConfig cfg = {}) : cfg_(cfg) {
    if (cfg_.r_max == 0) throw std::invalid_argument("deflation: r_max must be positive");
    if (cfg_.drop == 0) throw std::invalid_argument("deflation: drop must be positive");
  }
  ~Deflator() {
    if (d_) pgm_deflator_destroy(d_);
  }
  Deflator(const Deflator&) = delete;
  Deflator& operator=(const Deflator&) = delete;

  std::uint32_t rank() const { return info().r; }
  double mu() const { return info().mu; }
  std::uint32_t skipped_updates() const { return info().skipped; }
  void reset() {
    if (d_) detail::check(pgm_deflator_reset(d_), ctx_);
  }
  std::vector<DeflationRecord> history() const {
    const Info i = info();
    std::vector<pgm_deflation_record> raw(i.nh);
    if (i.nh) detail::check(pgm_deflator_history(d_, raw.data(), i.nh), ctx_);
    std::vector<DeflationRecord> out;
    for (const auto& r : raw) out.push_back({r.restart, r.r, r.mu, r.smallest_ritz});
    return out;
  }
  // restart,r,mu,smallest_ritz (deflation.cpp:266-273)
  void write_csv(std::ostream& os) const {
    os << "restart,r,mu,smallest_ritz\n";
    const auto prec = os.precision(17);
    for (const auto& h : history())
      os << h.restart << ',' << h.r << ',' << h.mu << ',' << h.smallest_ritz << '\n';
    os.precision(prec);
  }
  pgm_deflator* bind(pgm_context* ctx) {
    if (!d_) {
      pgm_deflation_config c{cfg_.r_max, cfg_.drop, cfg_.accept_tol, cfg_.inv_power_maxit,
                             cfg_.inv_power_tol, cfg_.power_maxit};
      detail::check(pgm_deflator_create(ctx, &c, &d_), ctx);
      ctx_ = ctx;
    } else if (ctx != ctx_) {
      throw std::invalid_argument("Deflator is bound to another executor");
    }
    return d_;
  }

 private:
  struct Info {
    std::uint32_t r = 0, skipped = 0, nh = 0;
    double mu = 0.0;
  };
  Info info() const {
    Info i;
    if (d_) detail::check(pgm_deflator_info(d_, &i.r, &i.mu, &i.skipped, &i.nh), ctx_);
    return i;
  }
  DeflationConfig cfg_;
  pgm_deflator* d_ = nullptr;
  pgm_context* ctx_ = nullptr;
};

namespace detail {
inline GmresReport solve(const CsrMatrix& A, const DenseVector& b, DenseVector& x,
                         const GmresConfig& cfg, Deflator* d, DeviceExecutor& ex) {
  if (cfg.m == 0) throw std::invalid_argument("GmresWorkspace: m must be positive");
  pgm_matrix* m = ex.matrix(A);
  pgm_context* ctx = ex.handle();
  pgm_deflator* dd = d ? d->bind(ctx) : nullptr;
  pgm_gmres_config c{cfg.m, cfg.max_restarts, cfg.rel_tol, cfg.fixed_iterations ? 1 : 0,
                     cfg.breakdown_scale};
  x.resize(b.size());
  pgm_report r{};
  check(pgm_solve(ctx, m, dd, b.data(), x.data(), &c, 0, &r), ctx);
  GmresReport out;
  out.beta0 = r.beta0;
  out.restarts = r.restarts;
  out.total_inner = r.total_inner;
  out.converged = r.converged != 0;
  out.breakdown = r.breakdown != 0;
  out.final_relative = r.final_relative;
  out.solve_seconds = r.solve_seconds;
  for (std::uint32_t i = 0; i < r.n_inner; ++i)
    out.inner.push_back({r.inner_restart[i], r.inner_step[i], r.inner_monitored[i]});
  out.explicit_residual.assign(r.explicit_residual, r.explicit_residual + r.restarts);
  pgm_report_free(&r);
  return out;
}
}  // namespace detail

// deflation.hpp:97-98
inline GmresReport deflated_gmres(const CsrMatrix& A, const DenseVector& b, DenseVector& x,
                                  const GmresConfig& cfg, Deflator& d, DeviceExecutor& ex) {
  return detail::solve(A, b, x, cfg, &d, ex);
}

// gmres.hpp:110-113 for the production pair (opA = CSR SpMV, opM = nullptr).
inline GmresReport gmres_restarted(const CsrMatrix& A, std::nullptr_t, const DenseVector& b,
                                   DenseVector& x, const GmresConfig& cfg, DeviceExecutor& ex) {
  return detail::solve(A, b, x, cfg, nullptr, ex);
}

// ---- newton.hpp:15-54: the Newton driver, device-resident ------------------
struct NewtonConfig {  // newton.hpp:15-23
  std::uint32_t max_iters = 30;
  double update_tol = 1e-8;
  GmresConfig gmres{50, 100, 1e-10, false, 1e-14};
  DeflationConfig deflation{};
  bool use_deflation = true;
  bool continuation = false;
  std::uint32_t continuation_steps = 4;
};

struct NewtonIterRecord {  // newton.hpp:25-32
  std::uint32_t iter;
  double lambda;
  double update_inf;
  double residual_norm;
  std::uint32_t gmres_restarts;
  std::uint64_t gmres_inner;
};

struct NewtonReport {  // newton.hpp:34-43
  std::vector<NewtonIterRecord> iters;
  bool converged = false;
  double final_residual = 0.0;
  double final_update = 0.0;
  std::uint64_t total_inner = 0;
  double seconds = 0.0;
};

/// newton_solve(build_mesh(n_e), lambda, u, cfg, ex) for the Bratu problem:
/// assembly, solves, update and norms on the GPU (pgm_newton_solve).  u is the
/// global iterate (initial guess in, solution out).
inline NewtonReport newton_solve(std::uint32_t n_e, double lambda, DenseVector& u,
                                 const NewtonConfig& cfg, DeviceExecutor& ex) {
  if (cfg.max_iters == 0) throw std::invalid_argument("newton: max_iters must be positive");
  const std::size_t na = 2 * std::size_t(n_e) + 1;
  if (u.size() != na * na * na) u.assign(na * na * na, 0.0);
  pgm_context* ctx = ex.context(static_cast<index_t>(u.size()));
  pgm_newton_config c{};
  c.max_iters = cfg.max_iters;
  c.update_tol = cfg.update_tol;
  c.gmres = pgm_gmres_config{cfg.gmres.m, cfg.gmres.max_restarts, cfg.gmres.rel_tol,
                             cfg.gmres.fixed_iterations ? 1 : 0, cfg.gmres.breakdown_scale};
  c.deflation = pgm_deflation_config{cfg.deflation.r_max, cfg.deflation.drop,
                                     cfg.deflation.accept_tol, cfg.deflation.inv_power_maxit,
                                     cfg.deflation.inv_power_tol, cfg.deflation.power_maxit};
  c.use_deflation = cfg.use_deflation ? 1 : 0;
  c.continuation = cfg.continuation ? 1 : 0;
  c.continuation_steps = cfg.continuation_steps;
  pgm_newton_report r{};
  detail::check(pgm_newton_solve(ctx, n_e, lambda, u.data(), 0, &c, &r), ctx);
  NewtonReport out;
  for (std::uint32_t i = 0; i < r.n_iters; ++i)
    out.iters.push_back({r.iters[i].iter, r.iters[i].lambda, r.iters[i].update_inf,
                         r.iters[i].residual_norm, r.iters[i].gmres_restarts,
                         r.iters[i].gmres_inner});
  out.converged = r.converged != 0;
  out.final_residual = r.final_residual;
  out.final_update = r.final_update;
  out.total_inner = r.total_inner;
  out.seconds = r.seconds;
  pgm_newton_report_free(&r);
  return out;
}

}  // namespace pgmres

