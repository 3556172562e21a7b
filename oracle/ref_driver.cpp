// oracle/_ref driver — TEST INFRASTRUCTURE ONLY.
//
// A C-ABI harness around the UNMODIFIED reference sources
// (/root/reference/proj/src/*.cpp compiled verbatim by oracle/Makefile) so
// that Python tests, the golden-fixture generator and bench.py's CPU arm can
// call the reference's own public API:
//   * first Newton system J(0) x = -R(0)   (bratu_bench.cpp:135-144 pattern)
//   * deflated_gmres / gmres_restarted      (deflation.hpp:97-98, gmres.hpp:110-113)
//   * Deflator push/apply/truncate          (deflation.hpp:35-89)
//   * newton_solve                          (newton.hpp:53-54)
//   * the speedup timing loop               (bratu_bench.cpp:282-300)
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs load this library.  Nothing here is product code.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "dgmres/assembly.hpp"
#include "dgmres/deflation.hpp"
#include "dgmres/gmres.hpp"
#include "dgmres/mesh.hpp"
#include "dgmres/newton.hpp"
#include "dgmres/parallel.hpp"
#include "dgmres/sparse.hpp"

using namespace dgmres;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

struct System {
  StructuredMesh mesh;
  CsrMatrix jac;
  DenseVector rhs;
};

std::unique_ptr<Executor> make_exec(std::uint32_t ne, unsigned threads, int deterministic) {
  if (threads == 0 || ne == 0) return std::make_unique<Executor>();
  return std::make_unique<Executor>(partition_rows(build_mesh(ne), threads),
                                    deterministic != 0);
}

CsrMatrix csr_from(std::uint32_t n, std::uint64_t nnz, const std::uint32_t* rp,
                   const std::uint32_t* ci, const double* v) {
  CsrMatrix a;
  a.n = n;
  a.row_ptr.assign(rp, rp + n + 1);
  a.col_idx.assign(ci, ci + nnz);
  a.values.assign(v, v + nnz);
  return a;
}

}  // namespace

extern "C" {

struct RefdConfig {
  std::uint32_t m, max_restarts;
  double rel_tol;
  std::int32_t fixed_iterations;
  double breakdown_scale;
  std::int32_t use_deflation;
  std::uint32_t r_max, drop;
  double accept_tol;
  std::uint32_t inv_power_maxit;
  double inv_power_tol;
  std::uint32_t power_maxit;
  std::uint32_t ne;       // mesh for partition_rows (0 = sequential executor)
  std::uint32_t threads;  // executor workers (0 = sequential executor)
  std::int32_t deterministic;
  std::int32_t audit;     // per-restart U^T U / T audits (acceptance.cpp:100-122)
};

struct RefdReport {
  double beta0;
  std::uint32_t restarts;
  std::uint64_t total_inner;
  std::int32_t converged, breakdown;
  double final_relative;
  std::uint32_t n_inner;  // records written
  // deflation summary
  std::uint32_t rank, skipped, n_hist;
  double mu;
  double ortho_max, tmatch_max;
  std::uint32_t rank_max;
  double wall_s;
};

const char* refd_last_error() { return g_err.c_str(); }

// ---- first Newton system --------------------------------------------------
void* refd_system_create(std::uint32_t ne, double lambda, const double* u_in,
                         std::uint32_t threads) {
  try {
    auto s = std::make_unique<System>();
    s->mesh = build_mesh(ne);
    auto ex = make_exec(ne, threads, 1);
    DenseVector u(s->mesh.n_nodes, 0.0), r;
    if (u_in) u.assign(u_in, u_in + s->mesh.n_nodes);
    assemble_residual(s->mesh, lambda, u, r, *ex);
    assemble_jacobian(s->mesh, lambda, u, s->jac, *ex);
    s->rhs.resize(s->mesh.n_nodes);
    for (index_t i = 0; i < s->mesh.n_nodes; ++i) s->rhs[i] = -r[i];
    return s.release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
std::uint32_t refd_system_n(void* h) { return static_cast<System*>(h)->jac.n; }
std::uint64_t refd_system_nnz(void* h) { return static_cast<System*>(h)->jac.nnz(); }
void refd_system_export(void* h, std::uint32_t* rp, std::uint32_t* ci, double* v,
                        double* rhs) {
  const System& s = *static_cast<System*>(h);
  std::memcpy(rp, s.jac.row_ptr.data(), 4 * s.jac.row_ptr.size());
  std::memcpy(ci, s.jac.col_idx.data(), 4 * s.jac.col_idx.size());
  std::memcpy(v, s.jac.values.data(), 8 * s.jac.values.size());
  std::memcpy(rhs, s.rhs.data(), 8 * s.rhs.size());
}
void refd_system_free(void* h) { delete static_cast<System*>(h); }

std::uint64_t refd_pattern_nnz(std::uint32_t ne) { return pattern_nnz(build_mesh(ne)); }

int refd_residual(std::uint32_t ne, double lambda, const double* u_in, double* r_out) {
  try {
    const StructuredMesh mesh = build_mesh(ne);
    Executor ex;
    DenseVector u(u_in, u_in + mesh.n_nodes), r;
    assemble_residual(mesh, lambda, u, r, ex);
    std::memcpy(r_out, r.data(), 8 * r.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- kernels --------------------------------------------------------------
void refd_spmv(std::uint32_t n, std::uint64_t nnz, const std::uint32_t* rp,
               const std::uint32_t* ci, const double* v, const double* x, double* y) {
  const CsrMatrix a = csr_from(n, nnz, rp, ci, v);
  spmv(a, std::span<const double>(x, n), std::span<double>(y, n));
}

int refd_executor_kernels(std::uint32_t ne, std::uint32_t threads, std::int32_t det,
                          std::uint32_t n, std::uint64_t nnz, const std::uint32_t* rp,
                          const std::uint32_t* ci, const double* v, const double* x,
                          const double* w, double* y_out, double* dot_out) {
  try {
    const CsrMatrix a = csr_from(n, nnz, rp, ci, v);
    auto ex = make_exec(ne, threads, det);
    DenseVector xv(x, x + n), wv(w, w + n), y(n);
    ex->spmv(a, xv, y);
    std::memcpy(y_out, y.data(), 8 * n);
    dot_out[0] = ex->dot(xv, wv);
    dot_out[1] = ex->norm2(xv);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- the hot path: deflated_gmres / gmres_restarted ------------------------
int refd_solve(const RefdConfig* c, std::uint32_t n, std::uint64_t nnz,
               const std::uint32_t* rp, const std::uint32_t* ci, const double* v,
               const double* b_in, double* x_inout, RefdReport* rep,
               std::uint32_t* in_restart, std::uint32_t* in_step, double* in_mon,
               double* explicit_res, std::uint32_t* h_restart, std::uint32_t* h_r,
               double* h_mu, double* h_theta, double* t_out, double* u_out) {
  try {
    const CsrMatrix a = csr_from(n, nnz, rp, ci, v);
    auto ex = make_exec(c->ne, c->threads, c->deterministic);
    GmresConfig cfg;
    cfg.m = c->m;
    cfg.max_restarts = c->max_restarts;
    cfg.rel_tol = c->rel_tol;
    cfg.fixed_iterations = c->fixed_iterations != 0;
    cfg.breakdown_scale = c->breakdown_scale;
    DeflationConfig dcfg;
    dcfg.r_max = c->r_max;
    dcfg.drop = c->drop;
    dcfg.accept_tol = c->accept_tol;
    dcfg.inv_power_maxit = c->inv_power_maxit;
    dcfg.inv_power_tol = c->inv_power_tol;
    dcfg.power_maxit = c->power_maxit;
    Deflator d(dcfg);
    DenseVector b(b_in, b_in + n), x(x_inout, x_inout + n);

    double ortho_max = 0.0, tmatch_max = 0.0;
    std::uint32_t rank_max = 0;
    GmresReport g;
    const auto t0 = std::chrono::steady_clock::now();
    if (c->use_deflation) {
      if (!c->audit) {
        g = deflated_gmres(a, b, x, cfg, d, *ex);
      } else {
        // deflated_gmres with the acceptance-style audit hook wrapped around
        // the deflation hook (acceptance.cpp:87-125).
        const LinearOp opA = [&](const DenseVector& in, DenseVector& out) {
          out.resize(in.size());
          ex->spmv(a, in, out);
        };
        const LinearOp opM = [&](const DenseVector& in, DenseVector& out) {
          d.apply(in, out, *ex);
        };
        const RestartHook refresh = deflation_hook(d, opA, *ex);
        DenseVector tin(n), tout(n);
        const RestartHook hook = [&](const RestartContext& ctx) {
          refresh(ctx);
          const std::uint32_t r = d.rank();
          rank_max = std::max(rank_max, r);
          if (r == 0) return;
          const Eigen::MatrixXd& U = d.basis_matrix();
          const Eigen::MatrixXd t = d.T_block();
          double tscale = 0.0;
          for (std::uint32_t i = 0; i < r; ++i)
            for (std::uint32_t j = 0; j < r; ++j) tscale = std::max(tscale, std::abs(t(i, j)));
          tscale = std::max(tscale, 1e-300);
          std::vector<std::vector<double>> au(r);
          for (std::uint32_t j = 0; j < r; ++j) {
            std::memcpy(tin.data(), U.col(j).data(), 8 * n);
            ex->spmv(a, tin, tout);
            au[j] = tout;
          }
          for (std::uint32_t i = 0; i < r; ++i)
            for (std::uint32_t j = 0; j < r; ++j) {
              double uu = 0.0, ua = 0.0;
              const double* ui = U.col(i).data();
              const double* uj = U.col(j).data();
              for (std::uint32_t q = 0; q < n; ++q) {
                uu += ui[q] * uj[q];
                ua += ui[q] * au[j][q];
              }
              ortho_max = std::max(ortho_max, std::abs(uu - (i == j ? 1.0 : 0.0)));
              tmatch_max = std::max(tmatch_max, std::abs(t(i, j) - ua) / tscale);
            }
        };
        g = gmres_restarted(opA, opM, b, x, cfg, *ex, hook);
      }
    } else {
      const LinearOp opA = [&](const DenseVector& in, DenseVector& out) {
        out.resize(in.size());
        ex->spmv(a, in, out);
      };
      g = gmres_restarted(opA, nullptr, b, x, cfg, *ex);
    }
    const auto t1 = std::chrono::steady_clock::now();

    std::memcpy(x_inout, x.data(), 8 * n);
    rep->beta0 = g.beta0;
    rep->restarts = g.restarts;
    rep->total_inner = g.total_inner;
    rep->converged = g.converged;
    rep->breakdown = g.breakdown;
    rep->final_relative = g.final_relative;
    rep->n_inner = static_cast<std::uint32_t>(g.inner.size());
    for (std::size_t i = 0; i < g.inner.size(); ++i) {
      if (in_restart) in_restart[i] = g.inner[i].restart;
      if (in_step) in_step[i] = g.inner[i].inner;
      if (in_mon) in_mon[i] = g.inner[i].monitored;
    }
    if (explicit_res)
      for (std::size_t i = 0; i < g.explicit_residual.size(); ++i)
        explicit_res[i] = g.explicit_residual[i];
    rep->rank = d.rank();
    rep->mu = d.mu();
    rep->skipped = d.skipped_updates();
    rep->n_hist = static_cast<std::uint32_t>(d.history().size());
    for (std::size_t i = 0; i < d.history().size(); ++i) {
      const DeflationRecord& hr = d.history()[i];
      if (h_restart) h_restart[i] = hr.restart;
      if (h_r) h_r[i] = hr.r;
      if (h_mu) h_mu[i] = hr.mu;
      if (h_theta) h_theta[i] = hr.smallest_ritz;
    }
    const std::uint32_t r = d.rank();
    if (t_out && r > 0) {
      const Eigen::MatrixXd t = d.T_block();
      std::memcpy(t_out, t.data(), 8 * std::size_t(r) * r);
    }
    if (u_out && r > 0) {
      const Eigen::MatrixXd& U = d.basis_matrix();
      for (std::uint32_t j = 0; j < r; ++j) std::memcpy(u_out + std::size_t(j) * n, U.col(j).data(), 8 * n);
    }
    rep->ortho_max = ortho_max;
    rep->tmatch_max = tmatch_max;
    rep->rank_max = rank_max;
    rep->wall_s = std::chrono::duration<double>(t1 - t0).count();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- resumable deflated solve (bench.py's reference arm) ----------------------
// The reference solve advanced one call at a time: each refd_session_run is
// deflated_gmres(A, b, x, cfg, d, ex) with x and the Deflator carried over, so
// consecutive calls with max_restarts = 1, fixed_iterations = 1 are the
// consecutive restart cycles of one solve (the per-call beta is the previous
// cycle's explicit residual, gmres.cpp:141-147,193).  The system, executor and
// deflator are built once (no per-call CSR copy).
struct Session {
  System sys;
  DenseVector x;
  std::unique_ptr<Executor> ex;
  std::unique_ptr<Deflator> d;
};

void* refd_session_create(void* system, std::uint32_t ne, std::uint32_t threads,
                          std::uint32_t r_max) {
  // threads: the solve's executor workers (the system may have been assembled
  // with another count; assembly is not part of the timed solve)
  try {
    auto s = std::make_unique<Session>();
    s->sys = std::move(*static_cast<System*>(system));
    s->x.assign(s->sys.jac.n, 0.0);
    s->ex = make_exec(ne, threads, 1);
    DeflationConfig dc;
    dc.r_max = r_max;
    s->d = std::make_unique<Deflator>(dc);
    return s.release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

int refd_session_run(void* sp, std::uint32_t m, std::uint32_t max_restarts, double rel_tol,
                     std::int32_t fixed_iterations, RefdReport* rep) {
  try {
    Session& s = *static_cast<Session*>(sp);
    GmresConfig cfg;
    cfg.m = m;
    cfg.max_restarts = max_restarts;
    cfg.rel_tol = rel_tol;
    cfg.fixed_iterations = fixed_iterations != 0;
    const auto t0 = std::chrono::steady_clock::now();
    const GmresReport g = deflated_gmres(s.sys.jac, s.sys.rhs, s.x, cfg, *s.d, *s.ex);
    const auto t1 = std::chrono::steady_clock::now();
    std::memset(rep, 0, sizeof(*rep));
    rep->beta0 = g.beta0;
    rep->restarts = g.restarts;
    rep->total_inner = g.total_inner;
    rep->converged = g.converged;
    rep->breakdown = g.breakdown;
    rep->final_relative = g.final_relative;
    rep->rank = s.d->rank();
    rep->mu = s.d->mu();
    rep->skipped = s.d->skipped_updates();
    rep->wall_s = std::chrono::duration<double>(t1 - t0).count();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void refd_session_reset(void* sp) {
  Session& s = *static_cast<Session*>(sp);
  std::fill(s.x.begin(), s.x.end(), 0.0);
  s.d->reset();
}

void refd_session_free(void* sp) { delete static_cast<Session*>(sp); }

// ---- Deflator unit-level access (test_deflation.cpp patterns) ---------------
void* refd_deflator_create(std::uint32_t r_max, std::uint32_t drop) {
  try {
    DeflationConfig cfg;
    cfg.r_max = r_max;
    cfg.drop = drop;
    return new Deflator(cfg);
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void refd_deflator_free(void* d) { delete static_cast<Deflator*>(d); }
int refd_deflator_push(void* d, std::uint32_t n, std::uint64_t nnz, const std::uint32_t* rp,
                       const std::uint32_t* ci, const double* v, const double* cand) {
  const CsrMatrix a = csr_from(n, nnz, rp, ci, v);
  Executor ex;
  const LinearOp opA = [&](const DenseVector& in, DenseVector& out) {
    out.resize(in.size());
    ex.spmv(a, in, out);
  };
  return static_cast<Deflator*>(d)->push_vector(DenseVector(cand, cand + n), opA, ex) ? 1 : 0;
}
void refd_deflator_truncate(void* d) { static_cast<Deflator*>(d)->truncate(); }
void refd_deflator_observe(void* d, double v) { static_cast<Deflator*>(d)->observe_ritz(v); }
void refd_deflator_reset(void* d) { static_cast<Deflator*>(d)->reset(); }
void refd_deflator_apply(void* d, std::uint32_t n, const double* v, double* w) {
  Executor ex;
  DenseVector in(v, v + n), out;
  static_cast<Deflator*>(d)->apply(in, out, ex);
  std::memcpy(w, out.data(), 8 * n);
}
void refd_deflator_state(void* dp, std::uint32_t* rank, double* mu, std::uint32_t* skipped,
                         double* t_out, double* u_out, std::uint32_t n) {
  const Deflator& d = *static_cast<Deflator*>(dp);
  *rank = d.rank();
  *mu = d.mu();
  *skipped = d.skipped_updates();
  const std::uint32_t r = d.rank();
  if (r == 0) return;
  if (t_out) {
    const Eigen::MatrixXd t = d.T_block();
    std::memcpy(t_out, t.data(), 8 * std::size_t(r) * r);
  }
  if (u_out)
    for (std::uint32_t j = 0; j < r; ++j)
      std::memcpy(u_out + std::size_t(j) * n, d.basis_matrix().col(j).data(), 8 * n);
}

// ---- Newton (caller of the hot path) ---------------------------------------
struct RefdNewtonRec {
  std::uint32_t iter;
  double lambda, update_inf, residual_norm;
  std::uint32_t gmres_restarts;
  std::uint64_t gmres_inner;
};

int refd_newton(std::uint32_t ne, double lambda, std::uint32_t max_iters, double update_tol,
                std::uint32_t m, std::uint32_t max_restarts, double rel_tol,
                std::int32_t use_deflation, std::int32_t continuation,
                std::uint32_t cont_steps, std::uint32_t threads, double* u_out,
                RefdNewtonRec* recs, std::uint32_t rec_cap, std::uint32_t* n_recs,
                std::int32_t* converged, double* final_residual, double* wall_s) {
  try {
    const StructuredMesh mesh = build_mesh(ne);
    // REFD_EXEC=nondet: the reference's non-deterministic executor (per-worker
    // partials) — used to measure the reference's own run-to-run spread
    const char* ev = std::getenv("REFD_EXEC");
    const int det = (ev && std::string(ev) == "nondet") ? 0 : 1;
    auto ex = make_exec(ne, threads, det);
    NewtonConfig cfg;
    cfg.max_iters = max_iters;
    cfg.update_tol = update_tol;
    cfg.gmres.m = m;
    cfg.gmres.max_restarts = max_restarts;
    cfg.gmres.rel_tol = rel_tol;
    cfg.use_deflation = use_deflation != 0;
    cfg.continuation = continuation != 0;
    cfg.continuation_steps = cont_steps;
    DenseVector u;
    const auto t0 = std::chrono::steady_clock::now();
    const NewtonReport rep = newton_solve(mesh, lambda, u, cfg, *ex);
    *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::memcpy(u_out, u.data(), 8 * u.size());
    *n_recs = static_cast<std::uint32_t>(rep.iters.size());
    for (std::size_t i = 0; i < rep.iters.size() && i < rec_cap; ++i) {
      const auto& r = rep.iters[i];
      recs[i] = {r.iter, r.lambda, r.update_inf, r.residual_norm, r.gmres_restarts,
                 r.gmres_inner};
    }
    *converged = rep.converged;
    *final_residual = rep.final_residual;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
