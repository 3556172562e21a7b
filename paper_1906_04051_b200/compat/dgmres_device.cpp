// Implementation of the source-compatible dgmres API (include/compat/dgmres/
// gmres.hpp, deflation.hpp) over the C ABI in include/pgmres.h.  Compiled
// into the CALLER's build in place of the reference's src/gmres.cpp and
// src/deflation.cpp; links against libpgmres.so.
//
// Device resources: one pgm_context per problem size (process-wide, on
// CUDA device $PGMRES_DEVICE, default 0) and ONE resident matrix.  A solve
// keys the resident matrix on the pattern's identity — n, nnz and a 64-bit
// hash of row_ptr and col_idx — so a new pattern (or the same pattern in a
// new CsrMatrix) is recognised by content, not by object address, and the
// previous device copy is released; the values are re-sent on every solve
// (Newton rewrites them in place on a fixed pattern, assembly.cpp:253).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <exception>
#include <map>
#include <ostream>
#include <stdexcept>
#include <string>

#include "dgmres/deflation.hpp"
#include "dgmres/gmres.hpp"
#include "pgmres.h"
#include "pgmres/pattern_hash.hpp"

namespace dgmres {

struct DeviceSolveAccess {
  static GmresWorkspace view(pgm_context* ctx, index_t n, std::uint32_t m, std::uint32_t steps) {
    return GmresWorkspace(ctx, n, m, steps);
  }
};

namespace {

void check(pgm_status s, const pgm_context* ctx) {
  if (s == PGM_OK) return;
  const std::string msg = pgm_last_error(ctx);
  if (s == PGM_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

std::uint64_t pattern_hash(const CsrMatrix& A) {
  return pgmres::detail::pattern_hash(A.row_ptr.data(), A.n, A.col_idx.data(), A.col_idx.size());
}

// ---- process-wide device runtime ---------------------------------------------
struct Runtime {
  int device = 0;
  std::map<index_t, pgm_context*> ctxs;
  struct Resident {
    pgm_context* ctx = nullptr;
    index_t n = 0;
    std::uint64_t nnz = 0, hash = 0;
    pgm_matrix* mat = nullptr;
  } cur;

  Runtime() {
    if (const char* e = std::getenv("PGMRES_DEVICE")) device = std::atoi(e);
  }
  // contexts and the resident matrix are released with the process (device
  // teardown at exit; Deflators may outlive this object in static storage)

  pgm_context* context(index_t n) {
    auto it = ctxs.find(n);
    if (it != ctxs.end()) return it->second;
    pgm_context_config cfg{device, 0, 1, nullptr, nullptr, 0, n, 1};
    pgm_context* c = nullptr;
    check(pgm_context_create(&cfg, &c), nullptr);
    ctxs[n] = c;
    return c;
  }

  pgm_matrix* matrix(const CsrMatrix& A) {
    if (A.row_ptr.size() != std::size_t(A.n) + 1)
      throw std::invalid_argument("CsrMatrix: row_ptr must have n + 1 entries");
    if (A.values.size() != A.col_idx.size())
      throw std::invalid_argument("CsrMatrix: values and col_idx differ in length");
    pgm_context* ctx = context(A.n);
    const std::uint64_t h = pattern_hash(A);
    if (cur.mat && cur.ctx == ctx && cur.n == A.n && cur.nnz == A.nnz() && cur.hash == h) {
      check(pgm_matrix_update_values(cur.mat, A.values.data(), 0), ctx);
      return cur.mat;
    }
    if (cur.mat) pgm_matrix_destroy(cur.mat);
    cur = Resident{};
    pgm_csr_view v{A.n, A.nnz(), A.row_ptr.data(), A.col_idx.data(), A.values.data()};
    pgm_matrix* m = nullptr;
    check(pgm_matrix_upload(ctx, &v, 0, &m), ctx);
    cur = Resident{ctx, A.n, A.nnz(), h, m};
    return m;
  }
};

Runtime& runtime() {
  static Runtime* r = new Runtime();  // never destroyed (see above)
  return *r;
}

// ---- device operators recognised by gmres_restarted / push_vector -------------
struct CsrOp {
  const CsrMatrix* A;
  void operator()(const DenseVector&, DenseVector&) const {
    throw std::invalid_argument(
        "csr_operator: the device operator is applied inside the GPU solve, not on the host");
  }
};

const CsrMatrix* csr_of(const LinearOp& op) {
  if (!op) return nullptr;
  const CsrOp* c = op.target<CsrOp>();
  return c ? c->A : nullptr;
}

struct ObserverState {
  const RestartHook* hook;
  pgm_context* ctx;
  index_t n;
  std::uint32_t m;
  std::exception_ptr err;
};

int32_t observer_trampoline(void* user, std::uint32_t restart, std::uint32_t steps) {
  auto* s = static_cast<ObserverState*>(user);
  try {
    const GmresWorkspace ws = DeviceSolveAccess::view(s->ctx, s->n, s->m, steps);
    (*s->hook)(RestartContext{ws, steps, restart});
    return 0;
  } catch (...) {
    s->err = std::current_exception();
    return 1;
  }
}

GmresReport solve(const CsrMatrix& A, const DenseVector& b, DenseVector& x,
                  const GmresConfig& cfg, Deflator* d, const RestartHook* hook) {
  if (cfg.m == 0) throw std::invalid_argument("GmresWorkspace: m must be positive");
  if (b.size() != A.n) throw std::invalid_argument("gmres: b does not match the matrix");
  if (x.size() != A.n) x.assign(A.n, 0.0);
  Runtime& R = runtime();
  pgm_matrix* M = R.matrix(A);
  pgm_context* ctx = R.context(A.n);
  pgm_deflator* dd = d ? d->bind(A.n) : nullptr;
  const pgm_gmres_config c{cfg.m, cfg.max_restarts, cfg.rel_tol, cfg.fixed_iterations ? 1 : 0,
                           cfg.breakdown_scale};
  ObserverState st{hook, ctx, A.n, cfg.m, nullptr};
  const bool observe = hook && *hook;
  if (observe) check(pgm_set_restart_observer(ctx, observer_trampoline, &st), ctx);
  pgm_report r{};
  const pgm_status s = pgm_solve(ctx, M, dd, b.data(), x.data(), &c, 0, &r);
  if (observe) pgm_set_restart_observer(ctx, nullptr, nullptr);
  if (st.err) {
    pgm_report_free(&r);
    std::rethrow_exception(st.err);
  }
  check(s, ctx);
  GmresReport out;
  out.beta0 = r.beta0;
  out.restarts = r.restarts;
  out.total_inner = r.total_inner;
  out.converged = r.converged != 0;
  out.breakdown = r.breakdown != 0;
  out.final_relative = r.final_relative;
  out.inner.reserve(r.n_inner);
  for (std::uint32_t i = 0; i < r.n_inner; ++i)
    out.inner.push_back({r.inner_restart[i], r.inner_step[i], r.inner_monitored[i]});
  out.explicit_residual.assign(r.explicit_residual, r.explicit_residual + r.restarts);
  pgm_report_free(&r);
  return out;
}

}  // namespace

// ---- gmres.hpp -----------------------------------------------------------------
void GmresReport::write_csv(std::ostream& os) const {  // gmres.cpp:117-130 schema
  os << "restart,inner_step,monitored_residual,explicit_residual\n";
  os.precision(17);
  for (std::size_t i = 0; i < inner.size(); ++i) {
    const InnerRecord& rec = inner[i];
    const bool last_of_cycle = i + 1 == inner.size() || inner[i + 1].restart != rec.restart;
    os << rec.restart << ',' << rec.inner << ',' << rec.monitored << ',';
    if (last_of_cycle && rec.restart < explicit_residual.size())
      os << explicit_residual[rec.restart];
    os << '\n';
  }
}

const DenseVector& GmresWorkspace::basis(std::uint32_t j) const {
  if (j >= steps_) throw std::out_of_range("GmresWorkspace::basis: j >= steps");
  if (v_.size() < steps_) v_.resize(steps_);
  if (v_[j].empty()) {
    v_[j].resize(n_);
    check(pgm_restart_basis(ctx_, j, v_[j].data()), ctx_);
  }
  return v_[j];
}

double GmresWorkspace::hess(std::uint32_t i, std::uint32_t j) const {
  if (j >= steps_ || i > j + 1) throw std::out_of_range("GmresWorkspace::hess: outside the cycle");
  if (h_.empty()) {
    h_.resize(std::size_t(m_ + 1) * m_);
    check(pgm_restart_hessenberg(ctx_, h_.data()), ctx_);
  }
  return h_[i + std::size_t(j) * (m_ + 1)];
}

LinearOp csr_operator(const CsrMatrix& A) { return LinearOp(CsrOp{&A}); }

GmresReport gmres_restarted(const LinearOp& opA, const LinearOp& opM, const DenseVector& b,
                            DenseVector& x, const GmresConfig& cfg, Executor& ex,
                            const RestartHook& hook) {
  const CsrMatrix* A = csr_of(opA);
  if (!A)
    throw std::invalid_argument(
        "gmres_restarted: the device path needs opA = csr_operator(A) (arbitrary operators "
        "stay on the reference)");
  if (opM)
    throw std::invalid_argument(
        "gmres_restarted: the device path takes no opM; use deflated_gmres for the "
        "deflation preconditioner");
  (void)ex;
  return solve(*A, b, x, cfg, nullptr, &hook);
}

GmresReport gmres_restarted(const CsrMatrix& A, std::nullptr_t, const DenseVector& b,
                            DenseVector& x, const GmresConfig& cfg, Executor& ex,
                            const RestartHook& hook) {
  (void)ex;
  return solve(A, b, x, cfg, nullptr, &hook);
}

// ---- deflation.hpp -------------------------------------------------------------
Deflator::Deflator(DeflationConfig cfg) : cfg_(cfg) {  // deflation.cpp:86-89 checks
  if (cfg_.r_max == 0) throw std::invalid_argument("deflation: r_max must be positive");
  if (cfg_.drop == 0) throw std::invalid_argument("deflation: drop must be positive");
}

Deflator::~Deflator() {
  if (d_) pgm_deflator_destroy(d_);
}

pgm_deflator* Deflator::bind(index_t n) {
  if (d_ && n != n_) {
    std::uint32_t r = 0;
    check(pgm_deflator_info(d_, &r, nullptr, nullptr, nullptr), nullptr);
    if (r != 0)
      throw std::invalid_argument("Deflator: the basis belongs to a problem of another size");
    pgm_deflator_destroy(d_);
    d_ = nullptr;
  }
  if (!d_) {
    pgm_context* ctx = runtime().context(n);
    const pgm_deflation_config c{cfg_.r_max, cfg_.drop, cfg_.accept_tol, cfg_.inv_power_maxit,
                                 cfg_.inv_power_tol, cfg_.power_maxit};
    check(pgm_deflator_create(ctx, &c, &d_), ctx);
    n_ = n;
  }
  return d_;
}

std::uint32_t Deflator::rank() const {
  std::uint32_t r = 0;
  if (d_) check(pgm_deflator_info(d_, &r, nullptr, nullptr, nullptr), nullptr);
  return r;
}

double Deflator::mu() const {
  double mu = 0.0;
  if (d_) check(pgm_deflator_info(d_, nullptr, &mu, nullptr, nullptr), nullptr);
  return mu;
}

std::uint32_t Deflator::skipped_updates() const {
  std::uint32_t s = 0;
  if (d_) check(pgm_deflator_info(d_, nullptr, nullptr, &s, nullptr), nullptr);
  return s;
}

void Deflator::reset() {
  if (d_) check(pgm_deflator_reset(d_), nullptr);
  history_.clear();
}

void Deflator::apply(const DenseVector& v, DenseVector& w, Executor& ex) const {
  (void)ex;
  w.resize(v.size());
  if (!d_) {  // identity while the basis is empty (deflation.cpp:105-106)
    std::copy(v.begin(), v.end(), w.begin());
    return;
  }
  if (v.size() != n_) throw std::invalid_argument("Deflator::apply: size mismatch");
  check(pgm_deflator_apply(d_, v.data(), w.data(), 0), nullptr);
}

bool Deflator::update_from_restart(const RestartContext&, const LinearOp&, Executor&) {
  throw std::invalid_argument(
      "Deflator::update_from_restart: the device solve harvests restarts itself "
      "(deflated_gmres)");
}

bool Deflator::push_vector(const DenseVector& candidate, const LinearOp& opA, Executor& ex) {
  const CsrMatrix* A = csr_of(opA);
  if (!A) throw std::invalid_argument("Deflator::push_vector: opA must be csr_operator(A)");
  return push_vector(candidate, *A, ex);
}

bool Deflator::push_vector(const DenseVector& candidate, const CsrMatrix& A, Executor& ex) {
  (void)ex;
  if (candidate.size() != A.n) throw std::invalid_argument("Deflator::push_vector: size mismatch");
  pgm_matrix* M = runtime().matrix(A);
  pgm_deflator* d = bind(A.n);
  int32_t ok = 0;
  check(pgm_deflator_push(d, M, candidate.data(), 0, &ok), nullptr);
  return ok != 0;
}

void Deflator::observe_ritz(double value) {
  if (!d_) {
    throw std::invalid_argument(
        "Deflator::observe_ritz: the deflator has no device state yet (solve or push first)");
  }
  check(pgm_deflator_observe_ritz(d_, value), nullptr);
}

void Deflator::truncate() {
  if (d_) check(pgm_deflator_truncate(d_), nullptr);
}

const std::vector<DeflationRecord>& Deflator::history() const {
  history_.clear();
  std::uint32_t nh = 0;
  if (d_) check(pgm_deflator_info(d_, nullptr, nullptr, nullptr, &nh), nullptr);
  if (nh) {
    std::vector<pgm_deflation_record> raw(nh);
    check(pgm_deflator_history(d_, raw.data(), nh), nullptr);
    for (const auto& r : raw) history_.push_back({r.restart, r.r, r.mu, r.smallest_ritz});
  }
  return history_;
}

void Deflator::write_csv(std::ostream& os) const {  // deflation.cpp:266-273 schema
  os << "restart,r,mu,smallest_ritz\n";
  os.precision(17);
  for (const auto& rec : history())
    os << rec.restart << ',' << rec.r << ',' << rec.mu << ',' << rec.smallest_ritz << '\n';
}

DenseBlock Deflator::T_block() const {
  DenseBlock out;
  const std::uint32_t r = rank();
  out.rows = out.cols = r;
  out.data.assign(std::size_t(r) * r, 0.0);
  if (r) check(pgm_deflator_basis(d_, nullptr, out.data.data()), nullptr);
  return out;
}

DenseBlock Deflator::basis_matrix() const {
  DenseBlock out;
  const std::uint32_t r = rank();
  out.rows = n_;
  out.cols = r;
  out.data.assign(std::size_t(n_) * r, 0.0);
  if (r) check(pgm_deflator_basis(d_, out.data.data(), nullptr), nullptr);
  return out;
}

RestartHook deflation_hook(Deflator&, LinearOp, Executor&) {
  throw std::invalid_argument(
      "deflation_hook: the device solve harvests restarts itself (deflated_gmres)");
}

GmresReport deflated_gmres(const CsrMatrix& A, const DenseVector& b, DenseVector& x,
                           const GmresConfig& cfg, Deflator& d, Executor& ex) {
  (void)ex;
  return solve(A, b, x, cfg, &d, nullptr);
}

GmresReport deflated_gmres(const CsrMatrix& A, const DenseVector& b, DenseVector& x,
                           const GmresConfig& cfg, Deflator& d, Executor& ex,
                           const RestartHook& observer) {
  (void)ex;
  return solve(A, b, x, cfg, &d, &observer);
}

}  // namespace dgmres
