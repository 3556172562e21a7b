// compat/dgmres/gmres.hpp — source-compatible stand-in for the reference's
// dgmres/gmres.hpp (/root/reference/proj/include/dgmres/gmres.hpp:1-113),
// backed by libpgmres (include/pgmres.h).  Put include/compat BEFORE the
// reference's include directory and link paper_1906_04051_b200/compat/
// dgmres_device.cpp + -lpgmres instead of src/gmres.cpp and src/deflation.cpp:
// the reference's callers (src/newton.cpp, tools/bratu_bench.cpp) then compile
// unchanged and their linear solves run on the GPU.
//
// Same as the reference (field for field):
//   LinearOp (gmres.hpp:15), GmresConfig (:17-23), InnerRecord (:25-29),
//   GmresReport + write_csv (:31-44), RestartContext (:94-98), RestartHook
//   (:103), gmres_restarted's signature (:110-113).
// Different, by design (there is no CPU fallback on the device path):
//   * gmres_restarted runs on the device when opA comes from csr_operator(A)
//     (the production operator: CSR SpMV) and opM is empty; any other
//     std::function operator throws std::invalid_argument.  deflated_gmres
//     (deflation.hpp) is the production entry point and needs no wrapping.
//   * GmresWorkspace is the restart-time view a RestartHook receives:
//     basis(j) and hess(i, j) of the finished cycle, read from the device
//     (pgm_restart_basis / pgm_restart_hessenberg); the step-wise API
//     (begin_cycle, arnoldi_step, ...) is not exported.
#pragma once

#include <cstdint>
#include <functional>
#include <iosfwd>
#include <span>
#include <vector>

#include "dgmres/parallel.hpp"
#include "dgmres/sparse.hpp"

struct pgm_context;

namespace dgmres {

/// y = Op(x); x and y are distinct, sized n.
using LinearOp = std::function<void(const DenseVector&, DenseVector&)>;

struct GmresConfig {
  std::uint32_t m = 50;             // Krylov dimension per cycle
  std::uint32_t max_restarts = 100;
  double rel_tol = 1e-8;            // on ||b - Ax|| / ||b - Ax0||
  bool fixed_iterations = false;    // benchmark mode: run every restart, no test
  double breakdown_scale = 1e-14;   // h_{k+1,k} < scale * beta ends the cycle
};

struct InnerRecord {
  std::uint32_t restart;
  std::uint32_t inner;
  double monitored;  // |gamma_{k+1}| from the rotated least-squares rhs
};

struct GmresReport {
  double beta0 = 0.0;                     // ||b - A x0||
  std::vector<InnerRecord> inner;
  std::vector<double> explicit_residual;  // recomputed ||b - Ax|| per restart
  std::uint32_t restarts = 0;
  std::uint64_t total_inner = 0;
  bool converged = false;
  bool breakdown = false;                 // cycle ended on a tiny h (lucky)
  double final_relative = 0.0;

  /// restart,inner_step,monitored_residual,explicit_residual
  void write_csv(std::ostream& os) const;
};

/// The finished restart cycle as a RestartHook sees it (device data, read on
/// demand while the hook runs).
class GmresWorkspace {
 public:
  index_t n() const { return n_; }
  std::uint32_t m() const { return m_; }
  /// v_j of the cycle (j < steps).
  const DenseVector& basis(std::uint32_t j) const;
  /// Unrotated Hessenberg entry, i <= j+1, j < steps.
  double hess(std::uint32_t i, std::uint32_t j) const;

 private:
  friend struct DeviceSolveAccess;
  GmresWorkspace(pgm_context* ctx, index_t n, std::uint32_t m, std::uint32_t steps)
      : ctx_(ctx), n_(n), m_(m), steps_(steps) {}
  pgm_context* ctx_;
  index_t n_;
  std::uint32_t m_, steps_;
  mutable std::vector<DenseVector> v_;
  mutable std::vector<double> h_;
};

struct RestartContext {
  const GmresWorkspace& ws;
  std::uint32_t steps;    // Arnoldi steps completed this cycle
  std::uint32_t restart;  // 0-based cycle index
};

/// Called at the end of each restart cycle, after the iterate update and
/// before the basis is discarded.
using RestartHook = std::function<void(const RestartContext&)>;

/// The device operator for gmres_restarted / Deflator::push_vector: y = A x.
/// (Calling it on the host is not supported: it exists to be recognised.)
LinearOp csr_operator(const CsrMatrix& A);

/// Restarted GMRES (gmres.hpp:105-113).  Runs on the GPU for opA =
/// csr_operator(A) and an empty opM; throws std::invalid_argument otherwise.
GmresReport gmres_restarted(const LinearOp& opA, const LinearOp& opM,
                            const DenseVector& b, DenseVector& x,
                            const GmresConfig& cfg, Executor& ex,
                            const RestartHook& hook = {});

/// Device-path overload for the production pair (CSR operator, no
/// preconditioner).
GmresReport gmres_restarted(const CsrMatrix& A, std::nullptr_t, const DenseVector& b,
                            DenseVector& x, const GmresConfig& cfg, Executor& ex,
                            const RestartHook& hook = {});

}  // namespace dgmres
