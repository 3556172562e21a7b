// compat/dgmres/deflation.hpp — source-compatible stand-in for the reference's
// dgmres/deflation.hpp (/root/reference/proj/include/dgmres/deflation.hpp:1-100)
// backed by libpgmres: the Deflator's U, AU, T, T^-1 and history live on the
// GPU across solves (pgm_deflator_*), deflated_gmres runs the whole solve —
// Arnoldi, deflation apply, restart harvest, truncation — on the device.
//
// Same as the reference: DeflationConfig (:15-22), DeflationRecord (:24-29),
// Deflator's constructor checks and messages, rank / mu / skipped_updates /
// reset / apply / observe_ritz / truncate / history / write_csv, and
// deflated_gmres's signature (:97-98), so src/newton.cpp:60-64 compiles and
// runs unchanged.
// Different, by design:
//   * T_block() / basis_matrix() return DenseBlock (column-major, no Eigen);
//   * update_from_restart / deflation_hook are not callable on the host: the
//     device solve runs the harvest itself (deflated_gmres); audits attach a
//     RestartHook with the deflated_gmres overload below;
//   * push_vector needs the CSR operator (csr_operator(A) or the CsrMatrix
//     overload).
#pragma once

#include <cstdint>
#include <iosfwd>
#include <vector>

#include "dgmres/gmres.hpp"
#include "dgmres/parallel.hpp"
#include "dgmres/sparse.hpp"

struct pgm_deflator;

namespace dgmres {

struct DeflationConfig {
  std::uint32_t r_max = 20;  // basis size cap; exceeding it triggers truncation
  std::uint32_t drop = 1;    // directions removed per truncation
  double accept_tol = 1e-8;  // candidate norm after orthogonalization
  std::uint32_t inv_power_maxit = 500;
  double inv_power_tol = 1e-10;
  std::uint32_t power_maxit = 200;
};

struct DeflationRecord {
  std::uint32_t restart;
  std::uint32_t r;
  double mu;
  double smallest_ritz;
};

/// Column-major dense block (rows x cols) returned by the introspection calls.
struct DenseBlock {
  std::uint32_t rows = 0, cols = 0;
  std::vector<double> data;
  double operator()(std::uint32_t i, std::uint32_t j) const { return data[i + std::size_t(j) * rows]; }
};

class Deflator {
 public:
  explicit Deflator(DeflationConfig cfg = {});
  ~Deflator();
  Deflator(const Deflator&) = delete;
  Deflator& operator=(const Deflator&) = delete;

  std::uint32_t rank() const;
  double mu() const;
  std::uint32_t skipped_updates() const;
  void reset();
  /// w = v + U (|mu| T^{-1} - I) U^T v; identity while the basis is empty.
  void apply(const DenseVector& v, DenseVector& w, Executor& ex) const;
  /// Host-side harvest is not available (the device solve harvests).
  bool update_from_restart(const RestartContext& ctx, const LinearOp& opA, Executor& ex);
  /// Append a candidate (orthonormalised against U first) with opA the CSR
  /// operator (csr_operator(A)).
  bool push_vector(const DenseVector& candidate, const LinearOp& opA, Executor& ex);
  bool push_vector(const DenseVector& candidate, const CsrMatrix& A, Executor& ex);
  void observe_ritz(double value);
  void truncate();
  const std::vector<DeflationRecord>& history() const;
  /// restart,r,mu,smallest_ritz
  void write_csv(std::ostream& os) const;
  /// Active r x r block of T.
  DenseBlock T_block() const;
  /// Active n x r block of U.
  DenseBlock basis_matrix() const;

  // device binding (used by the solve entry points)
  pgm_deflator* bind(index_t n);

 private:
  DeflationConfig cfg_;
  pgm_deflator* d_ = nullptr;
  index_t n_ = 0;
  mutable std::vector<DeflationRecord> history_;
};

/// Not available on the device path (throws std::invalid_argument): the
/// harvest runs inside deflated_gmres.
RestartHook deflation_hook(Deflator& d, LinearOp opA, Executor& ex);

/// Deflated GMRES on a CSR matrix (deflation.hpp:94-98), on the GPU.
GmresReport deflated_gmres(const CsrMatrix& A, const DenseVector& b, DenseVector& x,
                           const GmresConfig& cfg, Deflator& d, Executor& ex);

/// Same, with a restart observer called after every cycle's x update and
/// deflation harvest (the criterion-8 audit of acceptance.cpp:100-122).
GmresReport deflated_gmres(const CsrMatrix& A, const DenseVector& b, DenseVector& x,
                           const GmresConfig& cfg, Deflator& d, Executor& ex,
                           const RestartHook& observer);

}  // namespace dgmres
