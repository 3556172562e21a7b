#include <algorithm>
// C++ drop-in check: the reference's call sequence (newton.cpp:53-63 for the
// first Newton system) written against include/pgmres/dgmres.hpp.  Prints one
// line "restarts total_inner rank final_relative mu x_norm" for the pytest
// harness (tests/test_gpu_dropin.py) and exercises the reference's exception
// types.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <stdexcept>

#include "pgmres/dgmres.hpp"

int main(int argc, char** argv) {
  const unsigned ne = argc > 1 ? std::atoi(argv[1]) : 10;
  const unsigned m = argc > 2 ? std::atoi(argv[2]) : 30;
  const unsigned na = 2 * ne + 1;
  pgmres::DeviceExecutor ex(0);
  pgm_context* ctx = ex.context(na * na * na);
  std::uint64_t nnz = 0;
  pgm_bratu_nnz(ctx, ne, &nnz);
  pgmres::CsrMatrix J;
  J.n = na * na * na;
  J.row_ptr.resize(J.n + 1);
  J.col_idx.resize(nnz);
  J.values.resize(nnz);
  pgmres::DenseVector rhs(J.n), delta(J.n, 0.0);
  if (pgm_bratu_assemble(ctx, ne, 6.8, nullptr, 0, J.row_ptr.data(), J.col_idx.data(),
                         J.values.data(), rhs.data()) != PGM_OK) {
    std::fprintf(stderr, "assembly failed: %s\n", pgm_last_error(ctx));
    return 2;
  }
  pgmres::GmresConfig cfg;
  cfg.m = m;
  cfg.max_restarts = 100;
  cfg.rel_tol = 1e-10;
  pgmres::Deflator deflator;
  deflator.reset();
  const pgmres::GmresReport rep = pgmres::deflated_gmres(J, rhs, delta, cfg, deflator, ex);
  double xn = 0.0;
  for (double v : delta) xn += v * v;
  std::printf("%u %llu %u %.17g %.17g %.17g\n", rep.restarts,
              (unsigned long long)rep.total_inner, deflator.rank(), rep.final_relative,
              deflator.mu(), std::sqrt(xn));
  std::ostringstream csv;
  rep.write_csv(csv);
  if (csv.str().rfind("restart,inner_step,monitored_residual,explicit_residual\n", 0) != 0)
    return 3;
  // std::invalid_argument for m = 0 (gmres.cpp:10)
  bool threw = false;
  try {
    pgmres::GmresConfig bad;
    bad.m = 0;
    pgmres::gmres_restarted(J, nullptr, rhs, delta, bad, ex);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  if (!threw) return 4;
  // std::runtime_error for a non-finite operator (gmres.cpp:151-153)
  pgmres::CsrMatrix nanA = J;
  nanA.values[0] = std::nan("");
  threw = false;
  try {
    pgmres::DeviceExecutor ex2(0);
    pgmres::DenseVector x2(J.n, 0.0);
    pgmres::gmres_restarted(nanA, nullptr, rhs, x2, pgmres::GmresConfig{}, ex2);
  } catch (const std::runtime_error& e) {
    threw = std::string(e.what()).find("gmres: ") == 0;
  }
  if (!threw) return 5;
  // newton_solve (newton.hpp:53-54) on the n_e = 8 system: the reference converges
  // in 8 iterations to max u = 1.323002464567 (test_output.txt, criterion 7)
  {
    pgmres::DeviceExecutor exn(0);
    pgmres::DenseVector u;
    auto nr = pgmres::newton_solve(8, 6.8, u, pgmres::NewtonConfig{}, exn);
    double umax = 0.0;
    for (double v : u) umax = std::max(umax, v);
    std::fprintf(stderr, "newton %zu iterations, max u %.12f\n", nr.iters.size(), umax);
    if (!nr.converged || nr.iters.size() != 8 || std::fabs(umax - 1.323002464567) > 1e-11)
      return 6;
  }
  return 0;
}
