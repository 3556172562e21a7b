// Host build of paper_1906_04051_b200/csrc/dense.cuh for CPU unit tests
// (tests/test_dense.py): the same single-thread routines the device runs.
#include <vector>
#include "../paper_1906_04051_b200/csrc/dense.cuh"
extern "C" {
int h_dominant_eigvec(const double* T, int n, double* v) {
  std::vector<double> work(4 * n * n + 6 * n + 8 * n * n);
  std::vector<int> iw(2 * n);
  return pgm::dense::dominant_eigvec(T, n, n, v, work.data(), iw.data());
}
int h_eigvals(const double* T, int n, double* wr, double* wi) {
  std::vector<double> h(T, T + n * n), z(2 * n * n + n);
  pgm::dense::hessenberg_reduce(h.data(), n, n);
  return pgm::dense::hessenberg_eigvals(h.data(), n, n, wr, wi, z.data()) ? 0 : 1;
}
void h_invert(const double* A, int n, double* inv) {
  std::vector<double> a(A, A + n * n), w(n);
  std::vector<int> p(n);
  pgm::dense::invert(a.data(), n, n, inv, n, p.data(), w.data());
}
}
