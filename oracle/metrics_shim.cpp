// metrics_shim.cpp — Eigen-free replacement for proj/src/metrics.cpp so the
// reference sources compile into oracle/_ref without Eigen (absent in this
// image).  TEST INFRASTRUCTURE ONLY.  Restates proj/src/metrics.cpp:19-41;
// only diagnostics (orthogonality error, condition numbers) depend on it.
#include <cmath>
#include <limits>
#include <vector>

#include "blkorth/errors.hpp"
#include "blkorth/metrics.hpp"

extern "C" {
#include "metrics_impl.h"
}

namespace blkorth {

double orthogonality_error(const DenseMatrix& q) {  // metrics.cpp:19-27
  if (q.empty()) return 0.0;
  const std::size_t k = q.cols();
  DenseMatrix d = transpose_times(q, q);
  for (std::size_t j = 0; j < k; ++j)
    for (std::size_t i = 0; i < k; ++i) d(i, j) = (i == j ? 1.0 : 0.0) - d(i, j);
  std::vector<double> ev(k);
  mi_sym_eigenvalues(d.data(), k, ev.data());
  double m = 0.0;
  for (double e : ev) m = std::max(m, std::abs(e));
  return m;
}

std::vector<double> singular_values(const DenseMatrix& m) {  // metrics.cpp:29-33
  std::vector<double> sv(std::min(m.rows(), m.cols()));
  if (!sv.empty()) mi_singular_values(m.data(), m.rows(), m.cols(), sv.data());
  return sv;
}

double condition_number(const DenseMatrix& v) {  // metrics.cpp:35-41
  const auto sv = singular_values(v);
  if (sv.empty() || sv.front() == 0.0) throw ZeroMatrix();
  const double smin = sv.back();
  if (smin == 0.0) return std::numeric_limits<double>::infinity();
  return sv.front() / smin;
}

}  // namespace blkorth
