// bo_hostdense.h — the small (non-tall) dense algebra that the reference runs
// redundantly on every process: Householder QR of sketched blocks, block CGS
// on the sketched history, coefficient updates (proj/src/dense.cpp,
// proj/src/block_orth.cpp:271-325).  These operate on m-hat x (<= 64) or
// (<= 64) x (<= 64) matrices on the host; identical element-level order to the
// reference.  Tall work never runs here.
#pragma once
#include <cmath>
#include <cstddef>
#include <vector>

namespace bo {
namespace hd {

struct Mat {
  size_t r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(size_t rr, size_t cc) : r(rr), c(cc), a(rr * cc, 0.0) {}
  double& operator()(size_t i, size_t j) { return a[i + j * r]; }
  double operator()(size_t i, size_t j) const { return a[i + j * r]; }
};

// dense.cpp:28-42
inline Mat transpose_times(const Mat& A, const Mat& B) {
  Mat C(A.c, B.c);
  for (size_t j = 0; j < B.c; ++j)
    for (size_t i = 0; i < A.c; ++i) {
      double s = 0.0;
      for (size_t r = 0; r < A.r; ++r) s += A(r, i) * B(r, j);
      C(i, j) = s;
    }
  return C;
}
// dense.cpp:60-73  B -= Q C
inline void subtract_product(Mat& B, const Mat& Q, const Mat& C) {
  for (size_t j = 0; j < B.c; ++j)
    for (size_t k = 0; k < Q.c; ++k) {
      const double ckj = C(k, j);
      if (ckj == 0.0) continue;
      for (size_t r = 0; r < B.r; ++r) B(r, j) -= Q(r, k) * ckj;
    }
}
// dense.cpp:44-58
inline Mat times(const Mat& A, const Mat& B) {
  Mat C(A.r, B.c);
  for (size_t j = 0; j < B.c; ++j)
    for (size_t k = 0; k < A.c; ++k) {
      const double bkj = B(k, j);
      if (bkj == 0.0) continue;
      for (size_t r = 0; r < A.r; ++r) C(r, j) += A(r, k) * bkj;
    }
  return C;
}
// dense.cpp:188-198 (upper T R)
inline Mat multiply_upper(const Mat& T, const Mat& R) {
  const size_t k = T.r;
  Mat O(k, k);
  for (size_t i = 0; i < k; ++i)
    for (size_t j = i; j < k; ++j) {
      double s = 0.0;
      for (size_t l = i; l <= j; ++l) s += T(i, l) * R(l, j);
      O(i, j) = s;
    }
  return O;
}
// block_orth.cpp:191-203
inline Mat update_projection(const Mat& proj, const Mat& t, const Mat& rdiag) {
  Mat tmp = times(t, rdiag);
  Mat out = proj;
  for (size_t j = 0; j < out.c; ++j)
    for (size_t i = 0; i < out.r; ++i) out(i, j) += tmp(i, j);
  return out;
}
// dense.cpp:75-102; returns failed_at (0 ok), R upper k x k
inline size_t cholesky(const Mat& G, Mat& R, double tol, double* failed_pivot) {
  const size_t k = G.r;
  R = Mat(k, k);
  double max_diag = 0.0;
  for (size_t i = 0; i < k; ++i) max_diag = max_diag < G(i, i) ? G(i, i) : max_diag;
  const double floor_ = tol * max_diag;
  for (size_t j = 0; j < k; ++j) {
    for (size_t i = 0; i < j; ++i) {
      double s = G(i, j);
      for (size_t t = 0; t < i; ++t) s -= R(t, i) * R(t, j);
      R(i, j) = s / R(i, i);
    }
    double piv = G(j, j);
    for (size_t t = 0; t < j; ++t) piv -= R(t, j) * R(t, j);
    if (piv <= floor_) {
      if (failed_pivot) *failed_pivot = piv;
      return j + 1;
    }
    R(j, j) = std::sqrt(piv);
  }
  return 0;
}
// dense.cpp:104-164 thin Householder QR, sign-normalised
inline void householder_qr(const Mat& V, Mat& Q, Mat& R) {
  const size_t n = V.r, k = V.c;
  Mat a = V, w(n, k);
  std::vector<double> tau(k, 0.0);
  for (size_t j = 0; j < k; ++j) {
    double norm2 = 0.0;
    for (size_t i = j; i < n; ++i) norm2 += a(i, j) * a(i, j);
    const double norm = std::sqrt(norm2);
    if (norm == 0.0) {
      tau[j] = 0.0;
      continue;
    }
    const double alpha = a(j, j) >= 0.0 ? -norm : norm;
    const double v0 = a(j, j) - alpha;
    w(j, j) = 1.0;
    for (size_t i = j + 1; i < n; ++i) w(i, j) = a(i, j) / v0;
    tau[j] = -v0 / alpha;
    a(j, j) = alpha;
    for (size_t i = j + 1; i < n; ++i) a(i, j) = 0.0;
    for (size_t c = j + 1; c < k; ++c) {
      double s = a(j, c);
      for (size_t i = j + 1; i < n; ++i) s += w(i, j) * a(i, c);
      s *= tau[j];
      a(j, c) -= s;
      for (size_t i = j + 1; i < n; ++i) a(i, c) -= s * w(i, j);
    }
  }
  Q = Mat(n, k);
  for (size_t j = 0; j < k; ++j) Q(j, j) = 1.0;
  for (size_t jj = k; jj-- > 0;) {
    if (tau[jj] == 0.0) continue;
    for (size_t c = jj; c < k; ++c) {
      double s = Q(jj, c);
      for (size_t i = jj + 1; i < n; ++i) s += w(i, jj) * Q(i, c);
      s *= tau[jj];
      Q(jj, c) -= s;
      for (size_t i = jj + 1; i < n; ++i) Q(i, c) -= s * w(i, jj);
    }
  }
  R = Mat(k, k);
  for (size_t i = 0; i < k; ++i) {
    const double flip = a(i, i) < 0.0 ? -1.0 : 1.0;
    for (size_t j = i; j < k; ++j) R(i, j) = flip * a(i, j);
    if (flip < 0.0)
      for (size_t r = 0; r < n; ++r) Q(r, i) = -Q(r, i);
  }
}

}  // namespace hd
}  // namespace bo
