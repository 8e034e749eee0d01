/*
 * metrics_impl.h — Eigen-free restatement of proj/src/metrics.cpp:19-41
 * (TEST INFRASTRUCTURE ONLY).  Shared by the C oracle (oracle.c) and the
 * metrics shim that lets the reference sources build without Eigen
 * (metrics_shim.cpp).  Diagnostics only: the reference's own metrics use
 * Eigen's SelfAdjointEigenSolver / JacobiSVD, which are absent here; values
 * agree to rounding, not bitwise.
 */
#ifndef BO_METRICS_IMPL_H
#define BO_METRICS_IMPL_H

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* cyclic Jacobi eigenvalues of a symmetric k x k matrix (destroys a) */
static void mi_sym_eigenvalues(double* a, size_t k, double* ev) {
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (size_t j = 0; j < k; ++j)
      for (size_t i = 0; i < j; ++i) off += a[i + j * k] * a[i + j * k];
    if (off == 0.0) break;
    for (size_t p = 0; p < k; ++p)
      for (size_t q = p + 1; q < k; ++q) {
        const double apq = a[p + q * k];
        if (apq == 0.0) continue;
        const double app = a[p + p * k], aqq = a[q + q * k];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (size_t r = 0; r < k; ++r) {
          const double arp = a[r + p * k], arq = a[r + q * k];
          a[r + p * k] = c * arp - s * arq;
          a[r + q * k] = s * arp + c * arq;
        }
        for (size_t r = 0; r < k; ++r) {
          const double apr = a[p + r * k], aqr = a[q + r * k];
          a[p + r * k] = c * apr - s * aqr;
          a[q + r * k] = s * apr + c * aqr;
        }
      }
  }
  for (size_t i = 0; i < k; ++i) ev[i] = a[i + i * k];
}

static int mi_cmp_desc(const void* x, const void* y) {
  const double a = *(const double*)x, b = *(const double*)y;
  return (a < b) - (a > b);
}

/* singular values, descending, count min(rows, cols); one-sided Jacobi */
static void mi_singular_values(const double* m, size_t rows, size_t cols, double* sv) {
  size_t r = rows, c = cols;
  double* a = (double*)malloc((rows * cols ? rows * cols : 1) * sizeof(double));
  if (rows >= cols) {
    memcpy(a, m, rows * cols * sizeof(double));
  } else {
    for (size_t j = 0; j < cols; ++j)
      for (size_t i = 0; i < rows; ++i) a[j + i * cols] = m[i + j * rows];
    r = cols;
    c = rows;
  }
  for (int sweep = 0; sweep < 80; ++sweep) {
    int rotated = 0;
    for (size_t p = 0; p < c; ++p)
      for (size_t q = p + 1; q < c; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        for (size_t i = 0; i < r; ++i) {
          alpha += a[i + p * r] * a[i + p * r];
          beta += a[i + q * r] * a[i + q * r];
          gamma += a[i + p * r] * a[i + q * r];
        }
        if (gamma == 0.0 || fabs(gamma) <= 2.3e-16 * sqrt(alpha * beta)) continue;
        rotated = 1;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (size_t i = 0; i < r; ++i) {
          const double x = a[i + p * r], y = a[i + q * r];
          a[i + p * r] = cs * x - sn * y;
          a[i + q * r] = sn * x + cs * y;
        }
      }
    if (!rotated) break;
  }
  for (size_t j = 0; j < c; ++j) {
    double s = 0;
    for (size_t i = 0; i < r; ++i) s += a[i + j * r] * a[i + j * r];
    sv[j] = sqrt(s);
  }
  qsort(sv, c, sizeof(double), mi_cmp_desc);
  free(a);
}

#endif
