// bo_tiny.cuh — the small factorizations of the block-orthogonalization path,
// run by one CTA on device right after the reduction of a streaming pass
// (redundantly on every GPU of a row-sharded run, as the paper does on CPU,
// PAPER.md:558,1056).  Every routine reproduces the reference element-level
// order with explicit non-fused operations, so for identical inputs the
// results are bit-identical to proj/src/dense.cpp.
#pragma once
#include "bo_common.cuh"

namespace bo {
namespace tiny {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }

// Cholesky R^T R = G (proj/src/dense.cpp:75-102).  The reference is
// up-looking; this right-looking schedule performs, for every entry, the same
// subtractions in the same order (t = 0, 1, ...), so it is bit-identical.
// On failure at 1-based step f the partial factor matches the reference:
// columns < f-1 complete, column f-1 holds rows < f-1, later columns zero.
// Whole CTA participates (blockDim >= 32).  G, R have ld kRld; sbuf: 16*16.
__device__ inline void cholesky(const double* G, int K, double tol, double* R, double* sbuf,
                         int* failed_at, double* failed_pivot) {
  const int tid = threadIdx.x, nth = blockDim.x;
  __shared__ double s_maxdiag;
  __shared__ int s_fail;
  __shared__ double s_piv;
  for (int e = tid; e < kRld * kRld; e += nth) {
    sbuf[e] = G[e];
    R[e] = 0.0;
  }
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < K; ++i) {
      const double d = G[i + i * kRld];
      m = m < d ? d : m;  // std::max(max_diag, d)
    }
    s_maxdiag = m;
    s_fail = 0;
    s_piv = 0.0;
  }
  __syncthreads();
  const double floor_ = mul(tol, s_maxdiag);
  for (int t = 0; t < K; ++t) {
    if (tid == 0) {
      const double piv = sbuf[t + t * kRld];
      if (piv <= floor_) {
        s_fail = t + 1;
        s_piv = piv;
      } else {
        R[t + t * kRld] = sqrt(piv);
      }
    }
    __syncthreads();
    if (s_fail) {
      // reference leaves row < t entries of column t (already in R) and zero beyond
      break;
    }
    for (int j = t + 1 + tid; j < K; j += nth) R[t + j * kRld] = div(sbuf[t + j * kRld], R[t + t * kRld]);
    __syncthreads();
    // trailing update s_ij -= r_ti r_tj for t < i <= j
    const int m = K - t - 1;
    for (int e = tid; e < m * m; e += nth) {
      const int i = t + 1 + e % m, j = t + 1 + e / m;
      if (i <= j) sbuf[i + j * kRld] = sub(sbuf[i + j * kRld], mul(R[t + i * kRld], R[t + j * kRld]));
    }
    __syncthreads();
  }
  if (tid == 0) {
    *failed_at = s_fail;
    *failed_pivot = s_piv;
  }
  __syncthreads();
  if (s_fail) {
    // The reference computes column f-1's off-diagonal entries r_i,f-1 (i < f-1)
    // before testing its pivot: they equal s_i,f-1 / r_ii at step i, which the
    // right-looking loop already stored in R.  Columns >= f stay zero in the
    // reference; here rows t < f-1 of columns >= f were filled: clear them.
    const int f = s_fail;
    for (int e = tid; e < kRld * kRld; e += nth) {
      const int i = e % kRld, j = e / kRld;
      if (j >= f) R[i + j * kRld] = 0.0;
    }
  }
  __syncthreads();
}

// R factor of the thin Householder QR (proj/src/dense.cpp:104-164), sign
// normalised.  Q is not formed (RandCholQR uses only R,
// proj/src/intra_orth.cpp:28-39).  A (m x K, ld lda) is destroyed.  Warp 0
// only; lanes own columns.
__device__ inline void householder_r(double* A, int lda, int m, int K, double* R, double* tau_buf) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  for (int j = 0; j < K; ++j) {
    double norm = 0.0, alpha = 0.0, v0 = 0.0, tau = 0.0;
    if (lane == 0) {
      double norm2 = 0.0;
      for (int i = j; i < m; ++i) norm2 = add(norm2, mul(A[i + j * lda], A[i + j * lda]));
      norm = sqrt(norm2);
    }
    norm = __shfl_sync(0xffffffffu, norm, 0);
    if (norm == 0.0) {
      if (lane == 0) tau_buf[j] = 0.0;
      __syncwarp();
      continue;
    }
    const double ajj = A[j + j * lda];
    alpha = ajj >= 0.0 ? -norm : norm;
    v0 = sub(ajj, alpha);
    tau = div(-v0, alpha);
    __syncwarp();
    // w(i,j) = a(i,j) / v0 stored in A's lower part (a(i,j) is zeroed in the reference)
    for (int i = j + 1 + lane; i < m; i += 32) A[i + j * lda] = div(A[i + j * lda], v0);
    __syncwarp();
    for (int c = j + 1 + lane; c < K; c += 32) {
      double s = A[j + c * lda];
      for (int i = j + 1; i < m; ++i) s = add(s, mul(A[i + j * lda], A[i + c * lda]));
      s = mul(s, tau);
      A[j + c * lda] = sub(A[j + c * lda], s);
      for (int i = j + 1; i < m; ++i) A[i + c * lda] = sub(A[i + c * lda], mul(s, A[i + j * lda]));
    }
    __syncwarp();
    if (lane == 0) {
      A[j + j * lda] = alpha;
      tau_buf[j] = tau;
    }
    __syncwarp();
  }
  // sign-normalise rows
  for (int e = lane; e < kRld * kRld; e += 32) {
    const int i = e % kRld, jj = e / kRld;
    double v = 0.0;
    if (i < K && jj < K && jj >= i) {
      const double flip = A[i + i * lda] < 0.0 ? -1.0 : 1.0;
      v = mul(flip, A[i + jj * lda]);
    }
    R[e] = v;
  }
  __syncwarp();
}

// out = T * R for upper-triangular T, R (proj/src/dense.cpp:188-198)
__device__ inline void multiply_upper(const double* T, const double* Rm, int K, double* out) {
  for (int e = threadIdx.x; e < kRld * kRld; e += blockDim.x) {
    const int i = e % kRld, j = e / kRld;
    double s = 0.0;
    if (i < K && j < K && j >= i)
      for (int l = i; l <= j; ++l) s = add(s, mul(T[i + l * kRld], Rm[l + j * kRld]));
    out[e] = s;
  }
}

// out = C1 + C2 * Rin  (proj/src/block_orth.cpp:191-203 update_projection,
// times() at proj/src/dense.cpp:44-58 skips zero coefficients)
__device__ inline void update_projection(const double* C1, const double* C2, int ldc, int p, int K,
                                  const double* Rin, double* out) {
  for (int e = threadIdx.x; e < p * K; e += blockDim.x) {
    const int r = e % p, j = e / p;
    double acc = 0.0;
    for (int k = 0; k < K; ++k) {
      const double bkj = Rin[k + j * kRld];
      if (bkj == 0.0) continue;
      acc = add(acc, mul(C2[r + k * ldc], bkj));
    }
    out[r + j * ldc] = add(C1[r + j * ldc], acc);
  }
}

}  // namespace tiny
}  // namespace bo
