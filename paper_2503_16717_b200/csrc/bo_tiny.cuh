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
// Warp 0 factors (K <= 16: at most 120 trailing entries per step, warp-level
// synchronisation instead of three CTA barriers per step); every thread of
// the CTA must call it.  G, R have ld kRld; sbuf: 16*16.
__device__ inline void cholesky(const double* G, int K, double tol, double* R, double* sbuf,
                         int* failed_at, double* failed_pivot) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    const int lane = tid;
    for (int e = lane; e < kRld * kRld; e += 32) {
      sbuf[e] = G[e];
      R[e] = 0.0;
    }
    double m = 0.0;
    for (int i = 0; i < K; ++i) {
      const double d = G[i + i * kRld];
      m = m < d ? d : m;  // std::max(max_diag, d)
    }
    const double floor_ = mul(tol, m);
    __syncwarp();
    int fail = 0;
    double fpiv = 0.0;
    for (int t = 0; t < K; ++t) {
      const double piv = sbuf[t + t * kRld];
      if (piv <= floor_) {  // uniform over the warp
        fail = t + 1;
        fpiv = piv;
        break;
      }
      const double rtt = sqrt(piv);
      if (lane == 0) R[t + t * kRld] = rtt;
      for (int j = t + 1 + lane; j < K; j += 32) R[t + j * kRld] = div(sbuf[t + j * kRld], rtt);
      __syncwarp();
      // trailing update s_ij -= r_ti r_tj for t < i <= j
      const int mm = K - t - 1;
      for (int e = lane; e < mm * mm; e += 32) {
        const int i = t + 1 + e % mm, j = t + 1 + e / mm;
        if (i <= j) sbuf[i + j * kRld] = sub(sbuf[i + j * kRld], mul(R[t + i * kRld], R[t + j * kRld]));
      }
      __syncwarp();
    }
    if (fail) {
      // The reference computes column f-1's off-diagonal entries r_i,f-1 (i < f-1)
      // before testing its pivot: they equal s_i,f-1 / r_ii at step i, which the
      // right-looking loop already stored in R.  Columns >= f stay zero in the
      // reference; here rows t < f-1 of columns >= f were filled: clear them.
      for (int e = lane; e < kRld * kRld; e += 32)
        if (e / kRld >= fail) R[e] = 0.0;
    }
    if (lane == 0) {
      *failed_at = fail;
      *failed_pivot = fpiv;
    }
  }
  __syncthreads();
}

// R factor of the thin Householder QR (proj/src/dense.cpp:104-164), sign
// normalised.  Q is not formed (RandCholQR uses only R,
// proj/src/intra_orth.cpp:28-39).  A (m x K, ld lda) is destroyed.  Warp 0
// only; lanes own columns; every sum keeps the reference's sequential row
// order.  (Register-staged operands with fully unrolled, predicated row loops
// measured slower: 20 -> 25 us per 22 x 11 factorization.)
__device__ inline void householder_r(double* A, int lda, int m, int K, double* R, double* tau_buf) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  for (int j = 0; j < K; ++j) {
    double norm = 0.0;
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
    const double alpha = ajj >= 0.0 ? -norm : norm;
    const double v0 = sub(ajj, alpha);
    const double tau = div(-v0, alpha);
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
    if (i < K && j < K && j >= i) {
      double t[kMaxK], r[kMaxK];
#pragma unroll
      for (int l = 0; l < kMaxK; ++l) {
        const bool in = l >= i && l <= j;
        t[l] = in ? T[i + l * kRld] : 0.0;
        r[l] = in ? Rm[l + j * kRld] : 0.0;
      }
#pragma unroll
      for (int l = 0; l < kMaxK; ++l)
        if (l >= i && l <= j) s = add(s, mul(t[l], r[l]));
    }
    out[e] = s;
  }
}

// out = C1 + C2 * Rin  (proj/src/block_orth.cpp:191-203 update_projection,
// times() at proj/src/dense.cpp:44-58 skips zero coefficients)
__device__ inline void update_projection(const double* C1, const double* C2, int ldc, int p, int K,
                                  const double* Rin, double* out) {
  for (int e = threadIdx.x; e < p * K; e += blockDim.x) {
    const int r = e % p, j = e / p;
    // operands first (independent global / shared loads), then the sum in
    // the reference order
    double c2[kMaxK], b[kMaxK];
#pragma unroll
    for (int k = 0; k < kMaxK; ++k) {
      b[k] = k < K ? Rin[k + j * kRld] : 0.0;
      c2[k] = k < K ? C2[r + k * ldc] : 0.0;
    }
    const double c1 = C1[r + j * ldc];
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < kMaxK; ++k) {
      if (k >= K || b[k] == 0.0) continue;
      acc = add(acc, mul(c2[k], b[k]));
    }
    out[r + j * ldc] = add(c1, acc);
  }
}

}  // namespace tiny
}  // namespace bo
