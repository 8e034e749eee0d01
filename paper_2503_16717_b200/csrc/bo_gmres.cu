// bo_gmres.cu — restarted s-step GMRES driver over the device block-
// orthogonalization path: a port of sstep_gmres_solve (proj/src/gmres.cpp:
// 270-512) whose tall work (matrix powers, orthogonalization, x update,
// residual norms, diagnostics) runs on the GPU and whose O(m^2) work
// (Hessenberg assembly, Givens least squares, recovery decisions) runs on the
// host exactly as in the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "bo_hostdense.h"
#include "bo_internal.h"

using namespace bo;
using namespace bo::host;


namespace bo {

// r = b - ax ; partial sums of r^2 per CTA (deterministic, fixed order)
__global__ void __launch_bounds__(256) residual_kernel(long long n, const double* __restrict__ b,
                                                       const double* __restrict__ ax, double* __restrict__ r,
                                                       double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    const double v = b[i] - ax[i];
    r[i] = v;
    s = fma(v, v, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// sum of squares of x (partial per CTA)
__global__ void __launch_bounds__(256) sumsq_kernel(long long n, const double* __restrict__ x, double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) s = fma(x[i], x[i], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// Standard GMRES (gmres.cpp:327-386), one column-wise projection step:
// w -= (*dot_a) q_a (when q_a is given; unfused, as the reference's
// w[t] -= dot * q(t, i)), then the per-CTA partial of q_b . w over the
// updated w (q_b == w: the norm; q_b == nullptr: none).  Fixed-order block sum.
__global__ void __launch_bounds__(256) cgs_update_dot_kernel(long long n, const double* __restrict__ qa,
                                                             const double* __restrict__ dot_a, double* w,
                                                             const double* qb, double* __restrict__ part) {
  __shared__ double red[256];
  const double d = qa ? *dot_a : 0.0;
  double s = 0.0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    double wi = w[i];
    if (qa) {
      wi = __dsub_rn(wi, __dmul_rn(d, qa[i]));
      w[i] = wi;
    }
    if (qb) s = fma(qb == w ? wi : qb[i], wi, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// sum of the per-CTA partials in a fixed order -> *out; optionally h += sum
__global__ void __launch_bounds__(256) finish_dot_kernel(int nparts, const double* __restrict__ part, double* out,
                                                         double* h_entry) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += 256) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *out = red[0];
    if (h_entry) *h_entry += red[0];
  }
}

__global__ void add_to_kernel(const double* src, double* dst) { *dst += *src; }

// y = alpha * x
__global__ void scale_kernel(long long n, double alpha, const double* __restrict__ x, double* __restrict__ y,
                             int divide) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = divide ? x[i] / alpha : alpha * x[i];
}

// x += Q(:, 0:q) y   (gmres.cpp:481-484)
__global__ void __launch_bounds__(256) xupdate_kernel(long long n, int q, const double* __restrict__ Q, long long ldq,
                                                      const double* __restrict__ y, double* __restrict__ x) {
  __shared__ double ys[256];
  for (int j = threadIdx.x; j < q; j += blockDim.x) ys[j] = y[j];
  __syncthreads();
  // eight column loads in flight per thread before their FMAs (memory-level
  // parallelism: one load per thread per iteration leaves HBM idle)
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double v = x[i];
    int j = 0;
    for (; j + 8 <= q; j += 8) {
      double c[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) c[u] = __ldcs(Q + (j + u) * ldq + i);
#pragma unroll
      for (int u = 0; u < 8; ++u) v = fma(c[u], ys[j + u], v);
    }
    for (; j < q; ++j) v = fma(__ldcs(Q + j * ldq + i), ys[j], v);
    x[i] = v;
  }
}

// Four consecutive rows per thread with 256-bit accesses (32-byte aligned x and
// Q columns): the same fma chain per element, in the same column order.
__global__ void __launch_bounds__(256) xupdate4_kernel(long long ngroups, int q, const double* __restrict__ Q,
                                                       long long ldq, const double* __restrict__ y,
                                                       double* __restrict__ x) {
  __shared__ double ys[256];
  for (int j = threadIdx.x; j < q; j += blockDim.x) ys[j] = y[j];
  __syncthreads();
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < ngroups;
       g += (long long)gridDim.x * blockDim.x) {
    const long long i = 4 * g;
    double v[4];
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                 : "l"(x + i));
    int j = 0;
    for (; j + 8 <= q; j += 8) {
      double c[8][4];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        asm("ld.global.cs.v4.f64 {%0, %1, %2, %3}, [%4];"
            : "=d"(c[u][0]), "=d"(c[u][1]), "=d"(c[u][2]), "=d"(c[u][3])
            : "l"(Q + (j + u) * ldq + i));
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = fma(c[u][e], ys[j + u], v[e]);
    }
    for (; j < q; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = fma(__ldcs(Q + j * ldq + i + e), ys[j], v[e]);
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(x + i), "d"(v[0]), "d"(v[1]), "d"(v[2]),
                 "d"(v[3])
                 : "memory");
  }
}

// w = aq - Q(:,0:p) h  ; partial sum of squares (Arnoldi residual column)
__global__ void __launch_bounds__(256) arnoldi_col_kernel(long long n, int p, const double* __restrict__ Q,
                                                          long long ldq, const double* __restrict__ h,
                                                          const double* __restrict__ aq, double* __restrict__ part) {
  __shared__ double hs[256];
  __shared__ double red[256];
  for (int j = threadIdx.x; j < p; j += blockDim.x) hs[j] = h[j];
  __syncthreads();
  double s = 0.0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    double v = aq[i];
    for (int j = 0; j < p; ++j) v = fma(-Q[j * ldq + i], hs[j], v);
    s = fma(v, v, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

}  // namespace bo

namespace {

constexpr double kHappyTol = 1e-8;  // gmres.cpp:161

bool trace_on() {
  static const bool on = getenv("BO_TRACE") != nullptr;
  return on;
}

struct Gm {
  bo_ctx ctx;
  bo_op op;
  double* part = nullptr;  // per-CTA partial sums (device)
  double* gsum = nullptr;  // allreduce buffer (device)
  double* ydev = nullptr;  // least-squares solution y (device)
  int grid = 0;
  std::vector<double> hpart;
  std::vector<cudaEvent_t> ev;  // phase timing of the deferred panel loop (device time)
  ~Gm() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
  cudaEvent_t event(size_t i) {
    while (ev.size() <= i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
    return ev[i];
  }
};

// global sum over ranks of per-CTA partials (fixed order) -> host
int reduce_sum(Gm& g, int nparts, double* out, bo_status* st) {
  bo_ctx ctx = g.ctx;
  g.hpart.resize(nparts);
  CU(cudaMemcpyAsync(g.hpart.data(), g.part, nparts * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  double s = 0.0;
  for (int i = 0; i < nparts; ++i) s += g.hpart[i];
  if (ctx->collective) {
    CU(cudaMemcpyAsync(g.gsum, &s, 8, cudaMemcpyHostToDevice, ctx->stream));
    TRY(comm_allreduce(ctx, g.gsum, 1, st));
    CU(cudaMemcpyAsync(&s, g.gsum, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  *out = s;
  return BO_OK;
}

int norm2(Gm& g, const double* x, double* out, bo_status* st) {
  bo_ctx ctx = g.ctx;
  sumsq_kernel<<<g.grid, 256, 0, ctx->stream>>>((long long)ctx->n_local, x, g.part);
  CU(cudaGetLastError());
  ctx->launches++;
  double s;
  TRY(reduce_sum(g, g.grid, &s, st));
  *out = std::sqrt(s);
  return BO_OK;
}

// gmres.cpp:289-295: r = b - A x ; one norm reduce
int true_residual(Gm& g, const double* b, const double* x, double* ax, double* r, double* gamma, uint64_t* extra,
                  bo_status* st) {
  bo_ctx ctx = g.ctx;
  TRY(op_apply(g.op, x, ax, st));
  residual_kernel<<<g.grid, 256, 0, ctx->stream>>>((long long)ctx->n_local, b, ax, r, g.part);
  CU(cudaGetLastError());
  ctx->launches++;
  extra[BO_LEDGER_NORM]++;
  double s;
  TRY(reduce_sum(g, g.grid, &s, st));
  *gamma = std::sqrt(s);
  return BO_OK;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// One restart cycle of standard GMRES (gmres.cpp:327-386): column-wise
// Arnoldi with two projection passes per column (within a pass each q_i is
// removed from the current w, in the reference's order), one projection reduce
// per pass and one norm reduce per column in the ledger.  Basis columns land
// in Q (ld), the Hessenberg entries in H ((m+1) x m, host).  A comparator
// (SURVEY.md §8(f)4): every dot is its own reduction, so it is launch bound.
int cgs2_cycle(Gm& g, double* Q, uint64_t ld, const double* q1, uint64_t m, double* w, double* dev, hd::Mat& H,
               uint64_t& q_in, bool& happy, uint64_t led[4], double* t_mpk, double* t_orth, bo_status* st) {
  bo_ctx ctx = g.ctx;
  const long long nl = (long long)ctx->n_local;
  double* hdev = dev;                 // (m + 1) x m Hessenberg, column-major
  double* dots = dev + (m + 1) * m;   // m + 1 projection coefficients
  double* nrm2 = dots + m + 1;        // 1
  CU(cudaMemsetAsync(hdev, 0, (m + 1) * m * 8, ctx->stream));
  CU(cudaMemcpyAsync(Q, q1, nl * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  H = hd::Mat(m + 1, m);
  q_in = m;
  happy = false;
  auto finish = [&](double* out, double* h_entry) -> int {
    finish_dot_kernel<<<1, 256, 0, ctx->stream>>>(g.grid, g.part, out, ctx->collective ? nullptr : h_entry);
    CU(cudaGetLastError());
    ctx->launches++;
    if (ctx->collective) {
      TRY(comm_allreduce(ctx, out, 1, st));
      if (h_entry) {
        add_to_kernel<<<1, 1, 0, ctx->stream>>>(out, h_entry);
        CU(cudaGetLastError());
        ctx->launches++;
      }
    }
    return BO_OK;
  };
  auto upd = [&](const double* qa, const double* da, const double* qb) -> int {
    cgs_update_dot_kernel<<<g.grid, 256, 0, ctx->stream>>>(nl, qa, da, w, qb, g.part);
    CU(cudaGetLastError());
    ctx->launches++;
    return BO_OK;
  };
  std::vector<double> hk(m + 2);
  for (uint64_t k = 0; k < m; ++k) {
    auto t0 = std::chrono::steady_clock::now();
    TRY(op_apply(g.op, Q + k * ld, w, st));
    *t_mpk += ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    TRY(upd(nullptr, nullptr, Q));  // q_0 . w
    for (int pass = 0; pass < 2; ++pass) {
      led[BO_LEDGER_PROJECTION]++;
      for (uint64_t i = 0; i <= k; ++i) {
        TRY(finish(dots + i, hdev + i + k * (m + 1)));
        const double* next = i < k ? Q + (i + 1) * ld : (pass == 0 ? Q : w);
        TRY(upd(Q + i * ld, dots + i, next));
      }
    }
    TRY(finish(nrm2, nullptr));  // ||w||^2
    led[BO_LEDGER_NORM]++;
    CU(cudaMemcpyAsync(hk.data(), hdev + k * (m + 1), (k + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(&hk[m + 1], nrm2, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    const double hnorm = std::sqrt(hk[m + 1]);
    double hcol = 0.0;
    for (uint64_t i = 0; i <= k; ++i) {
      H(i, k) = hk[i];
      hcol += hk[i] * hk[i];
    }
    *t_orth += ms_since(t0);
    if (hnorm <= 1e-12 * std::sqrt(hcol + hnorm * hnorm)) {
      q_in = k + 1;
      happy = true;
      break;
    }
    H(k + 1, k) = hnorm;
    scale_kernel<<<g.grid, 256, 0, ctx->stream>>>(nl, hnorm, w, Q + (k + 1) * ld, 1);
    CU(cudaGetLastError());
    ctx->launches++;
  }
  return BO_OK;
}

struct CycleState {
  bool happy = false, aborted = false;
  std::string detail;
  std::vector<double> happy_col;
};

// gmres.cpp:69-87
int solve_upper_right(const hd::Mat& B, const hd::Mat& U, hd::Mat& X, bo_status* st) {
  const size_t q = U.c;
  for (size_t j = 0; j < q; ++j)
    if (U(j, j) == 0.0)
      return set_st(st, BO_SINGULAR_TRIANGULAR, (long long)j, 0.0,
                    "triangular factor is singular: zero diagonal at index %zu", j);
  X = B;
  const size_t p = B.r;
  for (size_t j = 0; j < q; ++j) {
    for (size_t i = 0; i < j; ++i) {
      const double uij = U(i, j);
      if (uij == 0.0) continue;
      for (size_t r = 0; r < p; ++r) X(r, j) -= X(r, i) * uij;
    }
    for (size_t r = 0; r < p; ++r) X(r, j) /= U(j, j);
  }
  return BO_OK;
}

// gmres.cpp:106-151
double solve_lsq(const hd::Mat& H, double gamma, std::vector<double>& y) {
  const size_t p = H.r, q = H.c;
  hd::Mat work = H;
  std::vector<double> rhs(p, 0.0);
  rhs[0] = gamma;
  for (size_t k = 0; k < q && k + 1 < p; ++k) {
    const double a = work(k, k), b = work(k + 1, k);
    if (b == 0.0) continue;
    const double r = std::hypot(a, b);
    const double c = a / r, s = b / r;
    for (size_t j = k; j < q; ++j) {
      const double t0 = work(k, j), t1 = work(k + 1, j);
      work(k, j) = c * t0 + s * t1;
      work(k + 1, j) = -s * t0 + c * t1;
    }
    const double g0 = rhs[k], g1 = rhs[k + 1];
    rhs[k] = c * g0 + s * g1;
    rhs[k + 1] = -s * g0 + c * g1;
  }
  y.assign(q, 0.0);
  for (size_t kk = q; kk-- > 0;) {
    if (work(kk, kk) == 0.0) {
      y[kk] = 0.0;
      continue;
    }
    double s = rhs[kk];
    for (size_t j = kk + 1; j < q; ++j) s -= work(kk, j) * y[j];
    y[kk] = s / work(kk, kk);
  }
  std::vector<double> resid(p, 0.0);
  resid[0] = gamma;
  for (size_t j = 0; j < q; ++j)
    for (size_t i = 0; i < p; ++i) resid[i] -= H(i, j) * y[j];
  double s = 0.0;
  for (double v : resid) s += v * v;
  return std::sqrt(s);
}

// gmres.cpp:173-191
int assemble_hessenberg(bo_basis b, size_t q_in, const std::vector<double>* happy_col, hd::Mat& H, bo_status* st) {
  const size_t p = b->cols, cap = b->cap;
  hd::Mat rshift(p, q_in), ceff(q_in, q_in);
  std::vector<double> c(q_in);
  for (size_t k = 0; k < q_in; ++k) {
    if (happy_col && k + 1 == q_in) {
      for (size_t i = 0; i < p; ++i) rshift(i, k) = (*happy_col)[i];
    } else {
      for (size_t i = 0; i < p && i <= k + 1; ++i) rshift(i, k) = b->r[i + (k + 1) * cap];
    }
    bo_basis_input_coeff_col(b, k, q_in, c.data());
    for (size_t i = 0; i < q_in; ++i) ceff(i, k) = c[i];
  }
  return solve_upper_right(rshift, ceff, H, st);
}

// gmres.cpp:195-248
int recover_panel(Gm& g, bo_basis b, const double* v, uint64_t ldv, int w, bool overlap, const std::string& detail,
                  CycleState& cs, bo_status* st) {
  bo_ctx ctx = g.ctx;
  const bool eff = overlap && b->cols > 0;
  const uint64_t hi = b->cols - (eff ? 1 : 0);
  double* vhat = nullptr;
  CU(ctx_alloc(ctx, (void**)&vhat, ctx->ld * w * 8));
  std::vector<double> pc(std::max<uint64_t>(hi, 1) * w, 0.0);
  int rc = bo_bcgs_project_range(b, v, ldv, w, 0, hi, vhat, ctx->ld, pc.data(), st);
  if (rc) {
    ctx_free(ctx, vhat);
    return rc;
  }
  // recursive CholQR writes the kept columns straight into the slab at `hi`
  double* qdst = b->q + hi * ctx->ld;
  std::vector<double> coeffs(w * w);
  std::vector<uint64_t> kept(w), disc(w);
  std::vector<double> dn(w);
  uint64_t nk = 0, nd = 0, depth = 0;
  bo_status rst;
  rc = bo_recursive_cholqr(ctx, vhat, ctx->ld, w, qdst, ctx->ld, coeffs.data(), kept.data(), &nk, disc.data(),
                           dn.data(), &nd, &depth, b->ledger, &rst);
  ctx_free(ctx, vhat);
  if (rc == BO_CUDA || rc == BO_NCCL) {
    if (st) *st = rst;
    return rc;
  }
  if (rc != BO_OK) {
    cs.aborted = true;
    cs.detail = detail + "; recovery failed: " + rst.msg;
    return BO_OK;
  }
  const uint64_t d = nd == 0 ? (uint64_t)w : disc[0];
  if (d == 0) {
    cs.aborted = true;
    cs.detail = detail + "; recovery kept nothing";
    return BO_OK;
  }
  std::vector<double> proj(std::max<uint64_t>(hi, 1) * d), diag(d * d, 0.0);
  for (uint64_t j = 0; j < d; ++j)
    for (uint64_t i = 0; i < hi; ++i) proj[i + j * hi] = pc[i + j * hi];
  for (uint64_t i = 0; i < d; ++i)
    for (uint64_t j = i; j < d; ++j) diag[i + j * d] = coeffs[i + j * w];
  push_panel_host(b, d, proj.data(), hi, diag.data(), d, eff);
  if (d == (uint64_t)w) return BO_OK;
  for (uint64_t t = 0; t < nd; ++t) {
    const uint64_t c = disc[t];
    double vn;
    TRY(norm2(g, v + c * ldv, &vn, st));
    if (dn[t] > kHappyTol * vn) {
      char buf[128];
      snprintf(buf, sizeof buf, "; column %llu unexplained remainder %f", (unsigned long long)c, dn[t]);
      cs.aborted = true;
      cs.detail = detail + buf;
      return BO_OK;
    }
  }
  const uint64_t p = b->cols;
  cs.happy_col.assign(p, 0.0);
  for (uint64_t i = 0; i < hi; ++i) cs.happy_col[i] = pc[i + d * hi];
  for (uint64_t i = 0; i < d; ++i) cs.happy_col[hi + i] = coeffs[i + d * w];
  cs.happy = true;
  return BO_OK;
}

// ||I - Q^T Q||_2 (Gram on device, symmetric eigenvalues on host) and
// ||A Q - Q H||_F / ||A||_F (gmres.cpp:255-266)
int diagnostics(Gm& g, bo_basis b, const hd::Mat& H, size_t q_in, double a_fro, double* orth, double* arn,
                double* aq, bo_status* st);

}  // namespace

namespace bo {
namespace host {
int wide_gram_host(bo_ctx ctx, const double* q, uint64_t ld, int p, std::vector<double>& G, bo_status* st);
}
}  // namespace bo

namespace {
int diagnostics(Gm& g, bo_basis b, const hd::Mat& H, size_t q_in, double a_fro, double* orth, double* arn,
                double* aq, bo_status* st) {
  bo_ctx ctx = g.ctx;
  const size_t p = b->cols;
  *orth = 0.0;
  if (p > 0) {  // any width: the Gram is assembled from 64 x 64 blocks
    std::vector<double> G;
    TRY(wide_gram_host(ctx, b->q, ctx->ld, (int)p, G, st));
    std::vector<double> a(p * p);
    for (size_t j = 0; j < p; ++j)
      for (size_t i = 0; i < p; ++i) a[i + j * p] = (i == j ? 1.0 : 0.0) - G[i + j * p];
    for (int sweep = 0; sweep < 100; ++sweep) {
      double off = 0.0;
      for (size_t j = 0; j < p; ++j)
        for (size_t i = 0; i < j; ++i) off += a[i + j * p] * a[i + j * p];
      if (off == 0.0) break;
      for (size_t pp = 0; pp < p; ++pp)
        for (size_t qq = pp + 1; qq < p; ++qq) {
          const double apq = a[pp + qq * p];
          if (apq == 0.0) continue;
          const double app = a[pp + pp * p], aqq = a[qq + qq * p];
          const double th = (aqq - app) / (2.0 * apq);
          const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
          const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
          for (size_t r = 0; r < p; ++r) {
            const double arp = a[r + pp * p], arq = a[r + qq * p];
            a[r + pp * p] = c * arp - s * arq;
            a[r + qq * p] = s * arp + c * arq;
          }
          for (size_t r = 0; r < p; ++r) {
            const double apr = a[pp + r * p], aqr = a[qq + r * p];
            a[pp + r * p] = c * apr - s * aqr;
            a[qq + r * p] = s * apr + c * aqr;
          }
        }
    }
    for (size_t i = 0; i < p; ++i) *orth = std::max(*orth, std::fabs(a[i + i * p]));
  }
  // Arnoldi residual: column j: A q_j - Q h_j
  double* hd = nullptr;
  CU(ctx_alloc(ctx, (void**)&hd, std::max<size_t>(H.r, 1) * 8));
  double total = 0.0;
  for (size_t j = 0; j < q_in; ++j) {
    TRY(op_apply(g.op, b->q + j * ctx->ld, aq, st));
    std::vector<double> hcol(H.r);
    for (size_t i = 0; i < H.r; ++i) hcol[i] = H(i, j);
    CU(cudaMemcpyAsync(hd, hcol.data(), H.r * 8, cudaMemcpyHostToDevice, ctx->stream));
    arnoldi_col_kernel<<<g.grid, 256, 0, ctx->stream>>>((long long)ctx->n_local, (int)H.r, b->q, (long long)ctx->ld,
                                                         hd, aq, g.part);
    CU(cudaGetLastError());
    ctx->launches++;
    double s;
    TRY(reduce_sum(g, g.grid, &s, st));
    total += s;
  }
  ctx_free(ctx, hd);
  *arn = std::sqrt(total) / a_fro;
  return BO_OK;
}


}  // namespace

extern "C" int bo_sstep_gmres(bo_op op, const double* b, const double* x0, const bo_solver_config* cfg, double* x,
                              bo_solve_report* rep, bo_status* st) {
  ok_st(st);
  std::memset(rep, 0, sizeof *rep);
  bo_ctx ctx = op->ctx;
  CU(cudaSetDevice(ctx->device));
  // validate_config (gmres.cpp:34-46)
  if (!(cfg->rel_tol > 0.0 && cfg->rel_tol < 1.0)) return set_st(st, BO_INVALID, 0, 0.0, "rel_tol must lie in (0, 1)");
  if (cfg->max_restarts == 0) return set_st(st, BO_INVALID, 0, 0.0, "max_restarts must be positive");
  if (cfg->s < 1 || cfg->s > cfg->shat || cfg->shat > cfg->m) return set_st(st, BO_INVALID, 0, 0.0, "need 1 <= s <= shat <= m");
  if (cfg->shat % cfg->s != 0) return set_st(st, BO_INVALID, 0, 0.0, "s must divide shat");
  if (cfg->m % cfg->shat != 0) return set_st(st, BO_INVALID, 0, 0.0, "shat must divide m");
  if (op->ncols != ctx->n_global) return set_st(st, BO_INVALID, 0, 0.0, "coefficient matrix must be square");
  // engine limits (not reference limits): the x-update / Arnoldi kernels stage
  // y and h columns of up to 256 entries in shared memory, and the two-stage
  // big panel (shat + 1 columns) goes through the <= 64-column wide passes
  if (cfg->m + 1 > 256) return set_st(st, BO_INVALID, 0, 0.0, "m + 1 > 256 is not supported by the GPU driver");
  if ((cfg->scheme == BO_TWOSTAGE_PIP || cfg->scheme == BO_TWOSTAGE_RANDBCGS) && cfg->shat + 1 > 64)
    return set_st(st, BO_INVALID, 0, 0.0, "two-stage big panel shat + 1 > 64 columns is not supported by the GPU engine");
  if (cfg->n != 0 && cfg->n != ctx->n_global) return set_st(st, BO_INVALID, 0, 0.0, "config n does not match the matrix dimension");
  const bool cgs2 = cfg->scheme == BO_STANDARD_CGS2;
  if (!cgs2 && cfg->s + 1 > 16) return set_st(st, BO_INVALID, 0, 0.0, "s > 15 is outside the streaming-pass engine");
  const uint64_t n = ctx->n_global, nl = ctx->n_local, ld = ctx->ld;
  const uint64_t K = cfg->s + 1;

  Gm g;
  g.ctx = ctx;
  g.op = op;
  g.grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(ctx->num_sms * 2, (nl + 255) / 256));
  double *r = nullptr, *ax = nullptr, *panel = nullptr, *q1 = nullptr;
  // per-solve scratch from the ctx pool (stream-ordered, kept reserved between solves)
  struct Free {
    bo_ctx c;
    std::vector<void*> p;
    ~Free() {
      for (void* q : p) ctx_free(c, q);
    }
  } fr{ctx, {}};
  auto scratch = [&](void** p, size_t bytes) {
    const cudaError_t e = ctx_alloc(ctx, p, bytes);
    if (e == cudaSuccess) fr.p.push_back(*p);
    return e;
  };
  CU(scratch((void**)&g.part, 4096 * 8));
  CU(scratch((void**)&g.gsum, 64));
  CU(scratch((void**)&g.ydev, (cfg->m + 2) * 8));
  CU(scratch((void**)&r, ld * 8));
  CU(scratch((void**)&ax, ld * 8));
  CU(scratch((void**)&q1, ld * 8));
  CU(scratch((void**)&panel, ld * K * 8));
  CU(cudaMemsetAsync(panel, 0, ld * K * 8, ctx->stream));
  CU(cudaMemcpyAsync(x, x0, nl * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  double *wbuf = nullptr, *cgsdev = nullptr;  // standard GMRES: w and the Hessenberg / dot scratch
  if (cgs2) {
    CU(scratch((void**)&wbuf, ld * 8));
    CU(scratch((void**)&cgsdev, ((cfg->m + 1) * cfg->m + cfg->m + 2) * 8));
  }

  uint64_t extra[4] = {0, 0, 0, 0};
  // ||A||_F (gmres.cpp:286-288)
  double a_fro2 = op->a_fro_local2;
  if (ctx->collective) {
    CU(cudaMemcpyAsync(g.gsum, &a_fro2, 8, cudaMemcpyHostToDevice, ctx->stream));
    TRY(comm_allreduce(ctx, g.gsum, 1, st));
    ctx->allreduces--;  // setup, not a ledger event
    CU(cudaMemcpyAsync(&a_fro2, g.gsum, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  double a_fro = std::sqrt(a_fro2);
  if (a_fro == 0.0) a_fro = 1.0;

  auto t_start = std::chrono::steady_clock::now();
  double gamma;
  TRY(true_residual(g, b, x, ax, r, &gamma, extra, st));
  rep->t_residual += ms_since(t_start);
  const double gamma0 = gamma;
  rep->initial_residual = gamma0;
  if (gamma0 == 0.0) {
    rep->converged = 1;
    rep->final_relres = 0.0;
    return BO_OK;
  }
  auto acc_ledger = [&](const uint64_t* l) {
    for (int q = 0; q < 4; ++q) rep->reduce[q] += l[q];
    rep->reduce_total += l[0] + l[1] + l[2] + l[3];
  };
  const bool twostage = cfg->scheme == BO_TWOSTAGE_PIP || cfg->scheme == BO_TWOSTAGE_RANDBCGS;
  const int preproc = cfg->scheme == BO_TWOSTAGE_PIP ? BO_PREPROC_PIP : BO_PREPROC_RAND_BCGS;
  bo_basis store = nullptr;
  TRY(bo_basis_create(ctx, cfg->m + 1, &store, st));
  struct FreeB {
    bo_basis b;
    ~FreeB() { bo_basis_destroy(b); }
  } fb{store};

  bool done = false;
  auto t_cycle0 = std::chrono::steady_clock::now();
  cudaEvent_t ev_c0 = nullptr, ev_c1 = nullptr;
  CU(cudaEventCreate(&ev_c0));
  CU(cudaEventCreate(&ev_c1));
  struct FreeEv {
    cudaEvent_t a, b;
    ~FreeEv() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  } fev{ev_c0, ev_c1};
  CU(cudaEventRecord(ev_c0, ctx->stream));
  for (uint64_t cycle = 0; cycle < cfg->max_restarts && !done; ++cycle) {
    if (trace_on() && cycle > 0)
      fprintf(stderr, "[bo] cycle %llu wall %.3f ms (phases so far: sketch %.3f mpk %.3f orth %.3f)\n",
              (unsigned long long)(cycle - 1), ms_since(t_cycle0), rep->t_sketch, rep->t_mpk, rep->t_orth);
    t_cycle0 = std::chrono::steady_clock::now();
    rep->restarts++;
    const double cycle_gamma = gamma;
    bo_basis_reset(store);
    bo_sketch theta = nullptr;
    auto t0 = std::chrono::steady_clock::now();
    if (cfg->scheme == BO_BCGS2_RANDCHOLQR)
      TRY(bo_sketch_build(ctx, cfg->sketch, n, cfg->s, derive_seed(cfg->seed, cycle + 1), &theta, st));
    else if (cfg->scheme == BO_TWOSTAGE_RANDBCGS)
      TRY(bo_sketch_build(ctx, cfg->sketch, n, cfg->shat, derive_seed(cfg->seed, cycle + 1), &theta, st));
    if (theta && cfg->sketch == BO_SKETCH_COUNT_GAUSS && cycle + 1 < cfg->max_restarts)  // next restart's stage
      prefetch_theta_g(derive_seed(cfg->seed, cycle + 2), theta->mc, theta->mhat);
    struct FreeS {
      bo_sketch s;
      ~FreeS() { bo_sketch_destroy(s); }
    } fs{theta};
    rep->t_sketch += ms_since(t0);
    // q1 = r / gamma
    scale_kernel<<<g.grid, 256, 0, ctx->stream>>>((long long)nl, gamma, r, q1, 1);
    CU(cudaGetLastError());
    ctx->launches++;

    CycleState cs;
    hd::Mat H;
    uint64_t q_in = 0;
    double t_h = 0.0;
    if (cgs2) {  // standard GMRES comparator (gmres.cpp:327-386)
      uint64_t led[4] = {0, 0, 0, 0};
      TRY(cgs2_cycle(g, store->q, ld, q1, cfg->m, wbuf, cgsdev, H, q_in, cs.happy, led, &rep->t_mpk, &rep->t_orth,
                     st));
      acc_ledger(led);
      const uint64_t p = cs.happy ? q_in : q_in + 1;
      hd::Mat He(p, q_in);
      for (uint64_t j = 0; j < q_in; ++j)
        for (uint64_t i = 0; i < p; ++i) He(i, j) = H(i, j);
      H = He;
      store->cols = p;  // the diagnostics read Q[:, 0:p]
      t0 = std::chrono::steady_clock::now();
    } else {
      const uint64_t panels = cfg->m / cfg->s;
      const uint64_t ppb = twostage ? cfg->shat / cfg->s : panels;
      if (!twostage) {
        // One-stage schemes: the panels are enqueued back to back (matrix powers,
        // then bo_bcgs2_enqueue) and the host syncs once per restart.  A breakdown
        // at panel f leaves the store as it was after panel f - 1 (the calls after
        // it were device no-ops); panel f's matrix powers are recomputed and it is
        // recovered exactly as the call-by-call loop does (gmres.cpp:421-436),
        // then the remaining panels are enqueued again.
        const int intra = cfg->scheme == BO_BCGS2_CHOLQR2 ? BO_INTRA_CHOLQR2 : BO_INTRA_RAND_CHOLQR;
        uint64_t j0 = 0;
        while (j0 < panels && !cs.happy && !cs.aborted) {
          size_t ne = 0;
          for (uint64_t j = j0; j < panels; ++j) {
            const double* seed_vec = q1;
            if (j > 0) {
              const uint64_t k0 = store->cols - 1;  // speculative count: the columns are on the stream
              bo_basis_mark_seed(store, k0);       // replayed in order by bo_basis_sync
              seed_vec = store->q + k0 * ld;
            }
            CU(cudaEventRecord(g.event(ne++), ctx->stream));
            TRY(bo_mpk(op, seed_vec, cfg->s, panel, ld, st));
            CU(cudaEventRecord(g.event(ne++), ctx->stream));
            bo_status pst;
            const int prc = bo_bcgs2_enqueue(store, panel, ld, K, intra, theta, j > 0, &pst);
            CU(cudaEventRecord(g.event(ne++), ctx->stream));
            if (prc != BO_OK) {  // argument / launch errors, not breakdowns
              bo_status tmp;
              bo_basis_sync(store, nullptr, &tmp);
              if (st) *st = pst;
              return prc;
            }
          }
          uint64_t failed = 0;
          bo_status pst;
          const int prc = bo_basis_sync(store, &failed, &pst);
          for (size_t e = 0; e + 2 < ne; e += 3) {
            float a = 0.f, b2 = 0.f;
            cudaEventElapsedTime(&a, g.ev[e], g.ev[e + 1]);
            cudaEventElapsedTime(&b2, g.ev[e + 1], g.ev[e + 2]);
            rep->t_mpk += a;
            rep->t_orth += b2;
          }
          if (prc == BO_CUDA || prc == BO_NCCL || prc == BO_INVALID) {
            if (st) *st = pst;
            return prc;
          }
          if (prc == BO_OK) break;
          const uint64_t f = j0 + failed;
          t0 = std::chrono::steady_clock::now();
          const double* seed_vec = q1;
          if (f > 0) seed_vec = store->q + (store->cols - 1) * ld;  // seed mark replayed by the sync
          TRY(bo_mpk(op, seed_vec, cfg->s, panel, ld, st));
          CU(cudaStreamSynchronize(ctx->stream));
          rep->t_mpk += ms_since(t0);
          t0 = std::chrono::steady_clock::now();
          TRY(recover_panel(g, store, panel, ld, (int)K, f > 0, pst.msg, cs, st));
          rep->t_orth += ms_since(t0);
          j0 = f + 1;
        }
      }
      for (uint64_t j = 0; twostage && j < panels && !cs.happy && !cs.aborted; ++j) {
        t0 = std::chrono::steady_clock::now();
        const double* seed_vec = q1;
        if (j > 0) {
          const uint64_t k0 = store->cols - 1;
          bo_basis_mark_seed(store, k0);
          seed_vec = store->q + k0 * ld;
        }
        TRY(bo_mpk(op, seed_vec, cfg->s, panel, ld, st));
        rep->t_mpk += ms_since(t0);
        const bool overlap = j > 0;
        t0 = std::chrono::steady_clock::now();
        if (twostage && j % ppb == 0) bo_basis_begin_big_panel(store, theta ? theta->mhat : 0, overlap);
        bo_status pst;
        int prc = twostage ? bo_two_stage_panel(store, panel, ld, K, preproc, theta, overlap, &pst)
                           : bo_bcgs2(store, panel, ld, K,
                                      cfg->scheme == BO_BCGS2_CHOLQR2 ? BO_INTRA_CHOLQR2 : BO_INTRA_RAND_CHOLQR, theta,
                                      overlap, &pst);
        if (prc == BO_CUDA || prc == BO_NCCL || prc == BO_INVALID) {  // not a numerical breakdown
          if (st) *st = pst;
          return prc;
        }
        if (prc != BO_OK) {
          if (!twostage || store->cols == 0) {
            TRY(recover_panel(g, store, panel, ld, (int)K, overlap, pst.msg, cs, st));
          } else {
            cs.aborted = true;
            cs.detail = pst.msg;
          }
        }
        if (twostage && !cs.happy && !cs.aborted && (j + 1) % ppb == 0) {
          bo_status fst;
          int frc = bo_two_stage_finish(store, preproc, cfg->reorthogonalize, 0, nullptr, &fst);
          if (frc == BO_CUDA || frc == BO_NCCL || frc == BO_INVALID) {
            if (st) *st = fst;
            return frc;
          }
          if (frc != BO_OK) {
            cs.aborted = true;
            cs.detail = std::string("second stage: ") + fst.msg;
          }
        }
        rep->t_orth += ms_since(t0);
      }
      if (twostage && cs.aborted && store->cols > store->bp_lo && store->cols > 0) {
        bo_status fst;
        int frc = bo_two_stage_finish(store, preproc, cfg->reorthogonalize, 0, nullptr, &fst);
        if (frc == BO_CUDA || frc == BO_NCCL || frc == BO_INVALID) {
          if (st) *st = fst;
          return frc;
        }
        if (frc != BO_OK) {
          cs.detail += "; basis after the last completed big panel unusable";
          bo_basis_reset(store);  // BasisStore(n, 1): nothing to solve over, ledger dropped
        }
      }
      acc_ledger(store->ledger);

      const uint64_t p = store->cols;
      q_in = cs.happy ? p : (p > 0 ? p - 1 : 0);
      if (q_in == 0) {
        rep->breakdown = cs.aborted;
        snprintf(rep->breakdown_detail, sizeof rep->breakdown_detail, "%s", cs.detail.c_str());
        rep->final_relres = gamma / gamma0;
        done = true;
        continue;
      }
      t0 = std::chrono::steady_clock::now();
      TRY(assemble_hessenberg(store, q_in, cs.happy ? &cs.happy_col : nullptr, H, st));
      t_h = ms_since(t0);
    }
    std::vector<double> y;
    const double lsq = solve_lsq(H, gamma, y);
    const double t_l = ms_since(t0);
    CU(cudaMemcpyAsync(g.ydev, y.data(), q_in * 8, cudaMemcpyHostToDevice, ctx->stream));
    if (nl % 4 == 0 && ld % 4 == 0 && (uintptr_t)x % 32 == 0 && (uintptr_t)store->q % 32 == 0)
      xupdate4_kernel<<<(unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ctx->num_sms * 8, (nl / 4 + 255) / 256)),
                        256, 0, ctx->stream>>>((long long)(nl / 4), (int)q_in, store->q, (long long)ld, g.ydev, x);
    else
      xupdate_kernel<<<(unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ctx->num_sms * 8, (nl + 255) / 256)), 256,
                       0, ctx->stream>>>((long long)nl, (int)q_in, store->q, (long long)ld, g.ydev, x);
    CU(cudaGetLastError());
    ctx->launches++;
    const double t_k = ms_since(t0);
    CU(cudaStreamSynchronize(ctx->stream));
    rep->t_update += ms_since(t0);
    if (trace_on())
      fprintf(stderr, "[bo] cycle %llu update: hessenberg %.3f lsq %.3f launch %.3f sync %.3f ms\n",
              (unsigned long long)cycle, t_h, t_l - t_h, t_k - t_l, ms_since(t0) - t_k);
    t0 = std::chrono::steady_clock::now();
    TRY(true_residual(g, b, x, ax, r, &gamma, extra, st));
    rep->t_residual += ms_since(t0);
    rep->iterations += q_in;
    rep->happy_breakdown = rep->happy_breakdown || cs.happy;
    double orth = 0.0, arn = 0.0;
    if (cfg->diagnostics) {
      t0 = std::chrono::steady_clock::now();
      TRY(diagnostics(g, store, H, q_in, a_fro, &orth, &arn, ax, st));
      rep->t_diag += ms_since(t0);
    }
    if (rep->nhist < 256) {
      rep->relres[rep->nhist] = gamma / gamma0;
      rep->lsq[rep->nhist] = lsq;
      rep->orth[rep->nhist] = orth;
      rep->arnoldi[rep->nhist] = arn;
      rep->nhist++;
    }
    if (gamma / gamma0 <= cfg->rel_tol) {
      rep->converged = 1;
      done = true;
    } else if (cs.aborted) {
      rep->breakdown = 1;
      snprintf(rep->breakdown_detail, sizeof rep->breakdown_detail, "%s", cs.detail.c_str());
      done = true;
    } else if (cs.happy && gamma >= cycle_gamma * (1.0 - 1e-12)) {
      snprintf(rep->breakdown_detail, sizeof rep->breakdown_detail, "stagnated on an invariant subspace");
      done = true;
    }
  }
  CU(cudaEventRecord(ev_c1, ctx->stream));
  acc_ledger(extra);
  rep->final_relres = gamma / gamma0;
  CU(cudaStreamSynchronize(ctx->stream));
  float ms_c = 0.f;
  CU(cudaEventElapsedTime(&ms_c, ev_c0, ev_c1));
  rep->t_cycles = ms_c;
  return BO_OK;
}
