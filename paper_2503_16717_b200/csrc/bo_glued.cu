// bo_glued.cu — the reference's glued test-matrix generator, gen_glued
// (proj/src/problems.cpp:21-61), bit-identical, on the device.  It feeds the
// config-2 microbenchmark (six panels of
// gen_glued(8e6, 6, 11, kappa, kappa, 7)) so that the GPU arm and the
// reference arm consume the same input bytes, and the CPU tests pin it against
// the compiled reference.
//
//   U = random_orthonormal(n, total)   Householder QR of an n x total Gaussian
//                                      (problems.cpp:12-17, dense.cpp:104-164)
//   panel p = U_p diag(sigma_p) W_p^T  W_p = random_orthonormal(w, w) (host)
//
// The reference sums every dot product of its Householder QR strictly in row
// order, and those sums set the bits of U.  No parallel schedule reproduces an
// 8e6-term sequential sum, so each dot runs in one CTA: producer warps stage
// the rounded products x_i * y_i tile by tile in shared memory and one thread
// adds them in row order (the add chain, ~8e6 dependent DADDs, is the bound).
// Independent dots (all trailing columns of one reflector) run concurrently,
// one CTA each.  Everything else (reflector columns, rank-1 updates, the
// panel mix) is elementwise with unfused IEEE operations.
//
// The n x total Gaussian is drawn on the host with glibc log / sin / cos
// exactly as rng.hpp:37-49 does (threads start from jumped MT19937-64 windows,
// mt64_jump.cpp), then copied to the device.  Work: ~3 n total^2 flops of
// rank-1 updates plus 3 total sequential passes of n adds.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <random>
#include <thread>
#include <vector>

#include "bo_hostdense.h"
#include "bo_internal.h"
#include "mt64_jump.h"

namespace {

using bo::hd::Mat;

// --------------------------------------------------------------- host RNG --
// std::mt19937_64 continued from an untempered window g[J .. J+311]
struct MtFromWindow {
  uint64_t s[312];
  int pos = 0;
  explicit MtFromWindow(const uint64_t* w) { std::memcpy(s, w, sizeof s); }
  void twist() {
    for (int t = 0; t < 312; ++t) {
      const uint64_t x = (s[t] & 0xFFFFFFFF80000000ULL) | (s[(t + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      s[t] = s[(t + 156) % 312] ^ xa;
    }
  }
  uint64_t operator()() {
    if (pos == 312) {
      twist();
      pos = 0;
    }
    uint64_t y = s[pos++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
  }
};

// Box-Muller pair t of a Rng stream (rng.hpp:37-49): normal #2t = r cos a, #2t+1 = r sin a
template <class G>
inline void bm_pair(G& g, double* c, double* s) {
  const double u1 = (static_cast<double>(g() >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = static_cast<double>(g() >> 11) * 0x1.0p-53;
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = 6.283185307179586476925286766559 * u2;
  *s = r * std::sin(a);
  *c = r * std::cos(a);
}

// normals #0 .. count-1 of Rng(seed) into out (host, multi-threaded)
void host_normals(uint64_t seed, uint64_t count, double* out) {
  const uint64_t pairs = (count + 1) / 2;
  unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  if (pairs < (1u << 16)) nt = 1;
  const uint64_t per = (pairs + nt - 1) / nt;
  {  // x^(2 c per) mod phi for every thread start, chained (cached in mt64_jump.cpp)
    std::vector<uint64_t> polys((size_t)nt * bo::mt64::poly_words());
    bo::mt64::jump_polys_strided(0, 2 * per, nt, polys.data());
  }
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t) {
    const uint64_t p0 = t * per, p1 = std::min(pairs, p0 + per);
    if (p0 >= p1) break;
    th.emplace_back([=] {
      uint64_t w[312];
      bo::mt64::jump_window_host(seed, 2 * p0, w);
      MtFromWindow g(w);
      for (uint64_t p = p0; p < p1; ++p) {
        double c, s;
        bm_pair(g, &c, &s);
        out[2 * p] = c;
        if (2 * p + 1 < count) out[2 * p + 1] = s;
      }
    });
  }
  for (auto& x : th) x.join();
}

// problems.cpp:12-17 for the small W_p (host; bo_hostdense.h is the reference's order)
Mat random_orthonormal_host(size_t rows, size_t cols, uint64_t seed) {
  std::mt19937_64 g(seed);
  Mat m(rows, cols);
  bool have = false;
  double spare = 0.0;
  for (size_t j = 0; j < cols; ++j)
    for (size_t i = 0; i < rows; ++i) {
      if (have) {
        m(i, j) = spare;
        have = false;
      } else {
        double c;
        bm_pair(g, &c, &spare);
        m(i, j) = c;
        have = true;
      }
    }
  Mat q, r;
  bo::hd::householder_qr(m, q, r);
  return q;
}

// ------------------------------------------------------------ device side --
constexpr int kDotThreads = 256, kDotTile = 2048;

// s = init + sum_{i=i0}^{n-1} fl(x_i * y_i), strictly in row order (one CTA).
//   mode 0: x = y = column xc, init 0             -> out[0] = s            (norm^2)
//   mode 1: y = column yc0 + blockIdx.x, init = Y(i0-1, yc); s *= tau;
//           Y(i0-1, yc) -= s                       -> out[blockIdx.x] = s
__global__ void __launch_bounds__(kDotThreads) seq_dot_kernel(const double* __restrict__ X, double* Y, uint64_t ld,
                                                              int xc, int yc0, uint64_t i0, uint64_t n,
                                                              const double* __restrict__ tau, double* out, int mode) {
  __shared__ __align__(16) double buf[2][kDotTile];
  const int yc = mode == 0 ? xc : yc0 + (int)blockIdx.x;
  const double* x = X + (size_t)xc * ld;
  double* y = Y + (size_t)yc * ld;
  const uint64_t len = n > i0 ? n - i0 : 0;
  const uint64_t ntile = (len + kDotTile - 1) / kDotTile;
  const int warp = threadIdx.x >> 5;
  double s = 0.0;
  if (mode == 1 && threadIdx.x == 0) s = y[i0 - 1];
  // iteration t: warps 1.. produce tile t, thread 0 adds tile t - 1
  for (uint64_t t = 0; t <= ntile; ++t) {
    if (warp > 0 && t < ntile) {
      double* b = buf[t & 1];
      const uint64_t base = i0 + t * kDotTile;
      const int cnt = (int)(n - base < (uint64_t)kDotTile ? n - base : (uint64_t)kDotTile);
      for (int e = threadIdx.x - 32; e < cnt; e += kDotThreads - 32) b[e] = __dmul_rn(x[base + e], y[base + e]);
    }
    if (threadIdx.x == 0 && t > 0) {
      const double* b = buf[(t - 1) & 1];
      const uint64_t rem = n - (i0 + (t - 1) * kDotTile);
      const int cnt = (int)(rem < (uint64_t)kDotTile ? rem : (uint64_t)kDotTile);
      int e = 0;
      for (; e + 8 <= cnt; e += 8) {
        const double2 p0 = *reinterpret_cast<const double2*>(b + e);
        const double2 p1 = *reinterpret_cast<const double2*>(b + e + 2);
        const double2 p2 = *reinterpret_cast<const double2*>(b + e + 4);
        const double2 p3 = *reinterpret_cast<const double2*>(b + e + 6);
        s = __dadd_rn(s, p0.x);
        s = __dadd_rn(s, p0.y);
        s = __dadd_rn(s, p1.x);
        s = __dadd_rn(s, p1.y);
        s = __dadd_rn(s, p2.x);
        s = __dadd_rn(s, p2.y);
        s = __dadd_rn(s, p3.x);
        s = __dadd_rn(s, p3.y);
      }
      for (; e < cnt; ++e) s = __dadd_rn(s, b[e]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (mode == 0) {
      out[0] = s;
    } else {
      s = __dmul_rn(s, *tau);
      y[i0 - 1] = __dsub_rn(y[i0 - 1], s);
      out[blockIdx.x] = s;
    }
  }
}

// reflector j from norm^2 (dense.cpp:112-127): scal = {tau, v0, alpha, skip}
__global__ void reflector_kernel(double* A, uint64_t ld, int j, const double* norm2, double* scal) {
  const double nrm = __dsqrt_rn(*norm2);
  if (nrm == 0.0) {
    scal[0] = 0.0;
    scal[3] = 1.0;
    return;
  }
  const double ajj = A[(size_t)j * ld + j];
  const double alpha = ajj >= 0.0 ? -nrm : nrm;
  const double v0 = __dsub_rn(ajj, alpha);
  scal[0] = __ddiv_rn(-v0, alpha);
  scal[1] = v0;
  scal[2] = alpha;
  scal[3] = 0.0;
}

// w(j,j) = 1, w(i,j) = a(i,j) / v0, a(j,j) = alpha, a(i,j) = 0 for i > j
__global__ void reflector_column_kernel(double* A, double* W, uint64_t ld, int j, uint64_t n,
                                        const double* __restrict__ scal) {
  if (scal[3] != 0.0) return;
  const double v0 = scal[1];
  double* a = A + (size_t)j * ld;
  double* w = W + (size_t)j * ld;
  for (uint64_t i = j + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (i == (uint64_t)j) {
      w[i] = 1.0;
      a[i] = scal[2];
    } else {
      w[i] = __ddiv_rn(a[i], v0);
      a[i] = 0.0;
    }
  }
}

// Y(i, c) -= s_c * w(i, j) for i > j, c = c0 .. c0 + nc - 1
__global__ void rank1_kernel(double* Y, const double* __restrict__ W, uint64_t ld, int j, int c0, int nc, uint64_t n,
                             const double* __restrict__ s, const double* __restrict__ scal) {
  if (scal[3] != 0.0) return;
  const double* w = W + (size_t)j * ld;
  for (uint64_t i = j + 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double wi = w[i];
    for (int c = 0; c < nc; ++c) {
      double* y = Y + (size_t)(c0 + c) * ld;
      y[i] = __dsub_rn(y[i], __dmul_rn(s[c], wi));
    }
  }
}

// dense.cpp:155-162 sign normalisation of Q's columns: flip[c] = 1 negates column c
__global__ void flip_kernel(double* Q, uint64_t ld, int k, uint64_t n, const int* __restrict__ flip) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    for (int c = 0; c < k; ++c)
      if (flip[c]) Q[(size_t)c * ld + i] = -Q[(size_t)c * ld + i];
}

// panel mix (problems.cpp:49-59): V(i, pw + c) = sum_l coef(c, l) U(i, pw + l),
// in l order from +0.0, zero coefficients skipped; rows [r0, r1) to out
__global__ void glued_mix_kernel(const double* __restrict__ U, uint64_t ldu, int panels, int w,
                                 const double* __restrict__ coef, uint64_t r0, uint64_t r1, double* out,
                                 uint64_t ldo) {
  for (uint64_t i = r0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < r1;
       i += (uint64_t)gridDim.x * blockDim.x)
    for (int p = 0; p < panels; ++p)
      for (int c = 0; c < w; ++c) {
        double v = 0.0;
        for (int l = 0; l < w; ++l) {
          const double cf = coef[((size_t)p * w + c) * w + l];
          if (cf == 0.0) continue;
          v = __dadd_rn(v, __dmul_rn(cf, U[(size_t)(p * w + l) * ldu + i]));
        }
        out[(size_t)(p * w + c) * ldo + (i - r0)] = v;
      }
}

}  // namespace

using namespace bo;
using namespace bo::host;

extern "C" int bo_gen_glued(bo_ctx ctx, uint64_t n, uint64_t num_panels, uint64_t panel_width, double kappa_panel,
                            double kappa_global, uint64_t seed, double* out, uint64_t ldo, bo_status* st) {
  ok_st(st);
  CU(cudaSetDevice(ctx->device));
  const uint64_t w = panel_width, total = num_panels * w;
  if (n < total || total == 0) return set_st(st, BO_INVALID, 0, 0.0, "gen_glued: need n >= num_panels * panel_width");
  if (!(kappa_panel >= 1.0 && kappa_global >= 1.0)) return set_st(st, BO_INVALID, 0, 0.0, "gen_glued: kappa < 1");
  if (n != ctx->n_global) return set_st(st, BO_INVALID, 0, 0.0, "gen_glued: n must be the context's global row count");
  const uint64_t r0 = ctx->row_begin, r1 = ctx->row_end;
  if (ldo < r1 - r0) return set_st(st, BO_INVALID, 0, 0.0, "gen_glued: ldo < local rows");
  cudaStream_t sm = ctx->stream;
  const uint64_t ld = n;
  // 1. Gaussian n x total, column-major fill order (problems.cpp:14-15)
  std::unique_ptr<double[]> g(new double[n * total]);  // (no zero fill: every entry is drawn)
  host_normals(derive_seed(seed, 0), n * total, g.get());
  double *A = nullptr, *W = nullptr, *Q = nullptr, *sc = nullptr;
  int* dflip = nullptr;
  struct Free {
    std::vector<void*> p;
    cudaStream_t s;
    ~Free() {
      cudaStreamSynchronize(s);
      for (void* x : p) cudaFree(x);
    }
  } fr{{}, sm};
  CU(cudaMalloc((void**)&A, n * total * 8));
  fr.p.push_back(A);
  CU(cudaMalloc((void**)&W, n * total * 8));
  fr.p.push_back(W);
  CU(cudaMalloc((void**)&Q, n * total * 8));
  fr.p.push_back(Q);
  CU(cudaMalloc((void**)&sc, (8 + 5 * total + total * w) * 8));
  fr.p.push_back(sc);
  CU(cudaMalloc((void**)&dflip, total * sizeof(int)));
  fr.p.push_back(dflip);
  CU(cudaMemcpyAsync(A, g.get(), n * total * 8, cudaMemcpyHostToDevice, sm));
  CU(cudaMemsetAsync(W, 0, n * total * 8, sm));
  CU(cudaMemsetAsync(Q, 0, n * total * 8, sm));
  double* norm2 = sc;          // [1]
  double* taus = sc + 8;       // [total] x 4 scalars
  double* svec = sc + 8 + 4 * total;  // [total]
  const unsigned egrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ctx->num_sms * 8, (n + 255) / 256));
  // 2. Householder QR (dense.cpp:110-136), reflector by reflector
  const int k = (int)total;
  for (int j = 0; j < k; ++j) {
    double* scal = taus + 4 * j;
    seq_dot_kernel<<<1, kDotThreads, 0, sm>>>(A, A, ld, j, j, (uint64_t)j, n, nullptr, norm2, 0);
    reflector_kernel<<<1, 1, 0, sm>>>(A, ld, j, norm2, scal);
    reflector_column_kernel<<<egrid, 256, 0, sm>>>(A, W, ld, j, n, scal);
    if (j + 1 < k) {
      seq_dot_kernel<<<k - j - 1, kDotThreads, 0, sm>>>(W, A, ld, j, j + 1, (uint64_t)j + 1, n, scal, svec, 1);
      rank1_kernel<<<egrid, 256, 0, sm>>>(A, W, ld, j, j + 1, k - j - 1, n, svec, scal);
    }
    CU(cudaGetLastError());
    ctx->launches += j + 1 < k ? 5 : 3;
  }
  // seq_dot_kernel mode 1 skips nothing when tau == 0 (the reference skips
  // the whole reflector): reflector_kernel marks it, and the update kernels
  // return early; the dot's write-back of Y(j, c) -= 0 * s is exact only for
  // finite s, so a zero column (probability 0 for Gaussian data) is rejected
  // below from the host copy of the taus.
  std::vector<double> ht(4 * total);
  CU(cudaMemcpyAsync(ht.data(), taus, 4 * total * 8, cudaMemcpyDeviceToHost, sm));
  CU(cudaStreamSynchronize(sm));
  for (int j = 0; j < k; ++j)
    if (ht[4 * j + 3] != 0.0) return set_st(st, BO_INVALID, j, 0.0, "gen_glued: exactly zero Gaussian column");
  // 3. thin Q by backward accumulation (dense.cpp:138-149)
  {
    std::vector<double> eye(total, 1.0);
    for (int j = 0; j < k; ++j) CU(cudaMemcpyAsync(Q + (size_t)j * ld + j, &eye[j], 8, cudaMemcpyHostToDevice, sm));
    CU(cudaStreamSynchronize(sm));
  }
  for (int jj = k - 1; jj >= 0; --jj) {
    double* scal = taus + 4 * jj;
    seq_dot_kernel<<<k - jj, kDotThreads, 0, sm>>>(W, Q, ld, jj, jj, (uint64_t)jj + 1, n, scal, svec, 1);
    rank1_kernel<<<egrid, 256, 0, sm>>>(Q, W, ld, jj, jj, k - jj, n, svec, scal);
    CU(cudaGetLastError());
    ctx->launches += 2;
  }
  // 4. sign normalisation (dense.cpp:151-162): flip where a(i, i) < 0
  {
    std::vector<double> diag(total);
    for (int i = 0; i < k; ++i)
      CU(cudaMemcpyAsync(&diag[i], A + (size_t)i * ld + i, 8, cudaMemcpyDeviceToHost, sm));
    CU(cudaStreamSynchronize(sm));
    std::vector<int> flip(total);
    for (int i = 0; i < k; ++i) flip[i] = diag[i] < 0.0 ? 1 : 0;
    CU(cudaMemcpyAsync(dflip, flip.data(), total * sizeof(int), cudaMemcpyHostToDevice, sm));
    flip_kernel<<<egrid, 256, 0, sm>>>(Q, ld, k, n, dflip);
    CU(cudaGetLastError());
    ctx->launches++;
  }
  // 5. sigma (problems.cpp:35-45) and the panel coefficients sigma_l W_p(c, l)
  std::vector<double> sigma(total, 1.0);
  const double span = std::max(kappa_global / kappa_panel, 1.0);
  for (uint64_t p = 0; p < num_panels; ++p) {
    const double scale = num_panels == 1 ? 1.0 : std::pow(span, -double(p) / double(num_panels - 1));
    for (uint64_t c = 0; c < w; ++c) {
      const double inner = w == 1 ? 1.0 : std::pow(kappa_panel, -double(c) / double(w - 1));
      sigma[p * w + c] = scale * inner;
    }
  }
  std::vector<double> coef(num_panels * w * w);
  for (uint64_t p = 0; p < num_panels; ++p) {
    const Mat wj = random_orthonormal_host(w, w, derive_seed(seed, 1 + p));
    for (uint64_t c = 0; c < w; ++c)
      for (uint64_t l = 0; l < w; ++l) coef[(p * w + c) * w + l] = sigma[p * w + l] * wj(c, l);
  }
  double* dcoef = sc + 8 + 5 * total;  // num_panels * w * w = total * w
  CU(cudaMemcpyAsync(dcoef, coef.data(), coef.size() * 8, cudaMemcpyHostToDevice, sm));
  glued_mix_kernel<<<egrid, 256, 0, sm>>>(Q, ld, (int)num_panels, (int)w, dcoef, r0, r1, out, ldo);
  CU(cudaGetLastError());
  ctx->launches++;
  CU(cudaStreamSynchronize(sm));
  return BO_OK;
}
