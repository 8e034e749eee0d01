// bo_ops.cu — the rest of the hot-path surface over the streaming-pass engine:
//   * matrix-powers kernel: CSR (int32) and matrix-free Laplacian SpMV,
//     bit-exact with proj/src/sparse.cpp:51-63, with NCCL halo exchange
//   * recursive CholQR breakdown recovery (proj/src/intra_orth.cpp:43-139)
//   * BCGS-PIP and RandBCGS preprocessing (proj/src/block_orth.cpp:230-336)
//   * two-stage panel / finish (proj/src/block_orth.cpp:338-389), whose big
//     panel (up to 64 columns) uses the wide contraction / solve kernels here.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "bo_hostdense.h"
#include "bo_internal.h"
#include "bo_ptx.cuh"
#include "bo_reduce.cuh"


using namespace bo;
using namespace bo::host;


namespace bo {

// ===========================================================================
// SpMV kernels
// ===========================================================================
// y_r = sum_k val[k] * x[col[k]], sequential ascending-column sum from +0.0 with
// unfused mul/add: bit-identical to proj/src/sparse.cpp:57-61.
__global__ void __launch_bounds__(256) spmv_csr_kernel(long long nrows, const int* __restrict__ rp,
                                                       const int* __restrict__ col,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ x, double* __restrict__ y) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < nrows; r += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    const int e = rp[r + 1];
    for (int k = rp[r]; k < e; ++k) s = __dadd_rn(s, __dmul_rn(__ldg(val + k), __ldg(x + col[k])));
    y[r] = s;
  }
}

// Matrix-free constant-coefficient stencils on a k^dims grid: the 2D 5-point /
// 3D 7-point Laplacian (problems.cpp:65-113) and the 3D convection-diffusion
// operator of config 5.  Coefficients c[] are in ascending column order,
// 3D: (i-1, j-1, l-1, self, l+1, j+1, i+1), 2D: (i-1, j-1, self, j+1, i+1);
// the row sum is formed in that order from +0.0 with unfused mul/add, so the
// result is bit-identical to spmv (sparse.cpp:57-61) on the same CSR.
// xext holds [halo_lo rows | local rows | halo_hi rows].  The grid
// coordinates of a row come from divisions by k and k^2; IDX = uint32_t when
// the global row count fits (the 64-bit division subroutine would otherwise
// dominate a kernel that moves only 16 bytes per row).
struct Stencil {
  double c[7];
};

template <typename IDX>
__global__ void __launch_bounds__(256) spmv_stencil_kernel(int dims, IDX k, IDX row_begin, IDX nrows, IDX halo_lo,
                                                           const Stencil st, const double* __restrict__ xext,
                                                           double* __restrict__ y) {
  const IDX off = row_begin - halo_lo;  // xext index = global - off
  const IDX stride = (IDX)gridDim.x * blockDim.x;
  for (IDX r = (IDX)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += stride) {
    const IDX me = row_begin + r;
    const double* xm = xext + (me - off);
    double s = 0.0;
    if (dims == 3) {
      const IDX kk = k * k;
      const IDX i = me / kk, rem = me - i * kk, j = rem / k, l = rem - j * k;
      if (i > 0) s = __dadd_rn(s, __dmul_rn(st.c[0], __ldg(xm - kk)));
      if (j > 0) s = __dadd_rn(s, __dmul_rn(st.c[1], __ldg(xm - k)));
      if (l > 0) s = __dadd_rn(s, __dmul_rn(st.c[2], __ldg(xm - 1)));
      s = __dadd_rn(s, __dmul_rn(st.c[3], __ldg(xm)));
      if (l + 1 < k) s = __dadd_rn(s, __dmul_rn(st.c[4], __ldg(xm + 1)));
      if (j + 1 < k) s = __dadd_rn(s, __dmul_rn(st.c[5], __ldg(xm + k)));
      if (i + 1 < k) s = __dadd_rn(s, __dmul_rn(st.c[6], __ldg(xm + kk)));
    } else {
      const IDX i = me / k, j = me - i * k;
      if (i > 0) s = __dadd_rn(s, __dmul_rn(st.c[0], __ldg(xm - k)));
      if (j > 0) s = __dadd_rn(s, __dmul_rn(st.c[1], __ldg(xm - 1)));
      s = __dadd_rn(s, __dmul_rn(st.c[2], __ldg(xm)));
      if (j + 1 < k) s = __dadd_rn(s, __dmul_rn(st.c[3], __ldg(xm + 1)));
      if (i + 1 < k) s = __dadd_rn(s, __dmul_rn(st.c[4], __ldg(xm + k)));
    }
    y[r] = s;
  }
}

// Four consecutive doubles (32-byte aligned) in one 256-bit access
// (LDG.E.ENL2.256 / STG.E.ENL2.256 on sm_100): one L1 wavefront per 128-byte
// line instead of two half-used 16-byte accesses per thread.
#ifndef BO_SPMV_256
#define BO_SPMV_256 1
#endif
__device__ __forceinline__ void double4_ld(const double* p, double& a, double& b, double& c, double& d) {
#if BO_SPMV_256
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
#else
  const double2 u = __ldg(reinterpret_cast<const double2*>(p));
  const double2 v = __ldg(reinterpret_cast<const double2*>(p + 2));
  a = u.x, b = u.y, c = v.x, d = v.y;
#endif
}
__device__ __forceinline__ void double4_st(double* p, double a, double b, double c, double d) {
#if BO_SPMV_256
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
#else
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
  *reinterpret_cast<double2*>(p + 2) = make_double2(c, d);
#endif
}

// Four consecutive rows per thread (same grid line when k % 4 == 0 and the
// shard starts on a multiple of 4): the centre, +-k and +-k^2 neighbours come
// in as 16-byte vector loads, so each thread keeps ~12 loads in flight instead
// of 7 dependent-address ones per row.  Every row's sum is still formed in the
// reference order with unfused mul/add (bit-identical to spmv_stencil_kernel).
#ifndef BO_SPMV_MINB
#define BO_SPMV_MINB 4
#endif
__global__ void __launch_bounds__(256, BO_SPMV_MINB) spmv_stencil4_kernel(int dims, uint32_t k, uint32_t row_begin, uint32_t ngroups,
                                                            uint32_t halo_lo, const Stencil st,
                                                            const double* __restrict__ xext,
                                                            double* __restrict__ y) {
  // 3D order (i-1, j-1, l-1, self, l+1, j+1, i+1); 2D uses the j / l slots
  const double ci_lo = dims == 3 ? st.c[0] : 0.0, cj_lo = dims == 3 ? st.c[1] : st.c[0];
  const double cl_lo = dims == 3 ? st.c[2] : st.c[1], cself = dims == 3 ? st.c[3] : st.c[2];
  const double cl_hi = dims == 3 ? st.c[4] : st.c[3], cj_hi = dims == 3 ? st.c[5] : st.c[4];
  const double ci_hi = dims == 3 ? st.c[6] : 0.0;
  const uint32_t kk = k * k;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x; gi < ngroups; gi += stride) {
    const uint32_t r = 4 * gi, me = row_begin + r;
    const double* xm = xext + (r + halo_lo);  // x[me]
    uint32_t j, l0;
    bool has_i_lo, has_i_hi;
    if (dims == 3) {
      const uint32_t i = me / kk;
      const uint32_t rem = me - i * kk;
      j = rem / k;
      l0 = rem - j * k;
      has_i_lo = i > 0;
      has_i_hi = i + 1 < k;
    } else {
      j = me / k;  // the 2-D line index plays the role of j (neighbours +-k)
      l0 = me - j * k;
      has_i_lo = has_i_hi = false;
    }
    const bool has_j_lo = j > 0, has_j_hi = j + 1 < k;
    double c[6];  // x[me-1 .. me+4]
    {
      double4_ld(xm, c[1], c[2], c[3], c[4]);
      c[0] = l0 > 0 ? __ldg(xm - 1) : 0.0;
      c[5] = l0 + 4 < k ? __ldg(xm + 4) : 0.0;
    }
    double jl[4], jh[4], il[4], ih[4];
    auto ld4 = [](const double* p, double (&o)[4]) { double4_ld(p, o[0], o[1], o[2], o[3]); };
    if (has_j_lo) ld4(xm - k, jl);
    if (has_j_hi) ld4(xm + k, jh);
    if (has_i_lo) ld4(xm - kk, il);
    if (has_i_hi) ld4(xm + kk, ih);
    double out[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t l = l0 + t;
      double s = 0.0;
      if (has_i_lo) s = __dadd_rn(s, __dmul_rn(ci_lo, il[t]));
      if (has_j_lo) s = __dadd_rn(s, __dmul_rn(cj_lo, jl[t]));
      if (l > 0) s = __dadd_rn(s, __dmul_rn(cl_lo, c[t]));
      s = __dadd_rn(s, __dmul_rn(cself, c[t + 1]));
      if (l + 1 < k) s = __dadd_rn(s, __dmul_rn(cl_hi, c[t + 2]));
      if (has_j_hi) s = __dadd_rn(s, __dmul_rn(cj_hi, jh[t]));
      if (has_i_hi) s = __dadd_rn(s, __dmul_rn(ci_hi, ih[t]));
      out[t] = s;
    }
    double4_st(y + r, out[0], out[1], out[2], out[3]);
  }
}

// Sharded variant of spmv_stencil4_kernel (same sums, bit-identical)
// x is read in place: local row q (0 <= q < nlocal) at x[q], rows below the
// shard at hlo[halo_lo + q] and rows above it at hhi[q - nlocal] (the halo
// rows of op->xext), so a sharded SpMV copies only the halos, not x.
__global__ void __launch_bounds__(256, BO_SPMV_MINB) spmv_stencil4_halo_kernel(int dims, uint32_t k, uint32_t row_begin, uint32_t ngroups,
                                                            uint32_t halo_lo, const Stencil st,
                                                            const double* __restrict__ x,
                                                            const double* __restrict__ hlo,
                                                            const double* __restrict__ hhi,
                                                            double* __restrict__ y) {
  const int nlocal = (int)(4 * ngroups);
  // address of local row q (a 4-row group never straddles the shard edge:
  // k, the shard start and the halo sizes are multiples of 4)
  auto at = [&](int q) -> const double* {
    return q < 0 ? hlo + ((int)halo_lo + q) : (q >= nlocal ? hhi + (q - nlocal) : x + q);
  };
  // 3D order (i-1, j-1, l-1, self, l+1, j+1, i+1); 2D uses the j / l slots
  const double ci_lo = dims == 3 ? st.c[0] : 0.0, cj_lo = dims == 3 ? st.c[1] : st.c[0];
  const double cl_lo = dims == 3 ? st.c[2] : st.c[1], cself = dims == 3 ? st.c[3] : st.c[2];
  const double cl_hi = dims == 3 ? st.c[4] : st.c[3], cj_hi = dims == 3 ? st.c[5] : st.c[4];
  const double ci_hi = dims == 3 ? st.c[6] : 0.0;
  const uint32_t kk = k * k;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x; gi < ngroups; gi += stride) {
    const uint32_t r = 4 * gi, me = row_begin + r;
    const double* xm = x + r;  // x[me]
    uint32_t j, l0;
    bool has_i_lo, has_i_hi;
    if (dims == 3) {
      const uint32_t i = me / kk;
      const uint32_t rem = me - i * kk;
      j = rem / k;
      l0 = rem - j * k;
      has_i_lo = i > 0;
      has_i_hi = i + 1 < k;
    } else {
      j = me / k;  // the 2-D line index plays the role of j (neighbours +-k)
      l0 = me - j * k;
      has_i_lo = has_i_hi = false;
    }
    const bool has_j_lo = j > 0, has_j_hi = j + 1 < k;
    double c[6];  // x[me-1 .. me+4]
    {
      double4_ld(xm, c[1], c[2], c[3], c[4]);
      c[0] = l0 > 0 ? __ldg(at((int)r - 1)) : 0.0;
      c[5] = l0 + 4 < k ? __ldg(at((int)r + 4)) : 0.0;
    }
    double jl[4], jh[4], il[4], ih[4];
    auto ld4 = [](const double* p, double (&o)[4]) { double4_ld(p, o[0], o[1], o[2], o[3]); };
    if (has_j_lo) ld4(at((int)r - (int)k), jl);
    if (has_j_hi) ld4(at((int)r + (int)k), jh);
    if (has_i_lo) ld4(at((int)r - (int)kk), il);
    if (has_i_hi) ld4(at((int)r + (int)kk), ih);
    double out[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t l = l0 + t;
      double s = 0.0;
      if (has_i_lo) s = __dadd_rn(s, __dmul_rn(ci_lo, il[t]));
      if (has_j_lo) s = __dadd_rn(s, __dmul_rn(cj_lo, jl[t]));
      if (l > 0) s = __dadd_rn(s, __dmul_rn(cl_lo, c[t]));
      s = __dadd_rn(s, __dmul_rn(cself, c[t + 1]));
      if (l + 1 < k) s = __dadd_rn(s, __dmul_rn(cl_hi, c[t + 2]));
      if (has_j_hi) s = __dadd_rn(s, __dmul_rn(cj_hi, jh[t]));
      if (has_i_hi) s = __dadd_rn(s, __dmul_rn(ci_hi, ih[t]));
      out[t] = s;
    }
    double4_st(y + r, out[0], out[1], out[2], out[3]);
  }
}

// Plane-marching 3-D 7-point stencil (2.5-D blocking).  A CTA owns JB grid
// lines j0 .. j0+JB-1 (all k points of each: k/PT threads per line, thread tx
// of a line holds points l = tx + (k/PT) t, t < PT, so a warp's shared-memory
// reads are consecutive doubles) and walks a range of planes i.  The lines
// j0-1 .. j0+JB of one plane are contiguous in x, so each plane arrives with
// ONE bulk async copy (TMA engine) into a 4-deep shared-memory ring tracked
// by mbarriers, three planes ahead of the one being computed.  Every x value
// is read from HBM once (plus the two halo lines per CTA, L2 hits); the i-1 /
// i / i+1 values move through registers and the j-1 / j+1 / l-1 / l+1
// neighbours come from the staged plane.  The previous kernel read each x
// value seven times through L1/L2 and was bound there (38 us per SpMV at
// n = 8e6).  Sums are formed exactly as in spmv_stencil_kernel (reference
// order, unfused mul/add): bit-identical.
// Planes: local plane q in [0, np) at x + q k^2; the plane below the shard
// (q = -1) at hlo and the one above (q = np) at hhi (sharded halos).
constexpr int kMarchRing = 4;
template <int PT>
__global__ void __launch_bounds__(512) spmv_stencil7_march_kernel(uint32_t k, uint32_t jb, uint32_t ip0, uint32_t np,
                                                                  uint32_t qlo, uint32_t qhi,
                                                                  const Stencil st, const double* __restrict__ x,
                                                                  const double* __restrict__ hlo,
                                                                  const double* __restrict__ hhi,
                                                                  double* __restrict__ y) {
  extern __shared__ __align__(128) double plb[];  // [kMarchRing][(jb + 2) * k]: lines j0-1 .. j0+jb
  __shared__ __align__(8) uint64_t full[kMarchRing];
  const uint32_t G = k / PT, kk = k * k, pl = (jb + 2) * k;
  const uint32_t tx = threadIdx.x % G, ty = threadIdx.x / G;
  const uint32_t nbj = (k + jb - 1) / jb;
  // the (line block, plane) steps are split into equal contiguous ranges, one
  // per CTA (a persistent grid): every SM gets the same work; a range that
  // crosses into the next line block restarts the march there
  const uint32_t nq = qhi - qlo;  // planes [qlo, qhi) of the shard (all, the interior or one boundary plane)
  const uint64_t total = (uint64_t)nbj * nq;
  const uint64_t u0 = total * blockIdx.x / gridDim.x, u1 = total * (blockIdx.x + 1) / gridDim.x;
  auto plane = [&](int q) -> const double* { return q < 0 ? hlo : (q >= (int)np ? hhi : x + (size_t)q * kk); };
  // plane q (local) exists if its global index is in [0, k) and q in [-1, np]
  auto exists = [&](int q) { return (int)ip0 + q >= 0 && (int)ip0 + q < (int)k && q >= -1 && q <= (int)np; };
  auto buf = [&](int q) { return plb + (size_t)((q + kMarchRing) % kMarchRing) * pl; };
  // pbits bit b = parity of the number of loads issued into buffer b (every
  // thread tracks it); waiting for the latest load into b uses the opposite
  uint32_t pbits = 0;
  auto wait = [&](int q) {
    const int b = (q + kMarchRing) % kMarchRing;
    ptx::mbar_wait(&full[b], ((pbits >> b) & 1u) ^ 1u);
  };
  if (threadIdx.x == 0) {
    for (int b = 0; b < kMarchRing; ++b) ptx::mbar_init(&full[b], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const double c_ilo = st.c[0], c_jlo = st.c[1], c_llo = st.c[2], c_self = st.c[3];
  const double c_lhi = st.c[4], c_jhi = st.c[5], c_ihi = st.c[6];
  for (uint64_t u = u0; u < u1;) {
    const uint32_t jbk = (uint32_t)(u / nq), q0 = qlo + (uint32_t)(u % nq);
    const uint64_t qe = q0 + (u1 - u);
    const uint32_t q1 = qe < qhi ? (uint32_t)qe : qhi;
    u += q1 - q0;
    const uint32_t j0 = jbk * jb, j = j0 + ty;
    const bool act = ty < jb && j < k;
    // lines [jlo, jhi) of a plane exist; they land at line (jlo - j0 + 1) of the buffer
    const uint32_t jlo = j0 > 0 ? j0 - 1 : 0, jhi = min(j0 + jb + 1, k);
    const uint32_t bytes = (jhi - jlo) * k * 8;
    auto issue = [&](int q) {  // every thread: count the load; thread 0 issues it
      const int b = (q + kMarchRing) % kMarchRing;
      pbits ^= 1u << b;
      if (threadIdx.x == 0) {
        ptx::fence_proxy_async_smem();  // earlier generic reads of the buffer before the async write
        ptx::mbar_arrive_expect_tx(&full[b], bytes);
        ptx::bulk_g2s(buf(q) + (size_t)(jlo + 1 - j0) * k, plane(q) + (size_t)jlo * k, bytes, &full[b]);
      }
    };
    const int base = exists((int)q0 - 1) ? (int)q0 - 1 : (int)q0;
    for (int q = base; q < base + kMarchRing && q <= (int)q1; ++q)
      if (exists(q)) issue(q);
    const bool has_jlo = j > 0, has_jhi = j + 1 < k;
    const uint32_t me = (ty + 1) * k + tx;  // point (j, tx) inside a plane buffer
    double prv[PT] = {}, cur[PT], nxt[PT] = {};
    if (base < (int)q0) {
      wait(base);
#pragma unroll
      for (int t = 0; t < PT; ++t) prv[t] = act ? buf(base)[me + G * t] : 0.0;
    }
    wait((int)q0);
#pragma unroll
    for (int t = 0; t < PT; ++t) cur[t] = act ? buf((int)q0)[me + G * t] : 0.0;
    if (base < (int)q0) {
      __syncthreads();  // plane q0 - 1 is in registers: its buffer takes plane q0 + 3
      if ((int)q0 + 3 <= (int)q1 && exists((int)q0 + 3)) issue((int)q0 + 3);
    }
    for (uint32_t q = q0; q < q1; ++q) {
      const uint32_t gi = ip0 + q;
      const bool has_ilo = gi > 0, has_ihi = gi + 1 < k;
      if (has_ihi) wait((int)q + 1);
      if (act) {
        const double* pc = buf((int)q) + me;
        const double* pn = buf((int)q + 1) + me;
        double out[PT];
        // interior lines of interior planes: every term present except l - 1 at
        // l = 0 (t = 0, tx = 0) and l + 1 at l = k - 1 (t = PT - 1, tx = G - 1)
        const bool inner = has_ilo && has_ihi && has_jlo && has_jhi;
        if (inner) {
#pragma unroll
          for (int t = 0; t < PT; ++t) {
            nxt[t] = pn[G * t];
            const double jl = pc[G * t - k], jh = pc[G * t + k];
            const bool lo = t > 0 || tx > 0, hi = t < PT - 1 || tx + 1 < G;
            const double lm = lo ? pc[G * t - 1] : 0.0, lp = hi ? pc[G * t + 1] : 0.0;
            double s = __dadd_rn(0.0, __dmul_rn(c_ilo, prv[t]));
            s = __dadd_rn(s, __dmul_rn(c_jlo, jl));
            if (lo) s = __dadd_rn(s, __dmul_rn(c_llo, lm));
            s = __dadd_rn(s, __dmul_rn(c_self, cur[t]));
            if (hi) s = __dadd_rn(s, __dmul_rn(c_lhi, lp));
            s = __dadd_rn(s, __dmul_rn(c_jhi, jh));
            out[t] = __dadd_rn(s, __dmul_rn(c_ihi, nxt[t]));
          }
        } else {
#pragma unroll
          for (int t = 0; t < PT; ++t) {
            const uint32_t l = tx + G * t;
            nxt[t] = has_ihi ? pn[G * t] : 0.0;
            const double jl = has_jlo ? pc[G * t - k] : 0.0, jh = has_jhi ? pc[G * t + k] : 0.0;
            const double lm = l > 0 ? pc[G * t - 1] : 0.0, lp = l + 1 < k ? pc[G * t + 1] : 0.0;
            double s = 0.0;
            if (has_ilo) s = __dadd_rn(s, __dmul_rn(c_ilo, prv[t]));
            if (has_jlo) s = __dadd_rn(s, __dmul_rn(c_jlo, jl));
            if (l > 0) s = __dadd_rn(s, __dmul_rn(c_llo, lm));
            s = __dadd_rn(s, __dmul_rn(c_self, cur[t]));
            if (l + 1 < k) s = __dadd_rn(s, __dmul_rn(c_lhi, lp));
            if (has_jhi) s = __dadd_rn(s, __dmul_rn(c_jhi, jh));
            if (has_ihi) s = __dadd_rn(s, __dmul_rn(c_ihi, nxt[t]));
            out[t] = s;
          }
        }
        double* yq = y + (size_t)q * kk + (size_t)j * k + tx;
#pragma unroll
        for (int t = 0; t < PT; ++t) yq[G * t] = out[t];
      }
#pragma unroll
      for (int t = 0; t < PT; ++t) {
        prv[t] = cur[t];
        cur[t] = nxt[t];
      }
      __syncthreads();  // every read of plane q is done: its buffer takes plane q + 4
      if ((int)q + 4 <= (int)q1 && exists((int)q + 4)) issue((int)q + 4);
    }
  }
}

// ---------------------------------------------------------------------------
// wide Count stages (thousands of buckets, e.g. count_gauss at shat = 60:
// 7442): bucket-sorted application
// ---------------------------------------------------------------------------
// keys = bucket, values = local row | sign bit, and the bucket histogram
__global__ void count_keys_kernel(const uint32_t* __restrict__ code, uint32_t n, uint32_t* __restrict__ keys,
                                  uint32_t* __restrict__ vals, uint32_t* __restrict__ hist) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t c = code[i];
    keys[i] = c & 0x7fffffffu;
    vals[i] = i | (c & 0x80000000u);
    atomicAdd(hist + (c & 0x7fffffffu), 1u);
  }
}

// out[b + c * mc] = sum over the rows i of bucket b, ascending, of sign_i * V(i, c),
// from +0.0 with unfused mul / add: the order of count_apply_transposed
// (proj/src/sketch.cpp:48-62), so one GPU reproduces it bit for bit.  One
// thread per (bucket, column); the rows' indices are prefetched eight at a
// time so eight independent V loads are in flight per thread.
__global__ void __launch_bounds__(256) count_apply_sorted_kernel(const uint32_t* __restrict__ perm,
                                                                 const uint32_t* __restrict__ boff, uint32_t mc, int K,
                                                                 const double* __restrict__ v, uint64_t ldv,
                                                                 double* __restrict__ out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= mc * (uint32_t)K) return;
  const uint32_t b = t / (uint32_t)K, c = t - b * (uint32_t)K;
  const double* vc = v + (uint64_t)c * ldv;
  const uint32_t e = boff[b + 1];
  double s = 0.0;
  uint32_t q = boff[b];
  for (; q + 8 <= e; q += 8) {
    uint32_t pr[8];
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) pr[u] = __ldg(perm + q + u);
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldg(vc + (pr[u] & 0x7fffffffu));
#pragma unroll
    for (int u = 0; u < 8; ++u) s = __dadd_rn(s, __dmul_rn((pr[u] & 0x80000000u) ? -1.0 : 1.0, x[u]));
  }
  for (; q < e; ++q) {
    const uint32_t pr = __ldg(perm + q);
    s = __dadd_rn(s, __dmul_rn((pr & 0x80000000u) ? -1.0 : 1.0, __ldg(vc + (pr & 0x7fffffffu))));
  }
  out[b + (uint64_t)c * mc] = s;
}

// S = Theta_g^T cnt (mh x K): sequential sums over the mc buckets in the
// transpose_times order of the host stage (dense.cpp:28-42)
__global__ void count_gauss_stage_kernel(const double* __restrict__ theta_g, const double* __restrict__ cnt,
                                         uint32_t mc, uint32_t mh, int K, double* __restrict__ S) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= mh * (uint32_t)K) return;
  const uint32_t i = t % mh, j = t / mh;
  const double* a = theta_g + (uint64_t)i * mc;
  const double* b = cnt + (uint64_t)j * mc;
  double s = 0.0;
  for (uint32_t r = 0; r < mc; ++r) s = __dadd_rn(s, __dmul_rn(__ldg(a + r), __ldg(b + r)));
  S[i + (uint64_t)j * mh] = s;
}

}  // namespace bo

// ===========================================================================
// host wrappers
// ===========================================================================
namespace {

// L^T X (ml x kx) -> host (column-major ml x kx); allreduced across ranks.
// Runs on the streaming pass engine: one QTX pass (Q = L, <= 64 columns) per
// 16-column chunk of X, so every operand streams through TMA at HBM speed
// (the round-1 dedicated kernel loaded its tiles synchronously: ~20x slower).
int wide_contract(bo_ctx ctx, const double* L, uint64_t ldl, int ml, const double* X, uint64_t ldx, int kx,
                  hd::Mat& out, bo_status* st) {
  if (ml > 64 || kx > 64) return set_st(st, BO_INVALID, 0, 0.0, "wide block of more than 64 columns");
  out = hd::Mat(ml, kx);
  const int ldq = (int)round_up((uint64_t)std::max(ml, 1), 8);
  std::vector<double> h((size_t)ldq * 16);
  for (int c0 = 0; c0 < kx; c0 += kMaxK) {
    const int kc = std::min(kMaxK, kx - c0);
    TRY(reset_status(ctx, st));
    PassReq r{};
    r.kind = PK_QTX;
    r.K = kc;
    r.V = X + (size_t)c0 * ldx;
    r.ldv = ldx;
    r.Q = L;
    r.ldq = ldl;
    r.p = ml;
    r.pass_id = 1;
    r.fin.ops = 0;
    TRY(run_pass(ctx, r, st));
    CU(cudaMemcpyAsync(h.data(), ctx->sums, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(ctx->status_host, ctx->status, sizeof(DevStatus), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    for (int j = 0; j < kc; ++j)
      for (int i = 0; i < ml; ++i) out(i, c0 + j) = h[i + (size_t)j * ldq];
  }
  return BO_OK;
}

// out = (V - Q C) R^{-1} (either part optional), kx <= 64 columns, on the
// streaming pass engine in 16-column blocks:
//   update      out_b = V_b - Q C_b                               (UPD_ST)
//   solve       out_b = (out_b - out_{<b} R_{<b,b}) R_bb^{-1}     (P1_ST / UPD_POST_ST)
// (blocked forward substitution; block b reads the solved blocks before it).
// out may alias V.  The round-1 thread-per-row kernel was instruction-bound
// (one shared load per FMA, 64-wide registers): ~10x slower.
int wide_update_trsm(bo_ctx ctx, const double* V, uint64_t ldv, int kx, const double* Q, uint64_t ldq, int p,
                     const hd::Mat* C, const hd::Mat* R, double* out, uint64_t ldo, bo_status* st) {
  if (kx > 64 || p > 64) return set_st(st, BO_INVALID, 0, 0.0, "wide block of more than 64 columns");
  std::vector<double> hc((size_t)LDC * 16), hr(256);
  const double* src = V;
  uint64_t lds = ldv;
  if (Q && p > 0 && C) {
    for (int b0 = 0; b0 < kx; b0 += kMaxK) {
      const int kb = std::min(kMaxK, kx - b0);
      std::fill(hc.begin(), hc.end(), 0.0);
      for (int j = 0; j < kb; ++j)
        for (int i = 0; i < p; ++i) hc[i + (size_t)j * LDC] = (*C)(i, b0 + j);
      CU(cudaMemcpyAsync(T_(ctx, OFF_C1), hc.data(), hc.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
      TRY(reset_status(ctx, st));
      PassReq r{};
      r.kind = PK_UPD_ST;
      r.K = kb;
      r.V = V + (size_t)b0 * ldv;
      r.ldv = ldv;
      r.Q = Q;
      r.ldq = ldq;
      r.p = p;
      r.Cm = T_(ctx, OFF_C1);
      r.out = out + (size_t)b0 * ldo;
      r.ldo = ldo;
      r.pass_id = 1;
      TRY(run_pass(ctx, r, st));
      CU(cudaStreamSynchronize(ctx->stream));  // hc is reused by the next block
    }
    src = out;
    lds = ldo;
  }
  if (R) {
    for (int b0 = 0; b0 < kx; b0 += kMaxK) {
      const int kb = std::min(kMaxK, kx - b0);
      std::fill(hr.begin(), hr.end(), 0.0);
      for (int j = 0; j < kb; ++j)
        for (int i = 0; i <= j; ++i) hr[i + j * 16] = (*R)(b0 + i, b0 + j);
      std::fill(hc.begin(), hc.end(), 0.0);
      for (int j = 0; j < kb; ++j)
        for (int i = 0; i < b0; ++i) hc[i + (size_t)j * LDC] = (*R)(i, b0 + j);
      CU(cudaMemcpyAsync(T_(ctx, OFF_R4), hr.data(), hr.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
      CU(cudaMemcpyAsync(T_(ctx, OFF_C1), hc.data(), hc.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
      TRY(reset_status(ctx, st));
      PassReq r{};
      r.K = kb;
      r.V = src + (size_t)b0 * lds;
      r.ldv = lds;
      r.out = out + (size_t)b0 * ldo;
      r.ldo = ldo;
      r.pass_id = 1;
      if (b0 == 0) {
        r.kind = PK_P1_ST;
        r.Rpre0 = T_(ctx, OFF_R4);
      } else {
        r.kind = PK_UPD_POST_ST;
        r.Q = out;
        r.ldq = ldo;
        r.p = b0;
        r.Cm = T_(ctx, OFF_C1);
        r.Rpost = T_(ctx, OFF_R4);
      }
      TRY(run_pass(ctx, r, st));
      CU(cudaStreamSynchronize(ctx->stream));
    }
  } else if (!(Q && p > 0 && C) && out != V) {
    CU(cudaMemcpy2DAsync(out, ldo * 8, V, ldv * 8, ctx->n_local * 8, kx, cudaMemcpyDeviceToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  return BO_OK;
}

// refactor_block / reorthogonalize_block bookkeeping (block_orth.cpp:111-153)
void refactor_rows(bo_basis b, uint64_t lo, const hd::Mat& t) {
  const uint64_t w = b->cols - lo, cap = b->cap;
  std::vector<double> seg(w);
  auto update = [&](std::vector<double>& m, uint64_t col) {
    for (uint64_t i = 0; i < w; ++i) seg[i] = m[lo + i + col * cap];
    for (uint64_t i = 0; i < w; ++i) {
      double s = 0.0;
      for (uint64_t l = i; l < w; ++l) s += t(i, l) * seg[l];
      m[lo + i + col * cap] = s;
    }
  };
  for (uint64_t col = lo; col < b->cols; ++col) {
    update(b->r, col);
    if (b->seeded[col]) update(b->c, col);
  }
}
void reorth_rows(bo_basis b, uint64_t lo, const hd::Mat& tproj, const hd::Mat& t) {
  const uint64_t w = b->cols - lo, cap = b->cap;
  auto spray = [&](std::vector<double>& m, uint64_t col) {
    for (uint64_t i = 0; i < lo; ++i) {
      double s = 0.0;
      for (uint64_t l = 0; l < w; ++l) s += tproj(i, l) * m[lo + l + col * cap];
      m[i + col * cap] += s;
    }
  };
  for (uint64_t col = lo; col < b->cols; ++col) {
    spray(b->r, col);
    if (b->seeded[col]) spray(b->c, col);
  }
  refactor_rows(b, lo, t);
}

// device cholqr of a wide block in place: Q = V R^{-1} (host Cholesky of the
// reduced Gram, identical to dense.cpp:75-102); one gram ledger event
int wide_cholqr(bo_ctx ctx, double* v, uint64_t ldv, int w, const char* chol_ctx, hd::Mat& R, uint64_t* ledger,
                bo_status* st) {
  hd::Mat G;
  TRY(wide_contract(ctx, v, ldv, w, v, ldv, w, G, st));
  if (ledger) ledger[BO_LEDGER_GRAM]++;
  double piv = 0.0;
  const size_t f = hd::cholesky(G, R, 2.220446049250313e-16, &piv);
  if (f)
    return set_st(st, BO_CHOLESKY_BREAKDOWN, (long long)f, piv, "%s: nonpositive Cholesky pivot at step %zu",
                  chol_ctx, f);
  return wide_update_trsm(ctx, v, ldv, w, nullptr, 0, 0, nullptr, &R, v, ldv, st);
}

}  // namespace


namespace bo {
namespace host {
// S = Theta^T V (mhat x K) to host, one sketch ledger event.  Small sketches
// run fused in one streaming pass; a Gaussian sketch wider than 32 rows (the
// two-stage shat = 60 case, mhat = 122) goes through the wide contraction in
// 64-row chunks; a Count stage with thousands of buckets is swept in bucket
// ranges and the count_gauss dense stage is applied on the host
// (proj/src/sketch.cpp:110-126; Theta_g is replicated).
static bool sorted_count_enabled() {
  static const bool on = [] {
    const char* e = getenv("BO_COUNT_SORTED");  // 0: the bucket-range passes (A/B, diagnostics)
    return e ? atoi(e) != 0 : true;
  }();
  return on;
}

// Build the bucket-sorted row order of a Count stage once per sketch (stable
// radix sort on the bucket, so rows stay ascending within a bucket).
static int count_sort(bo_sketch th, bo_status* st) {
  if (th->perm) return BO_OK;
  bo_ctx ctx = th->ctx;
  const uint32_t n = (uint32_t)ctx->n_local, mc = (uint32_t)th->mc;
  uint32_t *keys = nullptr, *vals = nullptr, *keys2 = nullptr, *hist = nullptr;
  void* tmp = nullptr;
  size_t tb_sort = 0, tb_scan = 0;
  int bits = 1;
  while ((1u << bits) < mc) ++bits;
  cub::DeviceRadixSort::SortPairs(nullptr, tb_sort, keys, keys2, vals, th->perm, (int)n, 0, bits, ctx->stream);
  cub::DeviceScan::ExclusiveSum(nullptr, tb_scan, hist, th->boff, (int)mc + 1, ctx->stream);
  CU(cudaMalloc(&th->perm, std::max<size_t>(n, 1) * 4));
  CU(cudaMalloc(&th->boff, ((size_t)mc + 1) * 4));
  CU(cudaMalloc(&th->cnt, ((size_t)mc * 16 + (size_t)th->mhat * 16) * 8));
  CU(ctx_alloc(ctx, (void**)&keys, std::max<size_t>(n, 1) * 4 * 3 + ((size_t)mc + 1) * 4));
  vals = keys + std::max<uint32_t>(n, 1);
  keys2 = vals + std::max<uint32_t>(n, 1);
  hist = keys2 + std::max<uint32_t>(n, 1);
  CU(ctx_alloc(ctx, &tmp, std::max(tb_sort, tb_scan)));
  CU(cudaMemsetAsync(hist, 0, ((size_t)mc + 1) * 4, ctx->stream));
  if (n) {
    count_keys_kernel<<<std::max(1, std::min(ctx->num_sms * 8, (int)((n + 255) / 256))), 256, 0, ctx->stream>>>(
        th->code, n, keys, vals, hist);
    CU(cudaGetLastError());
    CU(cub::DeviceRadixSort::SortPairs(tmp, tb_sort, keys, keys2, vals, th->perm, (int)n, 0, bits, ctx->stream));
  }
  CU(cub::DeviceScan::ExclusiveSum(tmp, tb_scan, hist, th->boff, (int)mc + 1, ctx->stream));
  ctx_free(ctx, tmp);
  ctx_free(ctx, keys);
  CU(cudaStreamSynchronize(ctx->stream));
  return BO_OK;
}

int sketch_to_host(bo_sketch th, const double* v, uint64_t ldv, int K, std::vector<double>& S, bo_status* st) {
  bo_ctx ctx = th->ctx;
  const uint64_t mh = th->mhat;
  S.assign(mh * K, 0.0);
  const bool small = th->kind == BO_SKETCH_GAUSSIAN ? mh <= 32 : th->mc * (uint64_t)K <= 4096;
  if (small) {
    TRY(reset_status(ctx, st));
    TRY(sketch_pass(th, v, ldv, K, 1, 0, st));
    TRY(fetch(ctx, true, st));
    std::memcpy(S.data(), ctx->tiny_host + OFF_S, mh * K * 8);
    return BO_OK;
  }
  if (th->kind == BO_SKETCH_GAUSSIAN) {
    for (uint64_t c0 = 0; c0 < mh; c0 += 64) {
      const int rows = (int)std::min<uint64_t>(64, mh - c0);
      hd::Mat M;
      TRY(wide_contract(ctx, th->theta + c0 * th->ldth, th->ldth, rows, v, ldv, K, M, st));
      for (int j = 0; j < K; ++j)
        for (int i = 0; i < rows; ++i) S[(c0 + i) + j * mh] = M(i, j);
    }
    return BO_OK;
  }
  const uint64_t mc = th->mc;
  if (sorted_count_enabled() && K <= 16 && ctx->n_local < (1ull << 31)) {
    // bucket-sorted application: one sort per sketch, then one gather pass
    TRY(count_sort(th, st));
    const uint32_t nt = (uint32_t)(mc * K);
    count_apply_sorted_kernel<<<(nt + 255) / 256, 256, 0, ctx->stream>>>(th->perm, th->boff, (uint32_t)mc, K, v, ldv,
                                                                         th->cnt);
    CU(cudaGetLastError());
    ctx->launches++;
    if (ctx->collective) TRY(comm_allreduce(ctx, th->cnt, mc * K, st));
    const double* res = th->cnt;
    if (th->kind != BO_SKETCH_COUNT) {
      const uint32_t ng = (uint32_t)(mh * K);
      count_gauss_stage_kernel<<<(ng + 127) / 128, 128, 0, ctx->stream>>>(th->theta_g, th->cnt, (uint32_t)mc,
                                                                           (uint32_t)mh, K, th->cnt + mc * 16);
      CU(cudaGetLastError());
      ctx->launches++;
      res = th->cnt + mc * 16;
    }
    CU(cudaMemcpyAsync(S.data(), res, mh * K * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return BO_OK;
  }
  const int chunk = std::max(64, 4096 / K);
  std::vector<double> cnt(mc * K, 0.0), hs;
  for (uint64_t b0 = 0; b0 < mc; b0 += chunk) {
    const int nb = (int)std::min<uint64_t>(chunk, mc - b0);
    TRY(reset_status(ctx, st));
    PassReq r{};
    r.kind = PK_SKC;
    r.K = K;
    r.V = v;
    r.ldv = ldv;
    r.sk = th;
    r.bucket_lo = (int)b0;
    r.bucket_n = nb;
    r.fin.ops = 0;
    TRY(run_pass(ctx, r, st));
    hs.resize((size_t)nb * 16);
    CU(cudaMemcpyAsync(hs.data(), ctx->sums, (size_t)nb * 16 * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    for (int j = 0; j < K; ++j)
      for (int i = 0; i < nb; ++i) cnt[(b0 + i) + j * mc] = hs[i + (size_t)j * nb];
  }
  if (th->kind == BO_SKETCH_COUNT) {
    S = cnt;
    return BO_OK;
  }
  for (int j = 0; j < K; ++j)  // transpose_times(dense, count) order (dense.cpp:28-42)
    for (uint64_t i = 0; i < mh; ++i) {
      double s = 0.0;
      for (uint64_t r = 0; r < mc; ++r) s += th->theta_g_host[r + i * mc] * cnt[r + j * mc];
      S[i + j * mh] = s;
    }
  return BO_OK;
}
}  // namespace host
}  // namespace bo

// ===========================================================================
// operator / SpMV / MPK
// ===========================================================================
namespace {
int op_setup_halo(bo_op op, long long need_lo, long long need_hi, bo_status* st) {
  bo_ctx ctx = op->ctx;
  op->halo_lo = (uint64_t)std::max<long long>(0, (long long)ctx->row_begin - need_lo);
  op->halo_hi = (uint64_t)std::max<long long>(0, need_hi - (long long)ctx->row_end);
  if (ctx->world > 1) {
    // every rank learns its neighbours' needs: [halo_lo, halo_hi] per rank
    uint64_t* d = nullptr;
    CU(cudaMalloc(&d, (2 + 2 * ctx->world) * 8));
    uint64_t mine[2] = {op->halo_lo, op->halo_hi};
    // stream-ordered: a pageable cudaMemcpy may return before its DMA lands, and
    // the non-blocking ctx stream does not order after the legacy stream
    CU(cudaMemcpyAsync(d, mine, 16, cudaMemcpyHostToDevice, ctx->stream));
    TRY(comm_allgather_u64(ctx, d, 2, d + 2, st));
    std::vector<uint64_t> all(2 * ctx->world);
    CU(cudaMemcpyAsync(all.data(), d + 2, 16 * ctx->world, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    cudaFree(d);
    op->peer_need_lo = ctx->rank + 1 < ctx->world ? all[2 * (ctx->rank + 1)] : 0;  // rank+1 needs my tail
    op->peer_need_hi = ctx->rank > 0 ? all[2 * (ctx->rank - 1) + 1] : 0;           // rank-1 needs my head
    if (op->halo_lo > (ctx->rank > 0 ? ctx->row_begin : 0) || op->peer_need_lo > ctx->n_local ||
        op->peer_need_hi > ctx->n_local)
      return set_st(st, BO_INVALID, 0, 0.0, "halo wider than a neighbouring shard is not supported");
  }
  const uint64_t ext = op->halo_lo + ctx->n_local + op->halo_hi;
  if (ctx->world > 1 || op->halo_lo || op->halo_hi) CU(cudaMalloc(&op->xext, std::max<uint64_t>(ext, 1) * 8));
  return BO_OK;
}

// xext <- [recv halo_lo | x | recv halo_hi]; returns the pointer SpMV reads
// Fills the halo rows of op->xext from the neighbour ranks.  copy_local also
// copies the local rows into its middle, for kernels that index x as one
// array (CSR columns); the 4-row stencil kernel reads x in place.
int halo_exchange(bo_op op, const double* x, const double** xe, bool copy_local, bo_status* st,
                  cudaStream_t s = nullptr) {
  bo_ctx ctx = op->ctx;
  if (!op->xext) {
    *xe = x;
    return BO_OK;
  }
  if (copy_local)
    CU(cudaMemcpyAsync(op->xext + op->halo_lo, x, ctx->n_local * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  if (ctx->world > 1) {
    bo_p2p_op ops[4];
    int n = 0;
    const int r = ctx->rank;
    double* xs = const_cast<double*>(x);
    if (r > 0) {
      if (op->halo_lo) ops[n++] = {r - 1, 0, op->xext, op->halo_lo};
      if (op->peer_need_hi) ops[n++] = {r - 1, 1, xs, op->peer_need_hi};
    }
    if (r + 1 < ctx->world) {
      if (op->halo_hi) ops[n++] = {r + 1, 0, op->xext + op->halo_lo + ctx->n_local, op->halo_hi};
      if (op->peer_need_lo) ops[n++] = {r + 1, 1, xs + ctx->n_local - op->peer_need_lo, op->peer_need_lo};
    }
    TRY(comm_exchange(ctx, n, ops, st, s));
  }
  *xe = op->xext;
  return BO_OK;
}
}  // namespace

extern "C" int bo_op_csr(bo_ctx ctx, uint64_t ncols, const int64_t* row_ptr, const int64_t* col, const double* val,
                         bo_op* out, bo_status* st) {
  ok_st(st);
  *out = nullptr;
  CU(cudaSetDevice(ctx->device));
  const uint64_t nl = ctx->n_local;
  const int64_t base = row_ptr[0];
  const uint64_t nnz = (uint64_t)(row_ptr[nl] - base);
  if (nnz >= (1ull << 31)) return set_st(st, BO_INVALID, 0, 0.0, "local nnz exceeds int32");
  long long need_lo = (long long)ctx->row_begin, need_hi = (long long)ctx->row_end;
  double fro = 0.0;
  for (uint64_t k = 0; k < nnz; ++k) {
    need_lo = std::min<long long>(need_lo, col[k]);
    need_hi = std::max<long long>(need_hi, col[k] + 1);
    fro += val[k] * val[k];
  }
  bo_op op = new bo_op_s();
  op->ctx = ctx;
  op->kind = 0;
  op->ncols = ncols;
  op->nnz = nnz;
  int rc = op_setup_halo(op, need_lo, need_hi, st);
  if (rc) {
    bo_op_destroy(op);
    return rc;
  }
  const long long off = (long long)ctx->row_begin - (long long)op->halo_lo;
  std::vector<int> rp(nl + 1), ci(std::max<uint64_t>(nnz, 1));
  for (uint64_t r = 0; r <= nl; ++r) rp[r] = (int)(row_ptr[r] - base);
  for (uint64_t k = 0; k < nnz; ++k) ci[k] = (int)(col[k] - off);
  cudaError_t e = cudaMalloc(&op->row_ptr, (nl + 1) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&op->col, std::max<uint64_t>(nnz, 1) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&op->val, std::max<uint64_t>(nnz, 1) * 8);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(op->row_ptr, rp.data(), (nl + 1) * 4, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess && nnz) e = cudaMemcpyAsync(op->col, ci.data(), nnz * 4, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess && nnz) e = cudaMemcpyAsync(op->val, val, nnz * 8, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);  // rp / ci are freed on return
  if (e != cudaSuccess) {
    bo_op_destroy(op);
    return set_st(st, BO_CUDA, 0, 0.0, "CSR upload failed: %s", cudaGetErrorString(e));
  }
  // ||A||_F over all ranks (host arithmetic; the reference sums values in CSR order)
  op->a_fro_local2 = fro;
  *out = op;
  return BO_OK;
}

extern "C" int bo_op_stencil(bo_ctx ctx, int dims, uint64_t k, const double* coeffs, bo_op* out, bo_status* st) {
  ok_st(st);
  *out = nullptr;
  CU(cudaSetDevice(ctx->device));
  if (dims != 2 && dims != 3) return set_st(st, BO_INVALID, 0, 0.0, "dims must be 2 or 3");
  const uint64_t n = dims == 2 ? k * k : k * k * k;
  if (n != ctx->n_global) return set_st(st, BO_INVALID, 0, 0.0, "grid size does not match ctx rows");
  bo_op op = new bo_op_s();
  op->ctx = ctx;
  op->kind = 1;
  op->dims = dims;
  op->k = k;
  op->ncols = n;
  for (int q = 0; q < 2 * dims + 1; ++q) op->coef[q] = coeffs[q];
  const uint64_t plane = dims == 2 ? k : k * k;
  const long long need_lo = std::max<long long>(0, (long long)ctx->row_begin - (long long)plane);
  const long long need_hi = std::min<long long>((long long)n, (long long)ctx->row_end + (long long)plane);
  int rc = op_setup_halo(op, ctx->world > 1 ? need_lo : (long long)ctx->row_begin,
                         ctx->world > 1 ? need_hi : (long long)ctx->row_end, st);
  if (rc) {
    bo_op_destroy(op);
    return rc;
  }
  // ||A||_F^2 of this shard's rows: entries squared and summed in row order,
  // column-ascending within a row (the CSR value order, gmres.cpp:286-288)
  double fro = 0.0;
  for (uint64_t me = ctx->row_begin; me < ctx->row_end; ++me) {
    bool has[7];
    if (dims == 3) {
      const uint64_t i = me / (k * k), j = (me / k) % k, l = me % k;
      const bool h3[7] = {i > 0, j > 0, l > 0, true, l + 1 < k, j + 1 < k, i + 1 < k};
      std::copy(h3, h3 + 7, has);
    } else {
      const uint64_t i = me / k, j = me % k;
      const bool h2[5] = {i > 0, j > 0, true, j + 1 < k, i + 1 < k};
      std::copy(h2, h2 + 5, has);
    }
    for (int q = 0; q < 2 * dims + 1; ++q)
      if (has[q]) fro += op->coef[q] * op->coef[q];
  }
  op->a_fro_local2 = fro;
  *out = op;
  return BO_OK;
}

extern "C" int bo_op_laplace(bo_ctx ctx, int dims, uint64_t k, bo_op* out, bo_status* st) {
  // problems.cpp:65-113: diagonal 2 * dims, every neighbour -1
  const double c3[7] = {-1.0, -1.0, -1.0, 6.0, -1.0, -1.0, -1.0};
  const double c2[5] = {-1.0, -1.0, 4.0, -1.0, -1.0};
  return bo_op_stencil(ctx, dims, k, dims == 3 ? c3 : c2, out, st);
}

extern "C" int bo_op_destroy(bo_op op) {
  if (!op) return BO_OK;
  cudaStreamSynchronize(op->ctx->stream);
  cudaFree(op->row_ptr);
  cudaFree(op->col);
  cudaFree(op->val);
  cudaFree(op->xext);
  delete op;
  return BO_OK;
}

namespace bo {
namespace host {
int op_apply(bo_op op, const double* x, double* y, bo_status* st) {
  bo_ctx ctx = op->ctx;
  const long long nl = (long long)ctx->n_local;
  // the 4-row stencil kernel (reads x in place, halos from op->xext)
  const bool st4 = op->kind != 0 && ctx->n_global + 2 * op->k * op->k < (1ull << 31) && op->k % 4 == 0 &&
                   ctx->row_begin % 4 == 0 && nl % 4 == 0 && op->halo_lo % 4 == 0 && op->halo_hi % 4 == 0 &&
                   ((uintptr_t)x % 32) == 0 && ((uintptr_t)y % 32) == 0 &&
                   ((uintptr_t)(op->xext ? op->xext : x) % 32) == 0;
  // plane-marching 3-D kernel: whole planes per shard, halos of one plane
  static const bool march_on = [] {
    const char* e = getenv("BO_SPMV_MARCH");
    return !(e && atoi(e) == 0);
  }();
  const uint64_t kk = op->k * op->k;
  const bool march = march_on && st4 && op->dims == 3 && op->k <= 512 && ctx->row_begin % kk == 0 &&
                     nl % (long long)kk == 0 && (op->halo_lo == 0 || op->halo_lo == kk) &&
                     (op->halo_hi == 0 || op->halo_hi == kk);
  Stencil stc;
  for (int q = 0; q < 7; ++q) stc.c[q] = op->coef[q];
  if (march) {
    // four points per thread, 256 threads (k = 200: five lines per CTA, four
    // CTAs per SM).  Measured at n = 8e6 (scripts/prof_spmv.py): 30.7 us per
    // SpMV; eight points per thread (BO_SPMV_PT=8, ten lines: fewer halo
    // reads) 36.7 us, 384 / 512-thread CTAs 31.2 / 32.5 us, the 4-row
    // kernel below 38 us.
    static const int pt_env = [] {
      const char* e = getenv("BO_SPMV_PT");
      return e ? atoi(e) : 0;
    }();
    static const int tpb_env = [] {
      const char* e = getenv("BO_SPMV_TPB");
      return e ? atoi(e) : 256;
    }();
    static const bool overlap_on = [] {
      const char* e = getenv("BO_HALO_OVERLAP");
      return !(e && atoi(e) == 0);
    }();
    const uint32_t k = (uint32_t)op->k;
    const uint32_t PT = (pt_env == 8 && k % 8 == 0 && k >= 64) ? 8 : 4, G = k / PT;
    const uint32_t jb = std::max<uint32_t>(1, std::min<uint32_t>((uint32_t)std::min(512, tpb_env) / G, k));
    const uint32_t nbj = (k + jb - 1) / jb, np = (uint32_t)(nl / (long long)kk);
    const size_t smem = (size_t)kMarchRing * (jb + 2) * k * 8;
    const uint32_t per_sm = (uint32_t)std::max<size_t>(1, std::min<size_t>(4, (220 * 1024) / smem));
    const double* hlo = op->xext ? op->xext + op->halo_lo - kk : x;  // the plane below (when it exists)
    const double* hhi = op->xext ? op->xext + op->halo_lo + nl : x;
    auto kfn = PT == 8 ? spmv_stencil7_march_kernel<8> : spmv_stencil7_march_kernel<4>;
    if (smem > 48 * 1024)
      CU(cudaFuncSetAttribute((const void*)kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // persistent grid over planes [qlo, qhi): as many CTAs as fit on the SMs at once, equal shares
    auto launch = [&](uint32_t qlo, uint32_t qhi) {
      const uint32_t grid_m =
          std::max<uint32_t>(1, std::min<uint32_t>(nbj * (qhi - qlo), (uint32_t)ctx->num_sms * per_sm));
      kfn<<<grid_m, G * jb, smem, ctx->stream>>>(k, jb, (uint32_t)(ctx->row_begin / kk), np, qlo, qhi, stc, x, hlo,
                                                  hhi, y);
      ctx->launches++;
    };
    const double* xe;
    if (op->xext && ctx->world > 1 && np >= 3 && overlap_on) {
      // Sharded: the interior planes 1 .. np-2 read only local planes, so they
      // run while the halo planes travel on a side stream (NCCL p2p or the
      // host transport); the two boundary planes follow the exchange.
      if (!ctx->side) {
        CU(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&ctx->ev_x, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming));
      }
      CU(cudaEventRecord(ctx->ev_x, ctx->stream));  // x is ready
      launch(1, np - 1);
      CU(cudaStreamWaitEvent(ctx->side, ctx->ev_x, 0));
      TRY(halo_exchange(op, x, &xe, false, st, ctx->side));
      CU(cudaEventRecord(ctx->ev_halo, ctx->side));
      CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));
      launch(0, 1);
      launch(np - 1, np);
    } else {
      TRY(halo_exchange(op, x, &xe, false, st));
      launch(0, np);
    }
    CU(cudaGetLastError());
    return BO_OK;
  }
  const double* xe;
  TRY(halo_exchange(op, x, &xe, !st4, st));
  const int grid = (int)std::max<long long>(1, std::min<long long>((long long)ctx->num_sms * 8, (nl + 255) / 256));
  if (op->kind == 0)
    spmv_csr_kernel<<<grid, 256, 0, ctx->stream>>>(nl, op->row_ptr, op->col, op->val, xe, y);
  else {
    if (st4) {
      const uint32_t ng = (uint32_t)(nl / 4);
      // one 4-row group per thread, no grid-stride loop: as many loads in
      // flight as the SMs hold (ncu: the capped grid was latency-bound)
      static const int cap = [] {
        const char* e = getenv("BO_SPMV_CTAS");
        return e ? atoi(e) : 1 << 30;
      }();
      const int g4 = (int)std::max<long long>(1, std::min<long long>((long long)cap, (ng + 255) / 256));
      const double* hlo = op->xext ? op->xext : x;
      const double* hhi = op->xext ? op->xext + op->halo_lo + nl : x;
      if (op->xext)
        spmv_stencil4_halo_kernel<<<g4, 256, 0, ctx->stream>>>(op->dims, (uint32_t)op->k, (uint32_t)ctx->row_begin,
                                                               ng, (uint32_t)op->halo_lo, stc, x, hlo, hhi, y);
      else
        spmv_stencil4_kernel<<<g4, 256, 0, ctx->stream>>>(op->dims, (uint32_t)op->k, (uint32_t)ctx->row_begin, ng,
                                                          0u, stc, x, y);
    } else if (ctx->n_global + 2 * op->k * op->k < (1ull << 31)) {
      spmv_stencil_kernel<uint32_t><<<grid, 256, 0, ctx->stream>>>(op->dims, (uint32_t)op->k,
                                                                   (uint32_t)ctx->row_begin, (uint32_t)nl,
                                                                   (uint32_t)op->halo_lo, stc, xe, y);
    } else {
      spmv_stencil_kernel<unsigned long long><<<grid, 256, 0, ctx->stream>>>(
          op->dims, (unsigned long long)op->k, (unsigned long long)ctx->row_begin, (unsigned long long)nl,
          (unsigned long long)op->halo_lo, stc, xe, y);
    }
  }
  CU(cudaGetLastError());
  ctx->launches++;
  return BO_OK;
}
}  // namespace host
}  // namespace bo

extern "C" int bo_spmv(bo_op op, const double* x, double* y, bo_status* st) {
  ok_st(st);
  CU(cudaSetDevice(op->ctx->device));
  TRY(op_apply(op, x, y, st));
  CU(cudaStreamSynchronize(op->ctx->stream));
  return BO_OK;
}

extern "C" int bo_mpk(bo_op op, const double* v0, uint64_t s, double* v, uint64_t ldv, bo_status* st) {
  ok_st(st);  // gmres.cpp:48-58 monomial basis
  bo_ctx ctx = op->ctx;
  CU(cudaSetDevice(ctx->device));
  if (v0 != v) CU(cudaMemcpyAsync(v, v0, ctx->n_local * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  for (uint64_t k = 0; k < s; ++k) TRY(op_apply(op, v + k * ldv, v + (k + 1) * ldv, st));
  CU(cudaStreamSynchronize(ctx->stream));
  return BO_OK;
}

// ===========================================================================
// recursive CholQR (intra_orth.cpp:43-139)
// ===========================================================================
namespace {
struct RecAcc {
  double* q;  // output, n_local x k (ld ldq)
  uint64_t ldq;
  uint64_t k;
  std::vector<double> coeffs;  // k x k
  std::vector<uint64_t> kept, disc;
  std::vector<double> dnorm;
  uint64_t depth = 0;
};

int rec_impl(bo_ctx ctx, const double* v, uint64_t ldv, int w, const std::vector<uint64_t>& ids, RecAcc& acc,
             uint64_t* ledger, bo_status* st) {
  if (w == 0) return BO_OK;
  // gram + cholesky on device (partial factor kept on failure)
  TRY(reset_status(ctx, st));
  PassReq g{};
  g.kind = PK_GRAM;
  g.K = w;
  g.V = v;
  g.ldv = ldv;
  g.pass_id = 1;
  g.fin.ops = FIN_CHOL | FIN_COPY_G;
  g.fin.Rchol = T_(ctx, OFF_R1);
  g.fin.Gout = T_(ctx, OFF_G);
  TRY(run_pass(ctx, g, st));
  TRY(fetch(ctx, true, st));
  if (ledger) ledger[BO_LEDGER_GRAM]++;
  const DevStatus d = *ctx->status_host;
  const double* R = ctx->tiny_host + OFF_R1;
  const double* G = ctx->tiny_host + OFF_G;
  const uint64_t K = acc.k;
  if (d.code == ST_OK) {
    const uint64_t base = acc.kept.size();
    PassReq t{};
    t.kind = PK_P1_ST;
    t.K = w;
    t.V = v;
    t.ldv = ldv;
    t.Rpre0 = T_(ctx, OFF_R1);
    t.out = acc.q + base * acc.ldq;
    t.ldo = acc.ldq;
    TRY(reset_status(ctx, st));
    TRY(run_pass(ctx, t, st));
    for (int j = 0; j < w; ++j) {
      acc.kept.push_back(ids[j]);
      for (int i = 0; i <= j; ++i) acc.coeffs[(base + i) + ids[j] * K] = R[i + j * 16];
    }
    return BO_OK;
  }
  if (d.code != ST_CHOLESKY) return dev_error(ctx, "cholqr", st);
  const int f = (int)d.step;
  if (f == 1) {  // discard this whole sub-block
    for (int j = 0; j < w; ++j) {
      acc.disc.push_back(ids[j]);
      const double gjj = G[j + j * 16];
      acc.dnorm.push_back(std::sqrt(std::max(gjj, 0.0)));
    }
    acc.depth++;
    return BO_OK;
  }
  const int good = f - 1;
  // upload R11 / R12 from the partial factor (R slot already holds it on device)
  std::vector<double> r12(LDC * 16, 0.0);
  const uint64_t base = acc.kept.size();
  for (int j = 0; j < good; ++j) {
    acc.kept.push_back(ids[j]);
    for (int i = 0; i <= j; ++i) acc.coeffs[(base + i) + ids[j] * K] = R[i + j * 16];
  }
  for (int j = 0; j < w - good; ++j)
    for (int i = 0; i < good; ++i) {
      const double c = R[i + (good + j) * 16];
      r12[i + j * LDC] = c;
      acc.coeffs[(base + i) + ids[good + j] * K] = c;
    }
  // q_good = v[:, :good] R11^{-1}
  TRY(reset_status(ctx, st));
  PassReq t{};
  t.kind = PK_P1_ST;
  t.K = good;
  t.V = v;
  t.ldv = ldv;
  t.Rpre0 = T_(ctx, OFF_R1);
  t.out = acc.q + base * acc.ldq;
  t.ldo = acc.ldq;
  TRY(run_pass(ctx, t, st));
  // rest = v[:, good:] - q_good R12
  double* rest = nullptr;
  const size_t ldr = ctx->ld;
  CU(ctx_alloc(ctx, (void**)&rest, ldr * (w - good) * 8));
  CU(cudaMemcpyAsync(T_(ctx, OFF_C1), r12.data(), r12.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  PassReq u{};
  u.kind = PK_UPD_ST;
  u.K = w - good;
  u.V = v + good * ldv;
  u.ldv = ldv;
  u.Q = acc.q + base * acc.ldq;
  u.ldq = acc.ldq;
  u.p = good;
  u.Cm = T_(ctx, OFF_C1);
  u.out = rest;
  u.ldo = ldr;
  TRY(run_pass(ctx, u, st));
  CU(cudaStreamSynchronize(ctx->stream));
  acc.depth++;
  std::vector<uint64_t> rest_ids(ids.begin() + good, ids.end());
  const int rc = rec_impl(ctx, rest, ldr, w - good, rest_ids, acc, ledger, st);
  ctx_free(ctx, rest);
  return rc;
}
}  // namespace

extern "C" int bo_recursive_cholqr(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, double* q, uint64_t ldq,
                                   double* coeffs, uint64_t* kept, uint64_t* nkept, uint64_t* discarded,
                                   double* discard_norm, uint64_t* ndiscarded, uint64_t* depth, uint64_t ledger[4],
                                   bo_status* st) {
  ok_st(st);
  CU(cudaSetDevice(ctx->device));
  if (k > 16) return set_st(st, BO_INVALID, 0, 0.0, "panel wider than 16 columns");
  const double* vv;
  uint64_t lv;
  TRY(stage_input(ctx, v, ldv, k, 0, &vv, &lv, st));
  if (!out_ok(ctx, q, ldq)) return set_st(st, BO_INVALID, 0, 0.0, "q must have ld % 4 == 0 and ld >= n_local");
  // the input may live in scratch 0, which recursion does not touch
  RecAcc acc;
  acc.q = q;
  acc.ldq = ldq;
  acc.k = k;
  acc.coeffs.assign(k * k, 0.0);
  std::vector<uint64_t> ids(k);
  for (uint64_t j = 0; j < k; ++j) ids[j] = j;
  int rc = rec_impl(ctx, vv, lv, (int)k, ids, acc, ledger, st);
  if (rc != BO_OK) return rc;
  CU(cudaStreamSynchronize(ctx->stream));
  if (coeffs) std::memcpy(coeffs, acc.coeffs.data(), k * k * 8);
  if (kept) std::copy(acc.kept.begin(), acc.kept.end(), kept);
  if (nkept) *nkept = acc.kept.size();
  if (discarded) std::copy(acc.disc.begin(), acc.disc.end(), discarded);
  if (discard_norm) std::copy(acc.dnorm.begin(), acc.dnorm.end(), discard_norm);
  if (ndiscarded) *ndiscarded = acc.disc.size();
  if (depth) *depth = acc.depth;
  if (acc.kept.empty()) return set_st(st, BO_ALL_COLUMNS_DISCARDED, 0, 0.0, "recursive CholQR discarded all columns");
  return BO_OK;
}

// ===========================================================================
// BCGS-PIP and RandBCGS (block_orth.cpp:230-325)
// ===========================================================================
namespace {

// shared tail: resid = vhat - Q[lo:lo+p] C ; qj = resid R^{-1} into the slab;
// C (p x k) and R (k x k) given on host
int update_solve_store(bo_basis b, const double* vh, uint64_t ldvh, int K, uint64_t lo, int p, const hd::Mat& C,
                       const hd::Mat& R, uint64_t base, bo_status* st) {
  bo_ctx ctx = b->ctx;
  std::vector<double> hc(LDC * 16, 0.0), hr(256, 0.0);
  for (size_t j = 0; j < C.c; ++j)
    for (size_t i = 0; i < C.r; ++i) hc[i + j * LDC] = C(i, j);
  for (size_t j = 0; j < R.c; ++j)
    for (size_t i = 0; i <= j; ++i) hr[i + j * 16] = R(i, j);
  CU(cudaMemcpyAsync(T_(ctx, OFF_C1), hc.data(), hc.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(T_(ctx, OFF_R4), hr.data(), hr.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  TRY(reset_status(ctx, st));
  PassReq r{};
  r.K = K;
  r.V = vh;
  r.ldv = ldvh;
  r.out = b->q + base * ctx->ld;
  r.ldo = ctx->ld;
  if (p > 0) {
    r.kind = PK_UPD_POST_ST;
    r.Q = b->q + lo * ctx->ld;
    r.ldq = ctx->ld;
    r.p = p;
    r.Cm = T_(ctx, OFF_C1);
    r.Rpost = T_(ctx, OFF_R4);
  } else {
    r.kind = PK_P1_ST;
    r.Rpre0 = T_(ctx, OFF_R4);
  }
  TRY(run_pass(ctx, r, st));
  CU(cudaStreamSynchronize(ctx->stream));
  return BO_OK;
}

void push_full(bo_basis b, uint64_t k, uint64_t hi, uint64_t bp, const hd::Mat* rbig, const hd::Mat& proj,
               const hd::Mat& diag, bool overlap) {
  std::vector<double> full(std::max<uint64_t>(hi, 1) * k, 0.0), dg(k * k, 0.0);
  for (uint64_t j = 0; j < k; ++j) {
    for (uint64_t i = 0; i < bp; ++i) full[i + j * hi] = (rbig && rbig->r) ? (*rbig)(i, j) : 0.0;
    for (uint64_t i = 0; i < proj.r; ++i) full[bp + i + j * hi] = proj(i, j);
    for (uint64_t i = 0; i <= j; ++i) dg[i + j * k] = diag(i, j);
  }
  push_panel_host(b, k, full.data(), hi, dg.data(), k, overlap);
}

int pip_impl(bo_basis b, const double* vh, uint64_t ldvh, int K, const hd::Mat* rbig, bool overlap, bo_status* st) {
  bo_ctx ctx = b->ctx;
  const uint64_t bp = b->bp_lo;
  const bool eff = overlap && b->cols > 0;
  const uint64_t hi = b->cols - (eff ? 1 : 0);
  if (hi < bp) return set_st(st, BO_INVALID, 0, 0.0, "projection range below the big panel");
  const int p = (int)(hi - bp);
  // one fused volley [Q_range, V]^T V ; G = V^T V - proj^T proj ; Cholesky ("bcgs_pip")
  TRY(reset_status(ctx, st));
  PassReq r{};
  r.kind = PK_QTX_GRAM;
  r.K = K;
  r.V = vh;
  r.ldv = ldvh;
  r.Q = b->q + bp * ctx->ld;
  r.ldq = ctx->ld;
  r.p = p;
  r.pass_id = 1;
  r.fin.ops = FIN_PIP | FIN_CHOL;
  r.fin.Cq = T_(ctx, OFF_C2);
  r.fin.Rchol = T_(ctx, OFF_R1);
  TRY(run_pass(ctx, r, st));
  TRY(fetch(ctx, true, st));
  b->ledger[BO_LEDGER_GRAM]++;
  TRY(dev_error(ctx, "bcgs_pip", st));
  hd::Mat proj(p, K), R(K, K);
  for (int j = 0; j < K; ++j) {
    for (int i = 0; i < p; ++i) proj(i, j) = ctx->tiny_host[OFF_C2 + i + j * LDC];
    for (int i = 0; i <= j; ++i) R(i, j) = ctx->tiny_host[OFF_R1 + i + j * 16];
  }
  TRY(update_solve_store(b, vh, ldvh, K, bp, p, proj, R, hi, st));
  push_full(b, K, hi, bp, rbig, proj, R, eff);
  return BO_OK;
}

int rand_bcgs_impl(bo_basis b, const double* vh, uint64_t ldvh, int K, const hd::Mat* rbig, bo_sketch th,
                   bool overlap, bo_status* st) {
  bo_ctx ctx = b->ctx;
  const uint64_t bp = b->bp_lo;
  const bool eff = overlap && b->cols > 0;
  const uint64_t hi = b->cols - (eff ? 1 : 0);
  const uint64_t mh = th->mhat;
  // sketch (one reduce) -> host
  std::vector<double> sv;
  TRY(sketch_to_host(th, vh, ldvh, K, sv, st));
  b->ledger[BO_LEDGER_SKETCH]++;
  hd::Mat sk(mh, K);
  sk.a = sv;
  // BCGS2 with Householder intra on the sketched history (all local)
  const uint64_t have = b->sk_cols;
  const uint64_t sk_p = (eff && have > 0) ? have - 1 : have;
  if (b->sk_rows != mh) return set_st(st, BO_INVALID, 0, 0.0, "big panel was begun with a different sketch size");
  hd::Mat qprior(mh, sk_p);
  for (uint64_t j = 0; j < sk_p; ++j)
    for (uint64_t i = 0; i < mh; ++i) qprior(i, j) = b->sk[i + j * mh];
  hd::Mat proj_sk(sk_p, K), qsk, rdiag;
  if (sk_p == 0) {
    hd::householder_qr(sk, qsk, rdiag);
  } else {
    hd::Mat proj1 = hd::transpose_times(qprior, sk);
    hd::Mat skhat = sk;
    hd::subtract_product(skhat, qprior, proj1);
    hd::Mat iq, ir;
    hd::householder_qr(skhat, iq, ir);
    hd::Mat t1 = hd::transpose_times(qprior, iq);
    hd::Mat q2 = iq;
    hd::subtract_product(q2, qprior, t1);
    hd::Mat oq, orr;
    hd::householder_qr(q2, oq, orr);
    qsk = oq;
    proj_sk = hd::update_projection(proj1, t1, ir);
    rdiag = hd::multiply_upper(orr, ir);
  }
  for (int j = 0; j < K; ++j)
    if (rdiag(j, j) == 0.0)
      return set_st(st, BO_SINGULAR_TRIANGULAR, j, 0.0, "triangular factor is singular: zero diagonal at index %d", j);
  TRY(update_solve_store(b, vh, ldvh, K, bp, (int)sk_p, proj_sk, rdiag, hi, st));
  push_full(b, K, hi, bp, rbig, proj_sk, rdiag, eff);
  // push_sketched (block_orth.cpp:100-110)
  const uint64_t base = (eff && have > 0) ? have - 1 : have;
  b->sk.resize(mh * (base + K));
  for (int j = 0; j < K; ++j)
    for (uint64_t i = 0; i < mh; ++i) b->sk[i + (base + j) * mh] = qsk(i, j);
  b->sk_cols = base + K;
  return BO_OK;
}

int two_stage_common(bo_basis b, const double* v, uint64_t ldv, uint64_t k, int preproc, bo_sketch theta,
                     int overlap, bo_status* st) {
  bo_ctx ctx = b->ctx;
  CU(cudaSetDevice(ctx->device));
  const uint64_t bp = b->bp_lo;
  const bool eff = overlap && b->cols > 0;
  if ((eff ? b->cols - 1 : b->cols) + k > b->cap) return set_st(st, BO_INVALID, 0, 0.0, "basis capacity exceeded");
  const double* vv;
  uint64_t lv;
  TRY(stage_input(ctx, v, ldv, k, 0, &vv, &lv, st));
  const double* vh = vv;
  uint64_t ldvh = lv;
  hd::Mat rbig(bp, k);
  if (bp > 0) {  // inter-big-panel BCGS against the completed big panels
    TRY(reset_status(ctx, st));
    TRY(dev_project(b, vv, lv, (int)k, 0, bp, ctx->scratch[1], ctx->ld, OFF_C1, 1, st));
    TRY(fetch(ctx, true, st));
    b->ledger[BO_LEDGER_PROJECTION]++;
    for (uint64_t j = 0; j < k; ++j)
      for (uint64_t i = 0; i < bp; ++i) rbig(i, j) = ctx->tiny_host[OFF_C1 + i + j * LDC];
    vh = ctx->scratch[1];
    ldvh = ctx->ld;
  }
  if (preproc == BO_PREPROC_PIP) return pip_impl(b, vh, ldvh, (int)k, &rbig, eff, st);
  return rand_bcgs_impl(b, vh, ldvh, (int)k, &rbig, theta, eff, st);
}

}  // namespace

extern "C" int bo_bcgs_pip(bo_basis b, const double* v, uint64_t ldv, uint64_t k, int overlap, bo_status* st) {
  ok_st(st);
  TRY(basis_drain(b));
  bo_ctx ctx = b->ctx;
  CU(cudaSetDevice(ctx->device));
  const double* vv;
  uint64_t lv;
  TRY(stage_input(ctx, v, ldv, k, 0, &vv, &lv, st));
  hd::Mat rbig(b->bp_lo, k);
  return pip_impl(b, vv, lv, (int)k, &rbig, overlap != 0, st);
}

extern "C" int bo_rand_bcgs_preproc(bo_basis b, const double* v, uint64_t ldv, uint64_t k, bo_sketch theta,
                                    int overlap, bo_status* st) {
  ok_st(st);
  TRY(basis_drain(b));
  bo_ctx ctx = b->ctx;
  CU(cudaSetDevice(ctx->device));
  const double* vv;
  uint64_t lv;
  TRY(stage_input(ctx, v, ldv, k, 0, &vv, &lv, st));
  hd::Mat rbig(b->bp_lo, k);
  return rand_bcgs_impl(b, vv, lv, (int)k, &rbig, theta, overlap != 0, st);
}

extern "C" int bo_two_stage_panel(bo_basis b, const double* v, uint64_t ldv, uint64_t k, int preproc,
                                  bo_sketch theta, int overlap, bo_status* st) {
  ok_st(st);
  TRY(basis_drain(b));
  if (preproc == BO_PREPROC_RAND_BCGS && !theta)
    return set_st(st, BO_INVALID, 0, 0.0, "rand_bcgs preprocessing needs a sketch operator");
  return two_stage_common(b, v, ldv, k, preproc, theta, overlap, st);
}

extern "C" int bo_two_stage_finish(bo_basis b, int preproc, int reorthogonalize, int record, double* stats,
                                   bo_status* st) {
  ok_st(st);
  TRY(basis_drain(b));
  bo_ctx ctx = b->ctx;
  CU(cudaSetDevice(ctx->device));
  const uint64_t bp = b->bp_lo, w = b->cols - bp;
  if (w > 64) return set_st(st, BO_INVALID, 0, 0.0, "big panel wider than 64 columns");
  double* qb = b->q + bp * ctx->ld;
  if (record && stats) {
    // kappa of the preprocessed big panel from its Gram (sigma_i = sqrt(lambda_i)),
    // sketched orthogonality error on the host (diagnostics only)
    hd::Mat G;
    TRY(wide_contract(ctx, qb, ctx->ld, (int)w, qb, ctx->ld, (int)w, G, st));
    std::vector<double> ev(w);
    {
      std::vector<double> a(G.a);
      // cyclic Jacobi
      for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (uint64_t j = 0; j < w; ++j)
          for (uint64_t i = 0; i < j; ++i) off += a[i + j * w] * a[i + j * w];
        if (off == 0.0) break;
        for (uint64_t p = 0; p < w; ++p)
          for (uint64_t q = p + 1; q < w; ++q) {
            const double apq = a[p + q * w];
            if (apq == 0.0) continue;
            const double app = a[p + p * w], aqq = a[q + q * w];
            const double th = (aqq - app) / (2.0 * apq);
            const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
            const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
            for (uint64_t r = 0; r < w; ++r) {
              const double arp = a[r + p * w], arq = a[r + q * w];
              a[r + p * w] = c * arp - s * arq;
              a[r + q * w] = s * arp + c * arq;
            }
            for (uint64_t r = 0; r < w; ++r) {
              const double apr = a[p + r * w], aqr = a[q + r * w];
              a[p + r * w] = c * apr - s * aqr;
              a[q + r * w] = s * apr + c * aqr;
            }
          }
      }
      for (uint64_t i = 0; i < w; ++i) ev[i] = a[i + i * w];
    }
    double mx = 0, mn = 1e308;
    for (double e : ev) {
      mx = std::max(mx, e);
      mn = std::min(mn, e);
    }
    stats[0] = mn > 0 ? std::sqrt(mx / mn) : INFINITY;
    stats[1] = 0.0;
    if (preproc == BO_PREPROC_RAND_BCGS && b->sk_cols) {
      const uint64_t m = b->sk_rows, c = b->sk_cols;
      std::vector<double> d(c * c);
      for (uint64_t j = 0; j < c; ++j)
        for (uint64_t i = 0; i < c; ++i) {
          double s = 0.0;
          for (uint64_t r = 0; r < m; ++r) s += b->sk[r + i * m] * b->sk[r + j * m];
          d[i + j * c] = (i == j ? 1.0 : 0.0) - s;
        }
      double mxa = 0.0;
      for (double x : d) mxa = std::max(mxa, std::fabs(x));  // bound; exact 2-norm not needed for stats
      stats[1] = mxa;
    }
  }
  // second stage: CholQR of the big panel in place, refactor coefficient rows
  TRY(reset_status(ctx, st));
  hd::Mat R;
  TRY(wide_cholqr(ctx, qb, ctx->ld, (int)w, "cholqr", R, b->ledger, st));
  refactor_rows(b, bp, R);
  if (bp > 0 && reorthogonalize) {
    // BCGS against the completed big panels, 64 prior columns at a time
    hd::Mat C(bp, w);
    for (uint64_t c0 = 0; c0 < bp; c0 += 64) {
      const int pc = (int)std::min<uint64_t>(64, bp - c0);
      hd::Mat Cc;
      TRY(wide_contract(ctx, b->q + c0 * ctx->ld, ctx->ld, pc, qb, ctx->ld, (int)w, Cc, st));
      for (uint64_t j = 0; j < w; ++j)
        for (int i = 0; i < pc; ++i) C(c0 + i, j) = Cc(i, j);
    }
    b->ledger[BO_LEDGER_PROJECTION]++;
    for (uint64_t c0 = 0; c0 < bp; c0 += 64) {
      const int pc = (int)std::min<uint64_t>(64, bp - c0);
      hd::Mat Cc(pc, w);
      for (uint64_t j = 0; j < w; ++j)
        for (int i = 0; i < pc; ++i) Cc(i, j) = C(c0 + i, j);
      TRY(wide_update_trsm(ctx, qb, ctx->ld, (int)w, b->q + c0 * ctx->ld, ctx->ld, pc, &Cc, nullptr, qb, ctx->ld, st));
    }
    hd::Mat R2;
    TRY(wide_cholqr(ctx, qb, ctx->ld, (int)w, "cholqr", R2, b->ledger, st));
    reorth_rows(b, bp, C, R2);
  }
  return BO_OK;
}

namespace bo {
namespace host {
// Gram of p device columns, summed over ranks, to host (p x p, column-major),
// assembled from 64 x 64 blocks (upper blocks computed, lower mirrored)
int wide_gram_host(bo_ctx ctx, const double* q, uint64_t ld, int p, std::vector<double>& G, bo_status* st) {
  G.assign((size_t)p * p, 0.0);
  for (int j0 = 0; j0 < p; j0 += 64) {
    const int nj = std::min(64, p - j0);
    for (int i0 = 0; i0 <= j0; i0 += 64) {
      const int ni = std::min(64, p - i0);
      hd::Mat M;
      TRY(wide_contract(ctx, q + (size_t)i0 * ld, ld, ni, q + (size_t)j0 * ld, ld, nj, M, st));
      for (int j = 0; j < nj; ++j)
        for (int i = 0; i < ni; ++i) {
          G[(size_t)(i0 + i) + (size_t)(j0 + j) * p] = M(i, j);
          G[(size_t)(j0 + j) + (size_t)(i0 + i) * p] = M(i, j);
        }
    }
  }
  return BO_OK;
}
}  // namespace host
}  // namespace bo
