// gpu_bcgs2.cpp — the reference's bcgs2 (proj/include/blkorth/block_orth.hpp:123,
// proj/src/block_orth.cpp:207-226) on the GPU, for the UNMODIFIED reference
// GMRES driver.  A maintainer switches sstep_gmres_solve (gmres.cpp:405-436)
// to the GPU by compiling gmres.cpp with -Dbcgs2=gpu_bcgs2 and linking this
// file plus libbo_cuda.so; nothing else in the reference changes (oracle/Makefile
// target `refgpu` is that build, INTEGRATION.md §3 the recipe).
//
// Same signature and contract as blkorth::bcgs2:
//   * the panel V (host DenseMatrix, the driver's mpk output) is uploaded and
//     orthogonalised by bo_bcgs2 against a device mirror of the store;
//   * on success the panel is pushed into the caller's host BasisStore with the
//     reference's own push_panel, from exactly the (proj, diag) the device run
//     pushed (bo_basis_last_push), so the host R / C / boundaries are the
//     reference's arithmetic on the GPU's coefficients; the store ledger gets
//     the same events;
//   * failures are rethrown as the reference exception types (blkorth_gpu.hpp
//     in BLKORTH_GPU_REFERENCE_TYPES mode), so the driver's
//     `catch (const Error& e)` routes a CholeskyBreakdown into recover_panel,
//     which then runs on the host store; the mirror re-imports that store on
//     the next call.
// Gaussian sketches are bridged bit-for-bit from the host operator's dense
// stage (bo_sketch_from_dense); Count-based sketches keep the CPU path.
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "blkorth/block_orth.hpp"
#include "blkorth/dense.hpp"
#include "blkorth/errors.hpp"
#include "blkorth/sketch.hpp"
#define BLKORTH_GPU_REFERENCE_TYPES
#include "blkorth_gpu.hpp"

namespace blkorth {

namespace {

struct Mirror {
  bo_ctx ctx = nullptr;
  cudaStream_t stream = nullptr;  // the context's stream: uploads are ordered before its passes
  uint64_t n = 0, ld = 0;
  bo_basis b = nullptr;
  uint64_t cap = 0;
  const BasisStore* owner = nullptr;
  double* panel = nullptr;  // device, ld x 16
  double* theta_dev = nullptr;
  uint64_t theta_cols = 0;
  bo_sketch sk = nullptr;
  const double* sk_key = nullptr;  // host dense stage the device sketch was built from
  double sk_first = 0.0, sk_last = 0.0;
};
Mirror g;  // one host thread per store (block_orth.hpp:25-26); intentionally not torn down at exit

void ok(int rc, const bo_status& st) { gpu::check(rc, st); }

void cuda_ok(cudaError_t e) {
  if (e != cudaSuccess) throw gpu::DeviceError(std::string("gpu_bcgs2: ") + cudaGetErrorString(e));
}

void ensure_ctx(uint64_t n) {
  if (g.ctx && g.n == n) return;
  if (g.sk) bo_sketch_destroy(g.sk);
  if (g.b) bo_basis_destroy(g.b);
  if (g.panel) cudaFree(g.panel);
  if (g.theta_dev) cudaFree(g.theta_dev);
  if (g.ctx) bo_ctx_destroy(g.ctx);
  if (g.stream) cudaStreamDestroy(g.stream);
  g = Mirror{};
  bo_status st{};
  // A pageable cudaMemcpy may return before its DMA lands, and a non-blocking
  // library stream is not ordered after the legacy stream: every upload goes
  // on the context's own stream instead.
  cuda_ok(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
  ok(bo_ctx_create(0, 0, 1, nullptr, n, 0, n, g.stream, &g.ctx, &st), st);
  g.n = n;
  g.ld = bo_ctx_ld(g.ctx);
  cuda_ok(cudaMalloc((void**)&g.panel, g.ld * 16 * sizeof(double)));
}

// bring the device mirror to the host store's state (after host-side pushes:
// recover_panel, or a new store)
void sync_store(const BasisStore& s) {
  bo_status st{};
  if (!g.b || g.cap != s.capacity()) {
    if (g.b) bo_basis_destroy(g.b);
    ok(bo_basis_create(g.ctx, s.capacity(), &g.b, &st), st);
    g.cap = s.capacity();
    g.owner = nullptr;
  }
  const uint64_t cols = s.cols();
  if (g.owner != &s || bo_basis_cols(g.b) != cols) {
    const DenseMatrix q = s.basis_copy();
    std::vector<double> r(cols * cols, 0.0), c(cols * cols, 0.0);
    std::vector<unsigned char> seeded(cols, 0);
    for (uint64_t j = 0; j < cols; ++j) {
      for (uint64_t i = 0; i <= j; ++i) r[i + j * cols] = s.r_entry(i, j);
      if (s.is_seed(j)) {
        seeded[j] = 1;
        const std::vector<double> cj = s.input_coeff_col(j, cols);
        for (uint64_t i = 0; i < cols; ++i) c[i + j * cols] = cj[i];
      }
    }
    const std::vector<std::size_t>& bd = s.panel_boundaries();
    std::vector<uint64_t> bounds(bd.begin(), bd.end());
    ok(bo_basis_import(g.b, cols, q.data(), g.n, r.data(), c.data(), seeded.data(), bounds.data(), bounds.size(),
                       &st),
       st);
    g.owner = &s;
  }
  for (uint64_t j = 0; j < cols; ++j)  // the driver's mark_seed (gmres.cpp:410-411)
    if (s.is_seed(j) && !bo_basis_is_seed(g.b, j)) bo_basis_mark_seed(g.b, j);
}

bo_sketch device_sketch(const SketchOperator* theta) {
  if (!theta) return nullptr;
  if (theta->kind() != SketchKind::gaussian)
    throw InvalidScheme("gpu_bcgs2: only Gaussian sketches are bridged to the device");
  const DenseMatrix& d = theta->dense_stage();
  const uint64_t mh = theta->sketch_size();
  if (g.sk && g.sk_key == d.data() && g.sk_first == d.data()[0] && g.sk_last == d.data()[g.n * mh - 1]) return g.sk;
  if (g.sk) bo_sketch_destroy(g.sk);
  g.sk = nullptr;
  if (g.theta_cols < mh) {
    if (g.theta_dev) cudaFree(g.theta_dev);
    cuda_ok(cudaMalloc((void**)&g.theta_dev, g.ld * mh * sizeof(double)));
    g.theta_cols = mh;
  }
  cuda_ok(cudaMemcpy2DAsync(g.theta_dev, g.ld * 8, d.data(), g.n * 8, g.n * 8, mh, cudaMemcpyHostToDevice, g.stream));
  bo_status st{};
  ok(bo_sketch_from_dense(g.ctx, g.theta_dev, g.ld, mh, &g.sk, &st), st);
  g.sk_key = d.data();
  g.sk_first = d.data()[0];
  g.sk_last = d.data()[g.n * mh - 1];
  return g.sk;
}

}  // namespace

void gpu_bcgs2(BasisStore& store, const DenseMatrix& v, IntraKind intra, const SketchOperator* theta, bool overlap) {
  const uint64_t n = store.ambient_dim(), k = v.cols();
  if (k > 16) throw InvalidScheme("gpu_bcgs2: panels wider than 16 columns");
  ensure_ctx(n);
  sync_store(store);
  bo_sketch sk = device_sketch(theta);
  cuda_ok(cudaMemcpy2DAsync(g.panel, g.ld * 8, v.data(), n * 8, n * 8, k, cudaMemcpyHostToDevice, g.stream));
  uint64_t led0[4], led1[4];
  bo_basis_ledger(g.b, led0);
  bo_status st{};
  const int rc = bo_bcgs2(g.b, g.panel, g.ld, k, intra == IntraKind::cholqr2 ? BO_INTRA_CHOLQR2 : BO_INTRA_RAND_CHOLQR,
                          sk, overlap ? 1 : 0, &st);
  bo_basis_ledger(g.b, led1);
  for (int p = 0; p < 4; ++p)  // the reduce events of the call, failed or not (block_orth.cpp records as it goes)
    for (uint64_t e = led0[p]; e < led1[p]; ++e) store.ledger().record((ReducePhase)p);
  ok(rc, st);
  // replay the device push on the host store with the reference's push_panel
  uint64_t base = 0, kk = 0;
  int ov = 0;
  bo_basis_last_push(g.b, &base, &kk, &ov, nullptr, nullptr);
  std::vector<double> proj(base * kk), diag(kk * kk);
  bo_basis_last_push(g.b, nullptr, nullptr, nullptr, proj.data(), diag.data());
  DenseMatrix qblock(n, kk), pm(base, kk);
  ok(bo_basis_cols_to_host(g.b, base, base + kk, qblock.data(), &st), st);
  for (uint64_t j = 0; j < kk; ++j)
    for (uint64_t i = 0; i < base; ++i) pm(i, j) = proj[i + j * base];
  UpperTriangular dg(kk);
  for (uint64_t j = 0; j < kk; ++j)
    for (uint64_t i = 0; i <= j; ++i) dg.at(i, j) = diag[i + j * kk];
  store.push_panel(qblock, pm, dg, ov != 0);
  g.owner = &store;
}

}  // namespace blkorth
