// cpp_gmres.cpp — C++ host code driving the GPU path through the C ABI via the
// blkorth::gpu adapter: config 1 of BASELINE.json (2D 5-point Laplacian 100^2,
// s = 5, m = 60, b = 1, x0 = 0) with the chosen scheme, plus one standalone
// bcgs2 call on the Krylov panel.  Prints restarts / iterations / ledger.
//   usage: cpp_gmres [scheme 0..3] [k=100] [s=5]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "blkorth_gpu.hpp"

int main(int argc, char** argv) {
  const int scheme = argc > 1 ? std::atoi(argv[1]) : BO_BCGS2_CHOLQR2;
  const uint64_t k = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 100;
  const uint64_t s = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 5;
  const uint64_t n = k * k;
  try {
    blkorth::gpu::Context ctx(n);
    auto A = blkorth::gpu::Operator::laplace(ctx, 2, k);
    double *b = nullptr, *x0 = nullptr, *x = nullptr;
    cudaMalloc(&b, n * 8);
    cudaMalloc(&x0, n * 8);
    cudaMalloc(&x, n * 8);
    std::vector<double> ones(n, 1.0);
    cudaMemcpy(b, ones.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemset(x0, 0, n * 8);
    // the pageable upload may still be in flight, and the context's private
    // non-blocking stream does not wait for the legacy stream
    cudaDeviceSynchronize();
    bo_solver_config cfg{};
    cfg.n = n;
    cfg.m = 60;
    cfg.s = s;
    cfg.shat = 60;
    cfg.scheme = scheme;
    cfg.sketch = BO_SKETCH_GAUSSIAN;
    cfg.rel_tol = 1e-6;
    cfg.max_restarts = 50;
    cfg.seed = 0;
    cfg.reorthogonalize = 1;
    cfg.diagnostics = 1;
    const bo_solve_report rep = blkorth::gpu::sstep_gmres_solve(A, b, x0, cfg, x);
    std::printf("scheme %d: converged=%d breakdown=%d restarts=%llu iterations=%llu final_relres=%.17g ledger=%llu/%llu/%llu/%llu total=%llu\n",
                scheme, rep.converged, rep.breakdown, (unsigned long long)rep.restarts,
                (unsigned long long)rep.iterations, rep.final_relres, (unsigned long long)rep.reduce[0],
                (unsigned long long)rep.reduce[1], (unsigned long long)rep.reduce[2], (unsigned long long)rep.reduce[3],
                (unsigned long long)rep.reduce_total);
    if (rep.breakdown) std::printf("detail: %s\n", rep.breakdown_detail);
    // one bcgs2 on a Krylov panel [b, Ab, ..., A^s b]
    blkorth::gpu::BasisStore store(ctx, s + 1);
    double* panel = nullptr;
    const uint64_t ld = ctx.ld();
    cudaMalloc(&panel, ld * (s + 1) * 8);
    A.mpk(b, s, {panel, ld, s + 1});
    blkorth::gpu::bcgs2(store, {panel, ld, s + 1}, blkorth::gpu::IntraKind::cholqr2);
    std::printf("bcgs2 on the Krylov panel: cols=%llu R00=%.17g ledger_total=%llu\n",
                (unsigned long long)store.cols(), store.r_entry(0, 0), (unsigned long long)store.ledger().total());
    cudaFree(panel);
    cudaFree(b);
    cudaFree(x0);
    cudaFree(x);
  } catch (const blkorth::gpu::Error& e) {
    std::printf("error: %s\n", e.what());
    return 1;
  }
  return 0;
}
