// Probe: does compute-sanitizer racecheck model mbarrier hand-offs?
// Warp 0 writes a shared buffer, then arrives on an mbarrier (arrive has
// .release.cta semantics); warp 1 waits on the barrier phase (try_wait has
// .acquire.cta semantics) and then reads the buffer.  The program is race free
// by the PTX memory model; if racecheck reports a hazard here, its reports on
// the pass engine's solved / full / empty mbarrier hand-offs
// (bo_pass.cuh:620 -> :677 / :754) are the same tool limitation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2503_16717_b200/csrc \
//        scripts/probes/racecheck_mbarrier.cu -o build/racecheck_mbarrier
//   compute-sanitizer --tool racecheck build/racecheck_mbarrier
#include <cstdio>
#include <cstdint>

#include "bo_ptx.cuh"

__global__ void probe(double* out) {
  __shared__ double buf[32];
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    bo::ptx::mbar_init(&bar, 1);
    bo::ptx::fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    buf[lane] = 1.0 + lane;
    __syncwarp();
    if (lane == 0) bo::ptx::mbar_arrive(&bar);
  } else {
    bo::ptx::mbar_wait(&bar, 0);
    out[lane] = buf[lane];
  }
}

int main() {
  double* d;
  cudaMalloc(&d, 32 * sizeof(double));
  probe<<<1, 64>>>(d);
  double h[32];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("probe %s (h[31] = %g)\n", cudaGetLastError() == cudaSuccess ? "ran" : "failed", h[31]);
  return 0;
}
