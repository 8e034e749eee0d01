// FP64 latency / single-warp throughput probe: dependent DFMA and DMMA chains,
// and independent chains (ILP) from one warp per SM sub-partition.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_lat.cu -o fp64_lat
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_chain(double* out, int iters, double a, double b) {
  double x[ILP];
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += x[i];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1 << 20] = (double)(t1 - t0) / iters;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int ILP>
__global__ void dmma_chain(double* out, int iters, double a, double b) {
  double d[ILP][2];
  for (int i = 0; i < ILP; ++i) d[i][0] = d[i][1] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) dmma(d[i][0], d[i][1], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += d[i][0] + d[i][1];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1 << 20] = (double)(t1 - t0) / iters;
}

template <typename F>
void run(const char* nm, F f, int warps, int ilp, double* d) {
  const int iters = 4096;
  f<<<1, 32 * warps>>>(d, iters, 1.0000001, 1e-9);
  cudaDeviceSynchronize();
  f<<<1, 32 * warps>>>(d, iters, 1.0000001, 1e-9);
  double cyc;
  cudaMemcpy(&cyc, d + (1 << 20), 8, cudaMemcpyDeviceToHost);
  printf("%-6s warps/CTA %2d ILP %2d: %7.2f cycles per iteration (%6.2f per instr per warp)\n", nm, warps, ilp, cyc,
         cyc / ilp);
}

int main() {
  double* d;
  cudaMalloc(&d, ((1 << 20) + 8) * 8);
  for (int w : {1, 4, 8}) {
    run("DFMA", dfma_chain<1>, w, 1, d);
    run("DFMA", dfma_chain<4>, w, 4, d);
    run("DFMA", dfma_chain<8>, w, 8, d);
    run("DFMA", dfma_chain<16>, w, 16, d);
    run("DMMA", dmma_chain<1>, w, 1, d);
    run("DMMA", dmma_chain<2>, w, 2, d);
    run("DMMA", dmma_chain<4>, w, 4, d);
    run("DMMA", dmma_chain<8>, w, 8, d);
    run("DMMA", dmma_chain<14>, w, 14, d);
  }
  return 0;
}
