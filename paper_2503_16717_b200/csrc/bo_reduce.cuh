// bo_reduce.cuh — deterministic cross-CTA reduction of per-CTA partial sums.
//
// Every CTA writes its partial vector (len doubles) to partials[blockIdx.x].
// CTAs are grouped in fixed groups of kRedGroup; the last CTA of a group to
// arrive sums the group's partials in CTA order into the group's first slot,
// and the last group to finish sums the group results in group order into
// `sums`.  The summation tree depends only on the grid size, so results are
// bitwise reproducible; the critical path after the slowest CTA is two short
// rounds of L2 loads (instead of one CTA reading all grid x len partials).
// counters: 1 + ceil(grid / kRedGroup) words, zero on entry, zero on exit.
#pragma once

namespace bo {

constexpr int kRedGroup = 8;
constexpr int kMaxRedCounters = 64;

// returns true in the single CTA that holds the final sums (callers then run
// their finalize); all threads of the CTA must call it
__device__ __forceinline__ bool cta_tree_reduce(double* partials, int len, double* sums, unsigned* counters) {
  __shared__ int s_flag;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int grid = (int)gridDim.x, b = (int)blockIdx.x;
  const int grp = b / kRedGroup, g0 = grp * kRedGroup;
  const int gsz = min(kRedGroup, grid - g0);
  const int ngroups = (grid + kRedGroup - 1) / kRedGroup;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_flag = (atomicAdd(&counters[1 + grp], 1u) == (unsigned)(gsz - 1));
  __syncthreads();
  if (!s_flag) return false;
  __threadfence();
  for (int e = tid; e < len; e += nth) {
    double v[kRedGroup];
#pragma unroll
    for (int q = 0; q < kRedGroup; ++q) v[q] = q < gsz ? __ldcg(partials + (size_t)(g0 + q) * len + e) : 0.0;
    double s = v[0];
#pragma unroll
    for (int q = 1; q < kRedGroup; ++q)
      if (q < gsz) s += v[q];
    partials[(size_t)g0 * len + e] = s;
  }
  if (tid == 0) counters[1 + grp] = 0u;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_flag = (atomicAdd(&counters[0], 1u) == (unsigned)(ngroups - 1));
  __syncthreads();
  if (!s_flag) return false;
  __threadfence();
  for (int e = tid; e < len; e += nth) {
    double s = 0.0;
    int q = 0;
    for (; q + 8 <= ngroups; q += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(partials + (size_t)(q + u) * kRedGroup * len + e);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; q < ngroups; ++q) s += __ldcg(partials + (size_t)q * kRedGroup * len + e);
    sums[e] = s;
  }
  if (tid == 0) counters[0] = 0u;
  __threadfence();
  __syncthreads();
  return true;
}

}  // namespace bo
