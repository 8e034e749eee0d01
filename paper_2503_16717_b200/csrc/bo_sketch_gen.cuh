// bo_sketch_gen.cuh — device regeneration of the reference sketch streams.
//
// The reference fills its sketches from one std::mt19937_64 stream
// (proj/src/sketch.cpp:30-45, proj/include/blkorth/rng.hpp:22-64):
//   Gaussian  Theta(i,j) = scale * normal #(j*n + i)   (column-major fill,
//             Box-Muller pairs on draws 2t (uniform_open) and 2t+1 (uniform))
//   Count     row i: bucket = hi64(draw(2i) * width), sign = draw(2i+1) & 1.
// Each CTA owns one chunk of the stream.  It jumps to the chunk start with
// g[J+t] = XOR_{k in p} g[k+t], p = x^J mod phi (host-computed, mt64_jump.cpp),
// using the 20248-word stream prefix held in shared memory, then twists the
// 312-word window in three parallel phases and tempers/transforms each word.
// Count (bucket, sign) is bit-identical to the reference; Gaussian values use
// the device libm log/sin/cos (<= 1-2 ulp from glibc's).
#pragma once
#include <cstdint>

#include "bo_tiny.cuh"

namespace bo {

struct GenArgs {
  const uint64_t* prefix;     // 20248 untempered words
  const uint64_t* polys;      // nchunks x 312
  const uint64_t* chunk_J;    // first draw of each chunk (even)
  const uint64_t* chunk_len;  // draws per chunk (even)
  int kind;                   // 0 gaussian, 1 count
  uint64_t n_global, row_begin, row_end;
  uint64_t width;             // count buckets
  int mhat;                   // gaussian columns
  double scale;               // 1/sqrt(mhat)
  double* theta;              // local gaussian rows, ld
  uint64_t ldth;
  uint32_t* code;             // local count codes: bucket | sign bit (1 = -1)
};

constexpr int kMtN = 312, kMtM = 156, kPrefixWords = 19937 + 311, kPolyWords = 312;

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}
__device__ __forceinline__ uint64_t mt_f(uint64_t hi_src, uint64_t lo_src) {
  const uint64_t x = (hi_src & 0xFFFFFFFF80000000ULL) | (lo_src & 0x7FFFFFFFULL);
  uint64_t xa = x >> 1;
  if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
  return xa;
}

__global__ void __launch_bounds__(320, 1) sketch_gen_kernel(const GenArgs a) {
  extern __shared__ __align__(16) uint64_t gsm[];
  uint64_t* pre = gsm;                       // kPrefixWords
  uint64_t* cur = gsm + kPrefixWords + 8;    // 312
  uint64_t* nxt = cur + kMtN;                // 312
  const int tid = threadIdx.x, nth = blockDim.x;
  const int c = blockIdx.x;
  for (int i = tid; i < kPrefixWords; i += nth) pre[i] = a.prefix[i];
  __syncthreads();
  // jump: window g[J .. J+311]
  if (tid < kMtN) {
    const uint64_t* poly = a.polys + (size_t)c * kPolyWords;
    uint64_t w = 0;
    for (int pw = 0; pw < kPolyWords; ++pw) {
      uint64_t bits = __ldg(poly + pw);
      while (bits) {
        const int b = __ffsll((long long)bits) - 1;
        bits &= bits - 1;
        w ^= pre[pw * 64 + b + tid];
      }
    }
    cur[tid] = w;
  }
  __syncthreads();
  const uint64_t J = a.chunk_J[c], len = a.chunk_len[c];
  for (uint64_t base = 0; base < len; base += kMtN) {
    // transform pairs of this 312-word block
    if (tid < kMtN / 2) {
      const uint64_t off = base + 2 * (uint64_t)tid;
      if (off < len) {
        const uint64_t d0 = J + off;  // even draw index
        const uint64_t y0 = mt_temper(cur[2 * tid]);
        const uint64_t y1 = mt_temper(cur[2 * tid + 1]);
        if (a.kind == 0) {
          // rng.hpp:37-49 (normal #d0 = r cos, #d0+1 = r sin)
          const double u1 = ((double)(y0 >> 11) + 1.0) * 0x1.0p-53;
          const double u2 = (double)(y1 >> 11) * 0x1.0p-53;
          const double rr = sqrt(tiny::mul(-2.0, log(u1)));
          const double ang = tiny::mul(6.283185307179586476925286766559, u2);
          double sn, cs;
          sincos(ang, &sn, &cs);
          const double v[2] = {tiny::mul(rr, cs), tiny::mul(rr, sn)};
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const uint64_t q = d0 + e;
            const uint64_t col = q / a.n_global, row = q - col * a.n_global;
            if ((int)col < a.mhat && row >= a.row_begin && row < a.row_end)
              a.theta[(row - a.row_begin) + col * a.ldth] = tiny::mul(a.scale, v[e]);
          }
        } else {
          // rng.hpp:52-58: bucket = hi64(u * width), sign = lsb
          const uint64_t row = d0 >> 1;
          if (row >= a.row_begin && row < a.row_end) {
            const uint64_t bucket = __umul64hi(y0, a.width);
            const uint32_t neg = (y1 & 1ULL) ? 0u : 0x80000000u;
            a.code[row - a.row_begin] = (uint32_t)bucket | neg;
          }
        }
      }
    }
    if (base + kMtN >= len) break;
    // twist the window: g[J+312+i] (std::mt19937_64 in-place order)
    if (tid < kMtM) nxt[tid] = cur[tid + kMtM] ^ mt_f(cur[tid], cur[tid + 1]);
    __syncthreads();
    if (tid >= kMtM && tid < kMtN - 1) nxt[tid] = nxt[tid - kMtM] ^ mt_f(cur[tid], cur[tid + 1]);
    __syncthreads();
    if (tid == kMtN - 1) nxt[tid] = nxt[tid - kMtM] ^ mt_f(cur[tid], nxt[0]);
    __syncthreads();
    if (tid < kMtN) cur[tid] = nxt[tid];
    __syncthreads();
  }
}

}  // namespace bo
