// bo_sketch_gen.cuh — device regeneration of the reference sketch streams.
//
// The reference fills its sketches from one std::mt19937_64 stream
// (proj/src/sketch.cpp:30-45, proj/include/blkorth/rng.hpp:22-64):
//   Gaussian  Theta(i,j) = scale * normal #(j*n + i)   (column-major fill,
//             Box-Muller pairs on draws 2t (uniform_open) and 2t+1 (uniform))
//   Count     row i: bucket = hi64(draw(2i) * width), sign = draw(2i+1) & 1.
// The stream is cut into chunks (about one per SM).  Each chunk starts from
// g[J+t] = XOR_{k in p} g[k+t], p = x^J mod phi (host-computed, mt64_jump.cpp),
// with the 20248-word stream prefix held in shared memory, then twists
// 312-word windows and tempers/transforms each word (mt_stream_kernel).
// Count (bucket, sign) is bit-identical to the reference; Gaussian values are
// the reference formula with correctly rounded log / sin / cos (bo_ddmath.cuh).
#pragma once
#include <cstdint>

#include "bo_ddmath.cuh"
#include "bo_ptx.cuh"
#include "bo_tiny.cuh"

namespace bo {

struct GenArgs {
  const uint64_t* prefix;     // 20248 untempered words
  const uint64_t* polys;      // nchunks x 312
  const uint64_t* chunk_J;    // first draw of each chunk (even)
  const uint64_t* chunk_len;  // draws per chunk (even)
  const uint16_t* jidx;       // set-bit indices of every chunk's jump polynomial
  const uint64_t* jidx_off;   // nchunks + 1 offsets into jidx
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

// One CTA per chunk of the stream (about one chunk per SM), 1024 threads.
//  1. Jump.  The 20248-word stream prefix g[0..) is staged in shared memory;
//     the chunk's first window is  w[t] = XOR_{k in K_c} g[k + t],  K_c the
//     set bits of x^J mod phi, given as a host-built list of bit indices.
//     Three 312-thread groups each XOR one third of the list; the partial
//     windows are combined through shared memory.
//  2. Generate.  Warps 27..31 (160 threads, one word each per half) twist
//     window after window into a ring of kRing shared-memory windows
//     (std::mt19937_64 order; each lane writes word t and word t + 156,
//     lane 155 recomputing new word 0, so one named barrier per window),
//     while warps 0..24, in 5 groups of 5, temper and
//     transform the 156 draw pairs of every 5th window (Box-Muller in FP64, or
//     the Count bucket/sign) and store them.  Full/empty mbarriers hand the
//     ring slots over; the FP64 transform is the bound.
constexpr int kRing = 16, kGenGroups = 5, kGenGroupWarps = 5, kGenProducer0 = 27, kGenProducerWarps = 5;

__device__ __forceinline__ void gen_transform(const GenArgs& a, const uint64_t* win, int pi, uint64_t q,
                                              uint64_t row, uint64_t col) {
  const uint64_t y0 = mt_temper(win[2 * pi]);
  const uint64_t y1 = mt_temper(win[2 * pi + 1]);
  if (a.kind == 0) {
    // rng.hpp:37-49 (normal #q = r cos, #q+1 = r sin)
    const double u1 = ((double)(y0 >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = (double)(y1 >> 11) * 0x1.0p-53;
    // correctly rounded log / sin / cos (bo_ddmath.cuh): the only differences
    // from the reference left are glibc's own misroundings (~0.1 % of inputs)
    const double rr = sqrt(tiny::mul(-2.0, ddm::log_cr(u1)));
    double sn, cs;
    ddm::sincos_bm_cr(u2, &sn, &cs);  // of ang = fl(2 pi u2), reduced through u2 (bo_ddmath.cuh)
    const double v0 = tiny::mul(a.scale, tiny::mul(rr, cs));
    const double v1 = tiny::mul(a.scale, tiny::mul(rr, sn));
    uint64_t c1 = col, r1 = row + 1;
    if (r1 == a.n_global) {
      r1 = 0;
      ++c1;
    }
    if ((int)col < a.mhat && row >= a.row_begin && row < a.row_end) a.theta[(row - a.row_begin) + col * a.ldth] = v0;
    if ((int)c1 < a.mhat && r1 >= a.row_begin && r1 < a.row_end) a.theta[(r1 - a.row_begin) + c1 * a.ldth] = v1;
  } else {
    // rng.hpp:52-58: bucket = hi64(u * width), sign = lsb
    const uint64_t r = q >> 1;
    if (r >= a.row_begin && r < a.row_end) {
      const uint64_t bucket = __umul64hi(y0, a.width);
      const uint32_t neg = (y1 & 1ULL) ? 0u : 0x80000000u;
      a.code[r - a.row_begin] = (uint32_t)bucket | neg;
    }
  }
}

__global__ void __launch_bounds__(1024, 1) mt_stream_kernel(const GenArgs a) {
  extern __shared__ __align__(16) uint64_t gsm[];
  uint64_t* pre = gsm;                          // kPrefixWords (jump only)
  uint64_t* ring = gsm + kPrefixWords + 8;      // kRing x 312
  uint64_t* bars = ring + kRing * kMtN;         // full[kRing], empty[kRing]
  uint64_t* full = bars;
  uint64_t* empty = bars + kRing;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = blockIdx.x;
  const uint64_t J = a.chunk_J[c], len = a.chunk_len[c];

  if (tid == 0) {
    for (int i = 0; i < kRing; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], kGenGroupWarps);
    }
    ptx::fence_mbar_init();
  }
  {
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(a.prefix);
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(pre);
    for (int i = tid; i < kPrefixWords / 2; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  // ---- 1. jump
  {
    const uint16_t* idx = a.jidx + a.jidx_off[c];
    const int L = (int)(a.jidx_off[c + 1] - a.jidx_off[c]);
    const int part = tid / kMtN, t = tid - part * kMtN;
    if (part < 3) {
      const int i0 = part * L / 3, i1 = (part + 1) * L / 3;
      const uint64_t* base = pre + t;
      uint64_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;
      int i = i0;
      for (; i + 4 <= i1; i += 4) {
        w0 ^= base[__ldg(idx + i)];
        w1 ^= base[__ldg(idx + i + 1)];
        w2 ^= base[__ldg(idx + i + 2)];
        w3 ^= base[__ldg(idx + i + 3)];
      }
      for (; i < i1; ++i) w0 ^= base[__ldg(idx + i)];
      ring[(1 + part) * kMtN + t] = w0 ^ w1 ^ w2 ^ w3;
    }
    __syncthreads();
    if (tid < kMtN) ring[tid] = ring[kMtN + tid] ^ ring[2 * kMtN + tid] ^ ring[3 * kMtN + tid];
    __syncthreads();
  }
  const uint64_t nwin = (len + kMtN - 1) / kMtN;
  // ---- 2. generate
  if (warp >= kGenProducer0) {
    const int pt = tid - kGenProducer0 * 32;  // 0..159
    if (pt == 0) ptx::mbar_arrive(&full[0]);
    for (uint64_t w = 1; w < nwin; ++w) {
      const int slot = (int)(w % kRing);
      if (w >= kRing) ptx::mbar_wait(&empty[slot], (uint32_t)((w / kRing - 1) & 1));
      const uint64_t* cur = ring + ((w - 1) % kRing) * kMtN;
      uint64_t* nxt = ring + slot * kMtN;
      if (pt < kMtM) {
        // word pt of the new window (mt19937_64 first half), then word
        // pt + 156, which needs new word pt (this lane's) and, for the last
        // word, new word 0: lane 155 recomputes it from the old window, so
        // one barrier per window suffices (the next window reads this one)
        const uint64_t lo = cur[pt + kMtM] ^ mt_f(cur[pt], cur[pt + 1]);
        nxt[pt] = lo;
        const uint64_t nx = pt + 1 < kMtM ? cur[pt + kMtM + 1] : (cur[kMtM] ^ mt_f(cur[0], cur[1]));
        nxt[pt + kMtM] = lo ^ mt_f(cur[pt + kMtM], nx);
      }
      ptx::named_bar_sync(1, kGenProducerWarps * 32);
      if (pt == 0) ptx::mbar_arrive(&full[slot]);
    }
  } else if (warp < kGenGroups * kGenGroupWarps) {
    const int grp = warp / kGenGroupWarps, wi = warp - grp * kGenGroupWarps;
    const int pi = wi * 32 + lane;  // draw pair within the window (valid < 156)
    const uint64_t n = a.n_global;
    uint64_t q = J + (uint64_t)grp * kMtN + 2 * (uint64_t)pi;
    uint64_t col = 0, row = 0;
    if (a.kind == 0) {
      col = q / n;
      row = q - col * n;
    }
    constexpr uint64_t kStep = (uint64_t)kGenGroups * kMtN;
    for (uint64_t w = grp; w < nwin; w += kGenGroups) {
      const int slot = (int)(w % kRing);
      ptx::mbar_wait(&full[slot], (uint32_t)((w / kRing) & 1));
      if (pi < kMtM && w * kMtN + 2 * (uint64_t)pi < len) gen_transform(a, ring + slot * kMtN, pi, q, row, col);
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[slot]);
      q += kStep;
      if (a.kind == 0) {
        row += kStep;
        while (row >= n) {
          row -= n;
          ++col;
        }
      }
    }
  }
}

}  // namespace bo
