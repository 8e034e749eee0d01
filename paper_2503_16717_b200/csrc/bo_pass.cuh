// bo_pass.cuh — the streaming pass engine.
//
// One persistent CTA per SM walks tiles of T local rows.  A producer warp
// stages every column segment the pass needs (panel V, projection range of
// the basis Q, Gaussian sketch rows, Count sketch codes) into a ring of
// shared-memory stages with bulk async copies (TMA engine) tracked by
// mbarriers.  Eight consumer warps then, per tile:
//   A  row-parallel triangular solves  X = V R_a^{-1} R_b^{-1}   (NPRE)
//   U  tensor-core update              X = X - Q C               (UPD, DMMA)
//   A' row-parallel triangular solve   X = X R^{-1}              (NPOST)
//   S  bulk async store of X to HBM                              (STORE)
//   R  tensor-core contractions Q^T X, X^T X, Theta^T X (DMMA) and the
//      deterministic Count-sketch scatter (QTX, GRAM, SK)
// Partial sums are reduced across warps, then across CTAs in fixed order by
// the last CTA to finish, which also runs the tiny factorization of the pass
// (bo_tiny.cuh) on one GPU.  Every HBM byte of the pass is read exactly once.
//
// Reference operations fused here (proj/src/dense.cpp): transpose_times :28,
// subtract_product :60, gram :10, apply_inv_upper :166, plus the sketch
// application proj/src/sketch.cpp:110-126.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "bo_common.cuh"
#include "bo_ptx.cuh"
#include "bo_reduce.cuh"

#ifndef BO_GAW
#define BO_GAW 2  // row-solve warps of pre-solve passes; 0: NW - 4 (see pass_kernel)
#endif
#ifndef BO_GAW_QTX
#define BO_GAW_QTX BO_GAW  // ... of the pre-solve projection passes (P2_QTX)
#endif
#ifndef BO_GAW_UPD
#define BO_GAW_UPD BO_GAW  // ... of the pre-solve update passes (P2_UPD_*)
#endif
#include "bo_tiny.cuh"

// Phase profiler (diagnostic builds only): lane 0 of every consumer warp
// accumulates clock64() cycles per phase and adds them to
// a.phase_prof[shape * 16 + phase] at exit (shape = NPRE * 4 + UPD * 2 + QTX).
#ifndef BO_PHASE_PROF
#define BO_PHASE_PROF 0
#endif
#ifndef BO_STORE_SPREAD
#define BO_STORE_SPREAD 1
#endif
// Tail columns on FP64 FMAs (see TN in pass_kernel), per site: the projection
// contraction Q^T X when it has at least BO_TAIL_QTX_MIN 8-column Q tiles, the
// update X - QC with at least BO_TAIL_UPD_MIN, the Gram X^T X.  0: DMMA.
#ifndef BO_DFMA_TAIL
#define BO_DFMA_TAIL 1
#endif
#ifndef BO_TAIL_QTX
#define BO_TAIL_QTX 1
#endif
#ifndef BO_TAIL_QTX_MIN
#define BO_TAIL_QTX_MIN 4
#endif
#ifndef BO_TAIL_UPD
#define BO_TAIL_UPD 0
#endif
#ifndef BO_TAIL_UPD_MIN
#define BO_TAIL_UPD_MIN 4
#endif
#ifndef BO_TAIL_GRAM
#define BO_TAIL_GRAM 0
#endif
// Pre-solve passes with a projection range: separate panel (V) and basis (Q)
// rings, the panel ring deeper (see DEC in pass_kernel); 0: one ring of joint stages
#ifndef BO_ROWG_RQ_WIDE
#define BO_ROWG_RQ_WIDE 2  // rows per thread per step of the row-mode Gram at K > 8 (1: 139 -> 2: 131 us at K = 11)
#endif
#ifndef BO_DEC_RING
#define BO_DEC_RING 1
#endif
#if BO_PHASE_PROF
#define PP_T0() long long pp_t = clock64()
#define PP_MARK(i)                      \
  do {                                  \
    const long long pp_n = clock64();   \
    pp_acc[i] += pp_n - pp_t;           \
    pp_t = pp_n;                        \
  } while (0)
#else
#define PP_T0() (void)0
#define PP_MARK(i) (void)0
#endif

namespace bo {


// ---------------------------------------------------------------------------
// finalize (one CTA): the tiny factorizations after a reduction
// ---------------------------------------------------------------------------
static __device__ void finalize_dev(const FinArgs& f, double* smem_scratch /* >= 7*256 + 32*16 doubles */) {
  // Every factor lives in shared memory while it is computed; global memory is
  // read once at the start (sums, input factors, coefficient blocks) and
  // written once at the end.
  const int tid = threadIdx.x, nth = blockDim.x;
  __shared__ int s_code;
  __shared__ int s_fail;
  __shared__ double s_piv;
  if (tid == 0) s_code = f.status->code;
  __syncthreads();
  if (s_code != ST_OK) return;
  const double* sums = f.sums;
  double* G = smem_scratch;             // 16 x 16
  double* sb = smem_scratch + 256;      // 16 x 16 scratch (Householder tau)
  double* Rc = smem_scratch + 512;      // Cholesky factor 16 x 16
  double* Rn = smem_scratch + 768;      // Rin 16 x 16
  double* Rh = smem_scratch + 1024;     // Householder R 16 x 16
  double* Rk = smem_scratch + 1280;     // Rcheck diagonal
  double* A = smem_scratch + 1536;      // sketch block for Householder (<= 32 x 16)
  const int K = f.K;

  if (f.ops & (FIN_COPY_Q | FIN_PIP)) {
    for (int e = tid; e < f.p * K; e += nth) {
      const int i = e % f.p, j = e / f.p;
      f.Cq[f.q_row_off + i + j * f.ldcq] = sums[f.off_q + i + j * f.ld_q];
    }
    __syncthreads();
  }
  if (f.ops & FIN_COPY_G) {
    for (int e = tid; e < 256; e += nth) f.Gout[e] = sums[f.off_g + e];
  }
  if (f.ops & (FIN_COEFF | FIN_MULT))
    for (int e = tid; e < 256; e += nth) Rn[e] = f.Rin[e];
  if (f.ops & FIN_CHECK_DIAG)
    for (int e = tid; e < 16; e += nth) Rk[e] = f.Rcheck[e + e * kRld];
  if (f.ops & (FIN_HH | FIN_COPY_S)) {
    // S = sketch block (mh x K); count-gauss: S = Theta_g^T * count (sequential sums,
    // proj/src/dense.cpp:28-42 order)
    const int mh = f.mh;
    for (int e = tid; e < mh * K; e += nth) {
      const int i = e % mh, j = e / mh;
      double v;
      if (f.theta_g) {
        double s = 0.0;
        for (int r = 0; r < f.mc; ++r)
          s = tiny::add(s, tiny::mul(f.theta_g[r + (long long)i * f.mc], sums[f.off_s + r + j * f.ld_s]));
        v = s;
      } else {
        v = sums[f.off_s + i + j * f.ld_s];
      }
      A[i + j * mh] = v;
      if (f.ops & FIN_COPY_S) f.Sout[i + j * mh] = v;
    }
    __syncthreads();
    if (f.ops & FIN_HH) {
      tiny::householder_r(A, mh, mh, K, Rh, sb);
      __syncthreads();
      for (int e = tid; e < 256; e += nth) f.Rhh[e] = Rh[e];
      if (tid == 0) {
        for (int j = 0; j < K; ++j)
          if (Rh[j + j * kRld] == 0.0) {  // apply_inv_upper throws SingularTriangular(j)
            f.status->code = ST_SINGULAR;
            f.status->pass = f.pass_id;
            f.status->step = j;
            f.status->pivot = 0.0;
            s_code = ST_SINGULAR;
            break;
          }
      }
      __syncthreads();
      if (s_code != ST_OK) return;
    }
  }
  if (f.ops & FIN_CHECK_DIAG) {
    __syncthreads();
    if (tid == 0) {
      for (int j = 0; j < K; ++j)
        if (Rk[j] == 0.0) {
          f.status->code = ST_SINGULAR;
          f.status->pass = f.pass_id;
          f.status->step = j;
          f.status->pivot = 0.0;
          s_code = ST_SINGULAR;
          break;
        }
    }
    __syncthreads();
    if (s_code != ST_OK) return;
  }
  if (f.ops & FIN_CHOL) {
    // G = GRAM block (optionally minus proj^T proj for BCGS-PIP, block_orth.cpp:245-251;
    // proj is read back from Cq, which holds every projection chunk)
    for (int e = tid; e < 256; e += nth) {
      const int i = e % 16, j = e / 16;
      double g = sums[f.off_g + e];
      if ((f.ops & FIN_PIP) && i < K && j < K) {
        double s = 0.0;
        for (int l = 0; l < f.p_total; ++l) s = tiny::add(s, tiny::mul(f.Cq[l + i * f.ldcq], f.Cq[l + j * f.ldcq]));
        g = tiny::sub(g, s);
      }
      G[e] = g;
    }
    __syncthreads();
    tiny::cholesky(G, K, f.pivot_tol, Rc, sb, &s_fail, &s_piv);
    __syncthreads();
    for (int e = tid; e < 256; e += nth) f.Rchol[e] = Rc[e];
    if (s_fail) {
      if (tid == 0) {
        f.status->code = ST_CHOLESKY;
        f.status->pass = f.pass_id;
        f.status->step = s_fail;
        f.status->pivot = s_piv;
      }
      __syncthreads();
      return;
    }
  } else if (f.ops & (FIN_COEFF | FIN_MULT)) {
    for (int e = tid; e < 256; e += nth) Rc[e] = f.Rchol[e];
    __syncthreads();
  }
  if (f.ops & FIN_COEFF) {
    tiny::update_projection(f.C1, f.C2, f.ldc, f.p_total, K, Rn, f.coeffs);
  }
  if (f.ops & (FIN_COEFF | FIN_MULT)) {
    tiny::multiply_upper(Rc, Rn, K, f.rjj);
  }
  __syncthreads();
}

// dynamic shared memory: (1536 + max(mh, 32) * 16 + 64) doubles (the sketch
// block of a Count sketch has one row per bucket)
static __global__ void __launch_bounds__(256) finalize_kernel(FinArgs f) {
  extern __shared__ __align__(16) double fin_scratch[];
  finalize_dev(f, fin_scratch);
}


// X = X R^{-1} for one row held in registers (proj/src/dense.cpp:166-186).
// Right-looking schedule: at step j, x_j is divided by r_jj and then removed
// from every later column l.  Each x_l still receives its subtractions in
// the reference order i = 0..l-1 before its division, so with EXACT the
// result is bit-identical to apply_inv_upper; the (K - j) independent
// updates per step give the ILP the left-looking loop lacks.  Without EXACT,
// subtractions are fused (FMA) and the division is a multiply by 1/r_jj.
template <bool EXACT, int KC>
__device__ __forceinline__ void row_trsm(double (&x)[kMaxK], const double* R, const double* rinv, int K) {
  constexpr int KM = KC ? KC : kMaxK;  // compile-time width when specialised
#pragma unroll
  for (int j = 0; j < KM; ++j) {
    if (KC || j < K) {
      x[j] = EXACT ? tiny::div(x[j], R[j + j * kRld]) : x[j] * rinv[j];
#pragma unroll
      for (int l = j + 1; l < KM; ++l) {
        if (KC || l < K) {
          const double rjl = R[j + l * kRld];
          if (EXACT) {
            if (rjl != 0.0) x[l] = tiny::sub(x[l], tiny::mul(rjl, x[j]));
          } else {
            x[l] = fma(-rjl, x[j], x[l]);  // branch-free: a zero coefficient is a no-op
          }
        }
      }
    }
  }
}


// Row solve against a row-major copy of R (Rt[j*16 + l] = R[j + l*16] for
// l > j, Rt[j*16 + j] = 1 / r_jj): the coefficients of step j are contiguous,
// so they arrive as 16-byte vector loads issued before the step's FMAs
// (with R read one entry per FMA, every FMA waits on its own shared load).
template <int KC, int NR>
__device__ __forceinline__ void row_trsm_t(double (&x)[NR][kMaxK], const double* Rt) {
#pragma unroll
  for (int j = 0; j < KC; ++j) {
    double r[16];
#pragma unroll
    for (int l2 = 0; l2 < 16; l2 += 2) {
      if (l2 + 1 >= j && l2 < KC) {
        const double2 v = *reinterpret_cast<const double2*>(Rt + j * 16 + l2);
        r[l2] = v.x;
        r[l2 + 1] = v.y;
      }
    }
#pragma unroll
    for (int q = 0; q < NR; ++q) x[q][j] *= r[j];
#pragma unroll
    for (int l = j + 1; l < KC; ++l)
#pragma unroll
      for (int q = 0; q < NR; ++q) x[q][l] = fma(-r[l], x[q][j], x[q][l]);
  }
}

// several independent rows per thread, interleaved for ILP
template <bool EXACT, int KC, int NR>
__device__ __forceinline__ void row_trsm_n(double (&x)[NR][kMaxK], const double* R, const double* rinv, int K) {
  constexpr int KM = KC ? KC : kMaxK;
#pragma unroll
  for (int j = 0; j < KM; ++j) {
    if (KC || j < K) {
      const double dj = rinv[j];
#pragma unroll
      for (int q = 0; q < NR; ++q) x[q][j] = EXACT ? tiny::div(x[q][j], R[j + j * kRld]) : x[q][j] * dj;
#pragma unroll
      for (int l = j + 1; l < KM; ++l) {
        if (KC || l < K) {
          const double rjl = R[j + l * kRld];
#pragma unroll
          for (int q = 0; q < NR; ++q) {
            if (EXACT) {
              if (rjl != 0.0) x[q][l] = tiny::sub(x[q][l], tiny::mul(rjl, x[q][j]));
            } else {
              x[q][l] = fma(-rjl, x[q][j], x[q][l]);
            }
          }
        }
      }
    }
  }
}

// slot = i % n and phase = (i / n) & 1 of a ring position i, advanced without
// the integer division (~25 instructions each for a runtime n: the four per
// tile of the consumer loops were 16% of the stall samples of a p = 11
// projection pass)
struct RingCursor {
  int slot = 0, n;
  uint32_t phase = 0;
  __device__ explicit RingCursor(int n_, int start = 0) : n(n_) {
    slot = start;
    while (slot >= n) slot -= n, phase ^= 1u;
  }
  __device__ __forceinline__ void next() {
    if (++slot == n) {
      slot = 0;
      phase ^= 1u;
    }
  }
};

// ---------------------------------------------------------------------------
// the pass kernel
// ---------------------------------------------------------------------------
// Warp roles (NW = consumer_warps(UPD) consumer warps + 1 producer):
//   warp NW       producer: one 2-D TMA box per operand per tile (V, Q range,
//                 Theta) + a 1-D bulk copy of the Count codes, mbarrier ring.
//   warps 0..NW-1 consumers.  Without a pre-TRSM they form one group that
//                 runs U -> A' -> S -> R on each tile.  With a pre-TRSM
//                 (NPRE > 0) warps 0-1 solve rows (A) into a double-buffered
//                 X tile while the others run U/S/R on the previous tile,
//                 handed over with named-barrier arrive/sync pairs.  Row mode
//                 (ROWG, below) gives every consumer warp whole tiles.
// Every staged operand block is zero-padded to a multiple of 8 columns and
// TMA zero-fills rows past the matrix, so the tensor-core loops need no masks;
// the number of 8-column tiles is dispatched to a compile-time constant.
template <int NT, int T, int NPRE, bool UPD, int NPOST, bool QTX, bool GRAM, int SK, bool STORE, bool EXACT,
          int KC = 0>
__global__ void __launch_bounds__(pass_threads(UPD, NPRE > 0 && QTX, NPRE > 0 && UPD), 1)
    pass_kernel(const __grid_constant__ PassArgs a, const __grid_constant__ CUtensorMap tmV,
                const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmT) {
  constexpr int S = TileGeom<T>::S;
  constexpr int NSUB = TileGeom<T>::NSUB;  // 128-row sub-tiles per tile (T = 256: 2)
  constexpr int NW = consumer_warps(UPD, NPRE > 0 && QTX, NPRE > 0 && UPD);
  constexpr bool SPLIT = NPRE > 0;
  // Row-solve warps.  Two, by measurement: NW - 4 (one U/S/R warp per SM
  // sub-partition) was 3% slower over the C2 sequence, since the update is
  // bound by the shared FP64 pipe, not by which sub-partition issues it.
  constexpr int GAW0 = (NPRE > 0 && QTX) ? BO_GAW_QTX : (NPRE > 0 && UPD) ? BO_GAW_UPD : BO_GAW;
  constexpr int GAWR = SPLIT ? (GAW0 > 0 ? GAW0 : NW - 4) : 0;
  constexpr int GAW = (SPLIT && GAWR * 128 < T) ? T / 128 : GAWR;  // at most four rows per solve thread
  // Solve warps of this launch.  The pre-solve projection passes (one solve,
  // QTX) take a.gaw = 1 where the basis block is wide (host: p >= 25), which
  // gives the contraction a sixth warp (measured P1_QTX p = 55 739 -> 667 us,
  // but 400 -> 466 us at p = 11, where one warp's solve is the bound).
  const int gaw = (SPLIT && QTX && a.gaw > 0 && a.gaw < GAW && a.gaw * 128 >= T) ? a.gaw : GAW;
  // warps of the U/S/R group.  a.gw_active < NW - gaw leaves the rest idle
  // (diagnostic: BO_QTX_GW_SMALLP; fewer contraction warps measured slower)
  const int GW = (SPLIT && QTX && a.gw_active > 0 && a.gw_active < NW - gaw) ? a.gw_active : NW - gaw;
  const int GT = GW * 32;
  constexpr int GBAR = SPLIT ? 6 : 1;      // named barrier of the U/S/R group
  constexpr bool XT = (NPRE > 0) || UPD || (NPOST > 0);  // X lives in the X tile
  // X is computed in place in the stage's V block (each row / row group is
  // owned by one thread / warp): no separate X tile, so the stage ring keeps
  // two stages at 128-row tiles even for 88-column stages (p = 55 + the
  // 22-row sketch), and the row-solve warps of pre-solve passes can run a
  // whole ring ahead (per-stage "solved" mbarriers) instead of two tiles.
  // A stage is released once its bulk store has read it.
  constexpr bool XIN = (UPD && NPRE == 0) || SPLIT;  // (pre-solve passes: the row solves write X in place)
  constexpr int KP = NT * 8;               // padded panel width
  constexpr int MQT = kMaxPTile / 8;
  constexpr int MST = 4;
  // Row mode: a triangular solve followed only by the Gram (P1_GRAM).  The
  // tensor-core Gram would waste 2/3 of its FLOPs on the 11 -> 16 padding and
  // leave the solve to two warps; instead every consumer warp takes whole
  // tiles, solves four rows per thread and accumulates the K(K+1)/2 Gram
  // entries with FP64 FMAs.
  constexpr bool ROWG = GRAM && !QTX && !UPD && SK == SK_NONE && !STORE && NPOST == 0 && NPRE > 0 && KC > 0 &&
                        KC <= 11 && T == 128;
  constexpr int NG = ROWG ? KC * (KC + 1) / 2 : 1;
  // Tail columns.  With 8 < K <= 11 (K = 11 at s = 10) the second 8-column
  // DMMA tile would carry 16 - K zero columns: 5 of its 8 at K = 11.  Its
  // TN = K - 8 live columns instead go through FP64 FMAs on the fragments
  // already in registers.  In a contraction, lane (g, t4) holds A[g][t4] (row
  // t4 of the k-step), so TN extra shared loads of X[row t4][8..K) feed TN FMAs
  // per A fragment.  In the update, lane (g, t4) holds Q[row g][col t4] and the
  // coefficients -C[t4][8..K) in registers; the TN partial sums are reduced
  // over the 4 t4 lanes per row group.  Per k-step and 8 rows: 3 DFMA (about
  // 7 FP64-pipe cycles per sub-partition) instead of one DMMA (16 cycles).
  constexpr int TN = (BO_DFMA_TAIL && NT == 2 && KC > 8 && KC <= 11 && !EXACT && SK != SK_GAUSS) ? KC - 8 : 0;
  constexpr int TNA = TN ? TN : 1;         // array extents
  constexpr int NPAIR = TN * (TN + 1) / 2; // tail x tail Gram entries, one per lane group g
  constexpr bool TQ = TN && QTX && BO_TAIL_QTX;   // per site (measured: the tail pays only where
  constexpr bool TU = TN && UPD && BO_TAIL_UPD;   // the DMMA work per k-step is large enough)
  constexpr bool TG = TN && GRAM && BO_TAIL_GRAM;
  constexpr int NTG = TG ? 1 : NT;                // Gram column tiles on DMMA
  static_assert(!(QTX && UPD), "a pass either projects or updates");
  static_assert(!STORE || XT, "stores come from the X tile");
  static_assert(!SPLIT || T <= GAW * 128, "row-solve group handles at most four rows per thread");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int K = KC ? KC : a.K;
  const int p = a.p, mh = a.mh;
  const long long nrows = a.nrows;

  const int ncolQ = (QTX || UPD) ? p : 0, ncolT = (SK == SK_GAUSS) ? mh : 0;
  const int mq = (ncolQ + 7) >> 3, ms = (ncolT + 7) >> 3;  // 8-column tiles
  // offset of row r of a P-column operand block (see TileGeom): c * S + so(r, P)
  auto so = [](int r, int P) { return NSUB > 1 ? (r >> 7) * P * S + (r & 127) : r; };
  const StageLayout L = stage_layout(K, ncolQ, ncolT, SK == SK_COUNT, T, !ROWG);
  // Decoupled rings (pre-solve passes with a projection range).  With joint
  // stages a stage is held from its arrival through the row solve AND the
  // U/S/R work, so at p = 55 (76 KB stages, 2 fit) the basis block of the next
  // tile is issued only after both: the solve latency is exposed once per tile
  // and the HBM stream idles (ncu: solve warps 67% of their samples waiting
  // for data, the producer half its time waiting for a free stage).  Here the
  // panel tiles (K columns, 17 KB) live in their own ring, VLA = NSV - NS
  // tiles ahead of the basis ring, so a tile's rows are solved before its
  // basis block lands and a basis slot is held only for the U/S/R work, as in
  // the passes without a solve.  Tile it uses basis slot it % NS and panel slot
  // it % NSV; the producer issues basis tile it and panel tile it + VLA when
  // the group releases tile it - NS, which frees both slots.
  // The host picks it per launch (a.nstages_v > 0) where joint stages would
  // leave only two in the ring (p >= 44 at K = 11); with deeper joint rings it
  // measured slower.
  constexpr bool DEC = BO_DEC_RING && SPLIT && !ROWG && (QTX || UPD) && BO_PRODUCER_WARP;
  const bool dec = DEC && a.nstages_v > 0;
  const int NS = a.nstages;                    // joint ring depth, or the basis ring's (dec)
  const int NSV = dec ? a.nstages_v : NS;      // panel ring depth (dec)
  const int VLA = NSV - NS;                    // panel lookahead in tiles (DEC)
  const int vsz = L.offQ, qsz = L.stage - L.offQ;  // DEC slot sizes (doubles)
  double* stages = reinterpret_cast<double*>(smem_raw);
  // V block of panel slot sv, and the basis-side blocks (Q, Theta, codes) of slot sq
  auto slotV = [&](int sv) { return dec ? stages + (size_t)sv * vsz : stages + (size_t)sv * L.stage + L.offV; };
  auto slotQ = [&](int sq) {
    return dec ? stages + (size_t)NSV * vsz + (size_t)sq * qsz : stages + (size_t)sq * L.stage + L.offQ;
  };
  double* xtile = stages + a.region0_dbl;                         // [2][NSUB][KP][S]
  double* rfac = xtile + ((XT && !ROWG && !XIN) ? 2 * NSUB * KP * S : 0); // [3][256]
  double* rinv = rfac + 3 * 256;                                  // [3][16]
  constexpr bool RFT = KC > 0 && !EXACT && (NPRE > 0 || NPOST > 0);
  double* rft = rinv + 48;                                        // [3][256] row-major R, 1/r_jj on the diagonal
  double* cacc = rft + (RFT ? 3 * 256 : 0);                       // count acc [mh][K]
  uint64_t* bars = reinterpret_cast<uint64_t*>(cacc + ((SK == SK_COUNT) ? mh * K : 0));
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages;
  uint64_t* solved = bars + 2 * kMaxStages;  // pre-solve passes: X of the stage is ready
  uint64_t* fullv = bars + 3 * kMaxStages;   // DEC: panel slot loaded
  __shared__ int s_skip;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      ptx::mbar_init(&full[s], 1);
      // DEC: only the U/S/R group releases (the solve warps are done with a
      // tile before the group starts it)
      if (BO_PRODUCER_WARP) ptx::mbar_init(&empty[s], ROWG ? 1 : (dec ? GW : gaw + GW));
      else reinterpret_cast<unsigned*>(&empty[s])[0] = 0u;  // arrival counter
    }
    for (int s = 0; s < NSV; ++s) {
      if (SPLIT) ptx::mbar_init(&solved[s], gaw);
      if (dec) ptx::mbar_init(&fullv[s], 1);
    }
    ptx::fence_mbar_init();
  }
  if (SK == SK_COUNT)
    for (int e = tid; e < mh * K; e += blockDim.x) cacc[e] = 0.0;
  // zero padding columns (never written by TMA or the phases)
  for (int s = 0; s < (ROWG ? 0 : NSV); ++s)
    for (int q = 0; q < NSUB; ++q) {
      double* sv = slotV(s);
      for (int e = tid; e < (KP - K) * S; e += blockDim.x) sv[q * KP * S + K * S + e] = 0.0;
    }
  for (int s = 0; s < (ROWG ? 0 : NS); ++s)
    for (int q = 0; q < NSUB; ++q) {
      double* sq = slotQ(s);
      for (int e = tid; e < (mq * 8 - ncolQ) * S; e += blockDim.x) sq[q * mq * 8 * S + ncolQ * S + e] = 0.0;
      for (int e = tid; e < (ms * 8 - ncolT) * S; e += blockDim.x)
        sq[(L.offT - L.offQ) + q * ms * 8 * S + ncolT * S + e] = 0.0;
    }
  if (XT && !ROWG && !XIN)
    for (int b = 0; b < 2 * NSUB; ++b)
      for (int e = tid; e < (KP - K) * S; e += blockDim.x) xtile[b * KP * S + K * S + e] = 0.0;
  if (tid == 0) s_skip = a.status->code != ST_OK;
  if (NPRE > 0)
    for (int e = tid; e < 256; e += blockDim.x) rfac[e] = a.Rpre0[e];
  if (NPRE > 1)
    for (int e = tid; e < 256; e += blockDim.x) rfac[256 + e] = a.Rpre1[e];
  if (NPOST > 0)
    for (int e = tid; e < 256; e += blockDim.x) rfac[512 + e] = a.Rpost[e];
  __syncthreads();
  if (tid < 48) {
    const int f = tid / 16, j = tid % 16;
    rinv[tid] = 1.0 / rfac[f * 256 + j + j * kRld];
  }
  if (RFT) {
    __syncthreads();
    for (int e = tid; e < 3 * 256; e += blockDim.x) {
      const int f = e / 256, j = (e % 256) / 16, l = e % 16;  // Rt_f[j*16 + l]
      rft[e] = l > j ? rfac[f * 256 + j + l * kRld] : (l == j ? rinv[f * 16 + j] : 0.0);
    }
  }
  // Tail update coefficients (TN > 0): ctls[r * 4 + c] = -C[r][8 + c], r < 64, in
  // the R-factor slot this pass does not use (a pre-solve pass has no post
  // factor; a post-solve pass no pre factor).  A lane reads its row t4 of a
  // k-step as one 16-byte and one 8-byte shared load (4 addresses per warp);
  // 48 coefficient registers per thread would spill at the 168-register cap.
  static_assert(!(TU && NPRE > 0 && NPOST > 0), "tail coefficients need a free R-factor slot");
  double* ctls = rfac + (NPOST > 0 ? 0 : 512);
  if (TU) {
    __syncthreads();  // rinv / rft have read the slot
    for (int e = tid; e < 256; e += blockDim.x) {
      const int r = e >> 2, c = e & 3;
      ctls[e] = (r < p && c < TN) ? -a.Cm[r + (8 + c) * a.ldc] : 0.0;
    }
  }
  __syncthreads();
  if (s_skip) return;  // an earlier pass broke down: this one is a no-op

  const int ntiles = a.ntiles;
  const int my_tiles = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  // ------------------------------------------------------------ producer
  // Warp NW issues the TMA loads.  8 warps per CTA (7 consumers + producer)
  // put 2 warps on each SM sub-partition, so a thread may use up to 255
  // registers (a 9th warp would cap every thread at 168 and spill).
  // Row mode: consumer warp w owns the stages w, w + NW, ... (NS / NW of
  // them) and its tiles w, w + NW, ... are loaded into them in order (a
  // private ring per warp: no phase aliasing between warps running apart).
  const uint32_t box_bytes = (uint32_t)(NSUB * S * 8 * (K + ncolQ + ncolT));
  const int nsub = ROWG ? NS / NW : NS;
  auto stage_of = [&](int it, int& s, int& use) {
    if (ROWG) {
      const int w = it % NW, j = it / NW;
      s = w + NW * (j % nsub);
      use = j / nsub;
    } else {
      s = it % NS;
      use = it / NS;
    }
  };
  auto issue = [&](int it, int s) {
    const long long row0 = (long long)(blockIdx.x + (long long)it * gridDim.x) * T;
    const long long valid = nrows - row0 < T ? nrows - row0 : T;
    const uint32_t cb = (SK == SK_COUNT) ? (uint32_t)(((valid + 3) & ~3LL) * 4) : 0u;
    double* st = stages + (size_t)s * L.stage;
    ptx::mbar_arrive_expect_tx(&full[s], box_bytes + cb);
#pragma unroll
    for (int q = 0; q < NSUB; ++q) {
      ptx::tma_load_2d(st + L.offV + q * KP * S, &tmV, (int)row0 + 128 * q, 0, &full[s]);
      if (ncolQ) ptx::tma_load_2d(st + L.offQ + q * mq * 8 * S, &tmQ, (int)row0 + 128 * q, 0, &full[s]);
      if (ncolT) ptx::tma_load_2d(st + L.offT + q * ms * 8 * S, &tmT, (int)row0 + 128 * q, 0, &full[s]);
    }
    if (SK == SK_COUNT) ptx::bulk_g2s(st + L.offC, a.code + row0, cb, &full[s]);
  };
  // DEC: the panel tile into panel slot sv, the basis-side blocks into basis slot sq
  auto issue_v = [&](int it, int sv) {
    const long long row0 = (long long)(blockIdx.x + (long long)it * gridDim.x) * T;
    double* dst = slotV(sv);
    ptx::mbar_arrive_expect_tx(&fullv[sv], (uint32_t)(NSUB * S * 8 * K));
#pragma unroll
    for (int q = 0; q < NSUB; ++q) ptx::tma_load_2d(dst + q * KP * S, &tmV, (int)row0 + 128 * q, 0, &fullv[sv]);
  };
  auto issue_q = [&](int it, int sq) {
    const long long row0 = (long long)(blockIdx.x + (long long)it * gridDim.x) * T;
    const long long valid = nrows - row0 < T ? nrows - row0 : T;
    const uint32_t cb = (SK == SK_COUNT) ? (uint32_t)(((valid + 3) & ~3LL) * 4) : 0u;
    double* dst = slotQ(sq);
    ptx::mbar_arrive_expect_tx(&full[sq], (uint32_t)(NSUB * S * 8 * (ncolQ + ncolT)) + cb);
#pragma unroll
    for (int q = 0; q < NSUB; ++q) {
      if (ncolQ) ptx::tma_load_2d(dst + q * mq * 8 * S, &tmQ, (int)row0 + 128 * q, 0, &full[sq]);
      if (ncolT) ptx::tma_load_2d(dst + (L.offT - L.offQ) + q * ms * 8 * S, &tmT, (int)row0 + 128 * q, 0, &full[sq]);
    }
    if (SK == SK_COUNT) ptx::bulk_g2s(dst + (L.offC - L.offQ), a.code + row0, cb, &full[sq]);
  };
  // A consumer warp calls release(it, s) after its last read of stage s for
  // tile it.  With a producer warp that is an mbarrier arrival; otherwise the
  // last warp to release a stage refills it with the tile NS ahead (row mode:
  // the owning warp refills its private ring), so no warp ever waits to issue.
  unsigned* arrivals = reinterpret_cast<unsigned*>(empty);
  auto release = [&](int it, int s) {
    __syncwarp();
    if (lane == 0) {
      if (BO_PRODUCER_WARP) {
        ptx::mbar_arrive(&empty[s]);
      } else if (ROWG) {
        if (it + NW * nsub < my_tiles) {
          ptx::fence_proxy_async_smem();  // our generic-proxy reads before the async-proxy refill
          issue(it + NW * nsub, s);
        }
      } else {
        __threadfence_block();
        if (atomicAdd(reinterpret_cast<unsigned*>(&empty[s]), 1u) == (unsigned)(NW - 1)) {
          reinterpret_cast<unsigned*>(&empty[s])[0] = 0u;
          __threadfence_block();
          if (it + NS < my_tiles) {
            ptx::fence_proxy_async_smem();
            issue(it + NS, s);
          }
        }
      }
    }
    __syncwarp();
  };
  (void)arrivals;
  if (!BO_PRODUCER_WARP) {
    if (ROWG ? lane == 0 : tid == 0) {
      ptx::prefetch_tmap(&tmV);
      if (ncolQ) ptx::prefetch_tmap(&tmQ);
      if (ncolT) ptx::prefetch_tmap(&tmT);
      if (ROWG) {
        for (int j = 0; j < nsub && warp + NW * j < my_tiles; ++j) issue(warp + NW * j, warp + NW * j);
      } else {
        for (int it = 0; it < NS && it < my_tiles; ++it) issue(it, it);
      }
    }
  }
  if (BO_PRODUCER_WARP && warp == NW) {
    if (lane == 0) {
      ptx::prefetch_tmap(&tmV);
      if (ncolQ) ptx::prefetch_tmap(&tmQ);
      if (ncolT) ptx::prefetch_tmap(&tmT);
      if (dec) {
        for (int j = 0; j < VLA && j < my_tiles; ++j) issue_v(j, j);
        RingCursor cq(NS), cv(NSV, VLA);
        for (int it = 0; it < my_tiles; ++it, cq.next(), cv.next()) {
          // tile it - NS released: its basis slot and its panel slot, which
          // panel tile it + VLA (= it - NS + NSV) takes
          if (it >= NS) ptx::mbar_wait(&empty[cq.slot], cq.phase ^ 1u);
          issue_q(it, cq.slot);
          if (it + VLA < my_tiles) issue_v(it + VLA, cv.slot);
        }
      } else if (!ROWG) {
        RingCursor c(NS);
        for (int it = 0; it < my_tiles; ++it, c.next()) {
          if (it >= NS) ptx::mbar_wait(&empty[c.slot], c.phase ^ 1u);
          issue(it, c.slot);
        }
      } else {
        for (int it = 0; it < my_tiles; ++it) {
          int s, use;
          stage_of(it, s, use);
          if (use > 0) ptx::mbar_wait(&empty[s], (use - 1) & 1);
          issue(it, s);
        }
      }
    }
  } else {
    // update coefficients as DMMA B fragments:  B[kk][j] = -C[c0+kk][nj*8+j]
    double cfr[UPD ? MQT * 2 : 1][NT];
    if (UPD) {
#pragma unroll
      for (int ks = 0; ks < MQT * 2; ++ks)
#pragma unroll
        for (int nj = 0; nj < NT; ++nj) {
          const int r = ks * 4 + t4, c = nj * 8 + g;
          cfr[ks][nj] = (r < p && c < K) ? -__ldg(a.Cm + r + c * a.ldc) : 0.0;  // L1: one miss per line per SM
        }
    }
    // tail accumulators (TN > 0): projections tq[mi][c] = sum Q[.][mi*8+g] X[.][8+c],
    // Gram tg[c] = sum X[.][g] X[.][8+c] and tgg = the lane group's tail x tail pair,
    // each a partial sum over the rows t4 of the k-steps (reduced over t4 at the end)
    double tq[TQ ? MQT : 1][TNA];
    double tg[TG ? TN : 1];
    double tgg = 0.0;
    int pa = 0, pb = 0;  // lane group g < NPAIR owns the tail pair (pa <= pb) number g
    {
      int e = 0;
#pragma unroll
      for (int ca = 0; ca < TN; ++ca)
#pragma unroll
        for (int cb = ca; cb < TN; ++cb) {
          if (e == g) pa = ca, pb = cb;
          ++e;
        }
    }
#pragma unroll
    for (int i = 0; i < (TQ ? MQT : 1); ++i)
#pragma unroll
      for (int c = 0; c < TNA; ++c) tq[i][c] = 0.0;
#pragma unroll
    for (int c = 0; c < (TG ? TN : 1); ++c) tg[c] = 0.0;
    double accq[QTX ? MQT : 1][NT][2];
    double accg[GRAM ? NT : 1][NT][2];
    double accs[(SK == SK_GAUSS) ? MST : 1][NT][2];
#pragma unroll
    for (int i = 0; i < (QTX ? MQT : 1); ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) accq[i][j][0] = accq[i][j][1] = 0.0;
#pragma unroll
    for (int i = 0; i < (GRAM ? NT : 1); ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) accg[i][j][0] = accg[i][j][1] = 0.0;
#pragma unroll
    for (int i = 0; i < ((SK == SK_GAUSS) ? MST : 1); ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) accs[i][j][0] = accs[i][j][1] = 0.0;

    const bool in_trsm_group = SPLIT && !ROWG && warp < gaw;
    const int gw = warp - gaw;  // warp index within the U/S/R group
    const int gtid = gw * 32 + lane;
    // bulk stores: column c is issued by lane c / GW of group warp c % GW, so
    // the issue cost (proxy fence + one bulk copy per column and sub-tile) is
    // spread over the group instead of serialising in one warp
    const int stc = BO_STORE_SPREAD ? gw + GW * lane : gtid;
    // Gram accumulators of the row modes: zeroed inside each role's branch so
    // they are not live (registers) across the row-solve warps' loop
    double gacc[NG];
#if BO_PHASE_PROF
    unsigned long long pp_acc[16] = {};
#endif

    if constexpr (ROWG) {
#pragma unroll
      for (int e = 0; e < NG; ++e) gacc[e] = 0.0;
      // ------------------------------------------- row mode (P1_GRAM)
      // warp w consumes tiles w, w + 8, ...; lane l holds rows l + 32 q
      // (q < 4): four independent rows per solve step (ILP, and one shared-
      // memory read of each R entry per four FMAs)
      constexpr int RQ = KC > 8 ? BO_ROWG_RQ_WIDE : 2;  // rows per thread per step (register budget)
      RingCursor cr(nsub);
      for (int j = 0, it = warp; it < my_tiles; ++j, it += NW, cr.next()) {
        const int s = warp + NW * cr.slot;
        const long long row0 = (long long)(blockIdx.x + (long long)it * gridDim.x) * T;
        const int valid = (int)(nrows - row0 < T ? nrows - row0 : T);
        const double* stV = stages + (size_t)s * L.stage + L.offV;
        ptx::mbar_wait(&full[s], cr.phase);
        for (int h = 0; h < T / (32 * RQ); ++h) {
          // keep the R entries in shared memory (re-read per step) rather than
          // hoisted into registers next to the K(K+1)/2 accumulators
          asm volatile("" ::: "memory");
          double x[RQ][kMaxK];
#pragma unroll
          for (int q = 0; q < RQ; ++q)
#pragma unroll
            for (int c = 0; c < kMaxK; ++c) x[q][c] = (c < KC) ? stV[c * S + lane + 32 * (h * RQ + q)] : 0.0;
          row_trsm_t<KC, RQ>(x, rft);
#pragma unroll
          for (int q = 0; q < RQ; ++q) {
            if (lane + 32 * (h * RQ + q) < valid) {
              int e = 0;
#pragma unroll
              for (int i = 0; i < KC; ++i)
#pragma unroll
                for (int j = i; j < KC; ++j) {
                  gacc[e] = fma(x[q][i], x[q][j], gacc[e]);
                  ++e;
                }
            }
          }
        }
        release(it, s);
      }
      // warp butterfly (fixed order) of every Gram entry
#pragma unroll
      for (int e = 0; e < NG; ++e) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) gacc[e] += __shfl_xor_sync(0xffffffffu, gacc[e], o);
      }
    } else if (in_trsm_group) {
      // ---------------------------------------------- A: row solves (warps 0-1)
      RingCursor cs(NS), csv(NSV);
      for (int it = 0; it < my_tiles; ++it, cs.next(), csv.next()) {
        const int s = cs.slot, sv = csv.slot;
        const long long row0 = (long long)(blockIdx.x + (long long)it * gridDim.x) * T;
        const int valid = (int)(nrows - row0 < T ? nrows - row0 : T);
        const double* stV = slotV(sv);
        double* xt = const_cast<double*>(stV);  // X in place
        PP_T0();
        if (dec) ptx::mbar_wait(&fullv[sv], csv.phase);
        else ptx::mbar_wait(&full[s], cs.phase);
        PP_MARK(8);
        auto solve = [&](auto gaw_c) {
          constexpr int GAWX = decltype(gaw_c)::value;
          constexpr int RPT = (T + GAWX * 32 - 1) / (GAWX * 32);  // rows per thread
          double x[RPT][kMaxK];
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const int r = tid + q * GAWX * 32;
#pragma unroll
            for (int c = 0; c < kMaxK; ++c) x[q][c] = (c < K && r < T) ? stV[c * S + so(r, KP)] : 0.0;
          }
          if constexpr (KC > 0 && !EXACT) {
            row_trsm_t<KC, RPT>(x, rft);
            if (NPRE > 1) row_trsm_t<KC, RPT>(x, rft + 256);
          } else {
            row_trsm_n<EXACT, KC, RPT>(x, rfac, rinv, K);
            if (NPRE > 1) row_trsm_n<EXACT, KC, RPT>(x, rfac + 256, rinv + 16, K);
          }
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const int r = tid + q * GAWX * 32;
            if (r < T) {
#pragma unroll
              for (int c = 0; c < kMaxK; ++c)
                if (c < K) xt[c * S + so(r, KP)] = (r < valid) ? x[q][c] : 0.0;
            }
          }
        };
        constexpr int GAWC = GAW ? GAW : 1;
        if constexpr (QTX && GAWC > 1 && T <= 128) {
          if (gaw == 1) solve(std::integral_constant<int, 1>{});
          else solve(std::integral_constant<int, GAWC>{});
        } else {
          solve(std::integral_constant<int, GAWC>{});
        }
        __syncwarp();
        PP_MARK(9);
        if (lane == 0) ptx::mbar_arrive(&solved[sv]);  // X of tile it is in the stage
        if (!dec) release(it, s);
        PP_MARK(10);
      }
#pragma unroll
      for (int e = 0; e < NG; ++e) gacc[e] = 0.0;
    } else {
      // ------------------------------------------- U / A' / S / R group
#pragma unroll
      for (int e = 0; e < NG; ++e) gacc[e] = 0.0;
      RingCursor cs(NS), csv(NSV);
      for (int it = 0; it < (gw < GW ? my_tiles : 0); ++it, cs.next(), csv.next()) {
        const int s = cs.slot, b = it & 1, sv = csv.slot;
        const long long row0 = (long long)(blockIdx.x + (long long)it * gridDim.x) * T;
        const int valid = (int)(nrows - row0 < T ? nrows - row0 : T);
        const double* stV = slotV(sv);
        const double* stQ = slotQ(s);
        const double* stT = stQ + (L.offT - L.offQ);
        const uint32_t* stC = reinterpret_cast<const uint32_t*>(stQ + (L.offC - L.offQ));
        double* xt = XIN ? const_cast<double*>(stV) : xtile + b * NSUB * KP * S;

        // X buffer b was last stored from by tile it - 2: only the group before
        // the most recent one (tile it - 1, other buffer) has to be drained
        PP_T0();
        if (!SPLIT && !XIN && STORE && stc < K) ptx::bulk_wait_read1();
        ptx::mbar_wait(&full[s], cs.phase);
        PP_MARK(0);
        if (SPLIT) ptx::mbar_wait(&solved[sv], csv.phase);  // solved rows of this tile are in the stage
        PP_MARK(1);

        // ---- U: X = X0 - Q C on tensor cores (rows past the matrix are zero in
        // the stage and the coefficients past p / K are zero: no masks)
        if (UPD) {
          const double* x0 = SPLIT ? xt : stV;
          // Each accumulator is a chain of 2 * mq dependent DMMAs; the even and
          // odd k-steps go to separate accumulators (summed at the end) so a
          // warp has 2 * NT independent chains in flight instead of NT.  Only
          // in pre-solve passes: the plain update passes are HBM-bound already
          // and the extra registers would spill their sketch accumulators.
          auto upd = [&](auto mq_c) {
            constexpr int MQc = decltype(mq_c)::value;
            constexpr bool TUc = TU && MQc >= BO_TAIL_UPD_MIN;
            constexpr int NTD = TUc ? 1 : NT;  // column tiles on DMMA
            for (int rg = gw; rg < T / 8; rg += GW) {
              const int r = rg * 8 + g;
              double av[2 * MQc > 0 ? 2 * MQc : 1];
#pragma unroll
              for (int ks = 0; ks < 2 * MQc; ++ks) av[ks] = stQ[(ks * 4 + t4) * S + so(r, mq * 8)];
              double d[NTD][2], d1[NTD][2], u[TNA];
#pragma unroll
              for (int nj = 0; nj < NTD; ++nj)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  d[nj][e] = x0[(nj * 8 + 2 * t4 + e) * S + so(r, KP)];
                  d1[nj][e] = 0.0;
                }
#pragma unroll
              for (int c = 0; c < TNA; ++c) u[c] = 0.0;
#pragma unroll
              for (int ks = 0; ks < 2 * MQc; ++ks) {
#pragma unroll
                for (int nj = 0; nj < NTD; ++nj) {
                  if (SPLIT && (ks & 1)) ptx::dmma(d1[nj][0], d1[nj][1], av[ks], cfr[ks][nj]);
                  else ptx::dmma(d[nj][0], d[nj][1], av[ks], cfr[ks][nj]);
                }
                if constexpr (TUc) {
                  const double* cr = ctls + (ks * 4 + t4) * 4;
                  const double2 c01 = *reinterpret_cast<const double2*>(cr);
                  const double ct[3] = {c01.x, c01.y, TN > 2 ? cr[2] : 0.0};
#pragma unroll
                  for (int c = 0; c < TN; ++c) u[c] = fma(av[ks], ct[c], u[c]);
                }
              }
#pragma unroll
              for (int nj = 0; nj < NTD; ++nj)
#pragma unroll
                for (int e = 0; e < 2; ++e) xt[(nj * 8 + 2 * t4 + e) * S + so(r, KP)] = SPLIT ? d[nj][e] + d1[nj][e] : d[nj][e];
              if constexpr (TUc) {
                // sum the tail partials over the four t4 lanes of row g; lane t4 < TN
                // then writes column 8 + t4 of that row
                double ux = 0.0;
#pragma unroll
                for (int c = 0; c < TN; ++c) {
                  u[c] += __shfl_xor_sync(0xffffffffu, u[c], 1);
                  u[c] += __shfl_xor_sync(0xffffffffu, u[c], 2);
                  if (c == t4) ux = u[c];
                }
                if (t4 < TN) {
                  double* xp = xt + (8 + t4) * S + so(r, KP);
                  *xp = x0[(8 + t4) * S + so(r, KP)] + ux;
                }
              }
            }
          };
          switch (mq) {
            case 0: upd(std::integral_constant<int, 0>{}); break;
            case 1: upd(std::integral_constant<int, 1>{}); break;
            case 2: upd(std::integral_constant<int, 2>{}); break;
            case 3: upd(std::integral_constant<int, 3>{}); break;
            case 4: upd(std::integral_constant<int, 4>{}); break;
            case 5: upd(std::integral_constant<int, 5>{}); break;
            case 6: upd(std::integral_constant<int, 6>{}); break;
            case 7: upd(std::integral_constant<int, 7>{}); break;
            default: upd(std::integral_constant<int, 8>{}); break;
          }
          PP_MARK(2);
          ptx::named_bar_sync(GBAR, GT);
          PP_MARK(3);
        }

        // ---- A': post-TRSM (thread per row)
        if (NPOST > 0) {
          for (int r = gtid; r < T; r += GT) {
            double x[1][kMaxK];
#pragma unroll
            for (int c = 0; c < kMaxK; ++c) x[0][c] = (c < K) ? xt[c * S + so(r, KP)] : 0.0;
            if constexpr (KC > 0 && !EXACT)
              row_trsm_t<KC, 1>(x, rft + 512);
            else
              row_trsm<EXACT, KC>(x[0], rfac + 512, rinv + 32, K);
#pragma unroll
            for (int c = 0; c < kMaxK; ++c)
              if (c < K) xt[c * S + so(r, KP)] = (r < valid) ? x[0][c] : 0.0;
          }
          ptx::named_bar_sync(GBAR, GT);
        }

        const double* X = XT ? xt : stV;

        // ---- S: bulk store of the X tile (one request per column)
        if (STORE && stc < K) {
          ptx::fence_proxy_async_smem();
#pragma unroll
          for (int q = 0; q < NSUB; ++q) {
            const int vq = valid - 128 * q;
            if (vq > 0)
              ptx::bulk_s2g(a.out + (long long)stc * a.ldo + row0 + 128 * q, xt + q * KP * S + stc * S,
                            (uint32_t)((((vq < 128 ? vq : 128) + 1) & ~1) * 8));
          }
          ptx::bulk_commit();
        }

        PP_MARK(4);
        // ---- R: contractions on tensor cores; each warp owns k-steps
        // gw, gw + GW, ...; fragments of the next k-step are loaded before the
        // DMMAs of the current one issue
        if (QTX || GRAM || SK == SK_GAUSS) {
          auto contract = [&](auto m_c) {
            constexpr int M = decltype(m_c)::value;          // Q or Theta tiles (may be 0)
            constexpr int MQc = QTX ? M : 0, MSc = (SK == SK_GAUSS) ? M : 0;
            constexpr bool TQc = TQ && M >= BO_TAIL_QTX_MIN;
            constexpr int NTQ = TQc ? 1 : NT;  // projection column tiles on DMMA
            // column tiles of X fragments needed, and whether the tail columns are loaded
            constexpr int NTD = ((QTX && !TQc) || (GRAM && !TG) || SK == SK_GAUSS) ? NT : 1;
            constexpr int XTN = (TQc || TG) ? TN : 0;
            double bx[2][NTD], xtl[2][TNA], aq[2][MQc > 0 ? MQc : 1], at[2][MSc > 0 ? MSc : 1];
            auto load = [&](int ks, auto slot_c) {
              constexpr int slot = decltype(slot_c)::value;  // register-resident fragment sets
              const int r = ks * 4 + t4;
#pragma unroll
              for (int nj = 0; nj < NTD; ++nj) bx[slot][nj] = X[(nj * 8 + g) * S + so(r, KP)];
#pragma unroll
              for (int c = 0; c < XTN; ++c) xtl[slot][c] = X[(8 + c) * S + so(r, KP)];  // 4 addresses per warp
              if (QTX) {
#pragma unroll
                for (int mi = 0; mi < MQc; ++mi) aq[slot][mi] = stQ[(mi * 8 + g) * S + so(r, mq * 8)];
              }
              if (SK == SK_GAUSS) {
#pragma unroll
                for (int mi = 0; mi < MSc; ++mi) at[slot][mi] = stT[(mi * 8 + g) * S + so(r, ms * 8)];
              }
            };
            auto mma = [&](auto slot_c) {
              constexpr int slot = decltype(slot_c)::value;
              if (QTX) {
#pragma unroll
                for (int mi = 0; mi < MQc; ++mi) {
#pragma unroll
                  for (int nj = 0; nj < NTQ; ++nj)
                    ptx::dmma(accq[mi][nj][0], accq[mi][nj][1], aq[slot][mi], bx[slot][nj]);
                  if constexpr (TQc) {
#pragma unroll
                    for (int c = 0; c < TN; ++c) tq[mi][c] = fma(aq[slot][mi], xtl[slot][c], tq[mi][c]);
                  }
                }
              }
              if (GRAM) {
#pragma unroll
                for (int mi = 0; mi < NTG; ++mi)
#pragma unroll
                  for (int nj = 0; nj < NTG; ++nj)
                    if (mi <= nj) ptx::dmma(accg[mi][nj][0], accg[mi][nj][1], bx[slot][mi], bx[slot][nj]);
                if constexpr (TG) {
#pragma unroll
                  for (int c = 0; c < TN; ++c) tg[c] = fma(bx[slot][0], xtl[slot][c], tg[c]);
                  double xa = xtl[slot][0], xb = xtl[slot][0];
#pragma unroll
                  for (int c = 1; c < TN; ++c) {
                    xa = pa == c ? xtl[slot][c] : xa;
                    xb = pb == c ? xtl[slot][c] : xb;
                  }
                  tgg = fma(xa, xb, tgg);
                }
              }
              if (SK == SK_GAUSS) {
#pragma unroll
                for (int mi = 0; mi < MSc; ++mi)
#pragma unroll
                  for (int nj = 0; nj < NTD; ++nj)
                    ptx::dmma(accs[mi][nj][0], accs[mi][nj][1], at[slot][mi], bx[slot][nj]);
              }
            };
            int ks = gw;
            if (ks < T / 4) load(ks, std::integral_constant<int, 0>{});
            while (ks < T / 4) {
              if (ks + GW < T / 4) load(ks + GW, std::integral_constant<int, 1>{});
              mma(std::integral_constant<int, 0>{});
              ks += GW;
              if (ks >= T / 4) break;
              if (ks + GW < T / 4) load(ks + GW, std::integral_constant<int, 0>{});
              mma(std::integral_constant<int, 1>{});
              ks += GW;
            }
          };
          const int mcase = QTX ? mq : ((SK == SK_GAUSS) ? ms : 1);
          switch (mcase) {
            case 0: contract(std::integral_constant<int, 0>{}); break;
            case 1: contract(std::integral_constant<int, 1>{}); break;
            case 2: contract(std::integral_constant<int, 2>{}); break;
            case 3: contract(std::integral_constant<int, 3>{}); break;
            case 4: contract(std::integral_constant<int, 4>{}); break;
            case 5: if (QTX) contract(std::integral_constant<int, QTX ? 5 : 1>{}); break;
            case 6: if (QTX) contract(std::integral_constant<int, QTX ? 6 : 1>{}); break;
            case 7: if (QTX) contract(std::integral_constant<int, QTX ? 7 : 1>{}); break;
            default: if (QTX) contract(std::integral_constant<int, QTX ? 8 : 1>{}); break;
          }
        }
        if (SK == SK_COUNT) {
          // deterministic scatter: warp gw owns buckets b % GW == gw; rows of a
          // bucket are added in ascending row order (proj/src/sketch.cpp:54-58)
          for (int g32 = 0; g32 < T / 32; ++g32) {
            const int r = g32 * 32 + lane;
            const bool rv = r < valid;
            const uint32_t code = rv ? stC[r] : 0u;
            const int bk = (int)(code & 0x7fffffffu) - a.bucket_lo;
            const bool mine = rv && bk >= 0 && bk < mh && (bk % GW) == gw;
            const unsigned key = mine ? (unsigned)bk : (0x80000000u | (unsigned)lane);
            const unsigned grp = __match_any_sync(0xffffffffu, key);
            if (mine && (__ffs(grp) - 1) == lane) {
              unsigned m = grp;
              while (m) {
                const int q = __ffs(m) - 1;
                m &= m - 1;
                const int rq = g32 * 32 + q;
                const double sg = (stC[rq] & 0x80000000u) ? -1.0 : 1.0;
                for (int c = 0; c < K; ++c)
                  cacc[bk + c * mh] = tiny::add(cacc[bk + c * mh], tiny::mul(sg, X[c * S + so(rq, KP)]));
              }
            }
          }
        }
        PP_MARK(5);
        if (XIN && STORE && stc < K) ptx::bulk_wait_read0();  // the X columns live in the stage
        PP_MARK(6);
        release(it, s);
        PP_MARK(7);
      }
      if (STORE && stc < K) ptx::bulk_wait0();
    }

#if BO_PHASE_PROF
    if (lane == 0 && a.phase_prof) {
      constexpr int shape = NPRE * 4 + (UPD ? 2 : 0) + (QTX ? 1 : 0);
      const bool storer = !in_trsm_group && gw == 0;  // the warp that issues the bulk stores
      for (int i = 0; i < 11; ++i)
        if (!(storer && i == 4)) atomicAdd(a.phase_prof + shape * 16 + i, pp_acc[i]);
      if (storer) {
        atomicAdd(a.phase_prof + shape * 16 + 13, pp_acc[4]);
        atomicAdd(a.phase_prof + shape * 16 + 14, (unsigned long long)my_tiles);
        atomicAdd(a.phase_prof + shape * 16 + 15, pp_acc[2] + pp_acc[5]);
      }
      atomicAdd(a.phase_prof + shape * 16 + (in_trsm_group ? 12 : 11), (unsigned long long)my_tiles);  // warp-tiles per role
    }
#endif
    // ---- per-warp fragments -> shared, then fixed-order sum over warps
    ptx::named_bar_sync(1, NW * 32);  // all stages consumed: reuse stage memory
    double* red = stages;             // [NW][dm_len]
    const int dm_len = a.dm_len;
    for (int e = lane; e < dm_len; e += 32) red[warp * dm_len + e] = 0.0;
    __syncwarp();
    if constexpr (TQ || TG) {
      // tail partial sums over the t4 lanes (fixed butterfly order)
#pragma unroll
      for (int c = 0; c < TN; ++c) {
        if (TQ) {
#pragma unroll
          for (int mi = 0; mi < MQT; ++mi) {
            tq[mi][c] += __shfl_xor_sync(0xffffffffu, tq[mi][c], 1);
            tq[mi][c] += __shfl_xor_sync(0xffffffffu, tq[mi][c], 2);
          }
        }
        if (TG) {
          tg[c] += __shfl_xor_sync(0xffffffffu, tg[c], 1);
          tg[c] += __shfl_xor_sync(0xffffffffu, tg[c], 2);
        }
      }
      if (TG) {
        tgg += __shfl_xor_sync(0xffffffffu, tgg, 1);
        tgg += __shfl_xor_sync(0xffffffffu, tgg, 2);
      }
    }
    if (QTX) {
#pragma unroll
      for (int mi = 0; mi < MQT; ++mi)
#pragma unroll
        for (int nj = 0; nj < NT; ++nj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = mi * 8 + g, j = nj * 8 + 2 * t4 + e;
            if (i < a.ld_q && j < 16) red[warp * dm_len + a.off_q + i + j * a.ld_q] = accq[mi][nj][e];
          }
      if constexpr (TQ) {
        // this launch's Q-tile count chose either the DMMA tile or the tail: the
        // other one is all zeros, so the sum is exact
        __syncwarp();
#pragma unroll
        for (int mi = 0; mi < MQT; ++mi)
#pragma unroll
          for (int c = 0; c < TN; ++c) {
            const int i = mi * 8 + g;
            if (t4 == 0 && i < a.ld_q) red[warp * dm_len + a.off_q + i + (8 + c) * a.ld_q] += tq[mi][c];
          }
      }
    }
    if (ROWG) {
      if (lane == 0) {
        int e = 0;
#pragma unroll
        for (int i = 0; i < KC; ++i)
#pragma unroll
          for (int j = i; j < KC; ++j) {
            red[warp * dm_len + a.off_g + i + j * 16] = gacc[e];
            red[warp * dm_len + a.off_g + j + i * 16] = gacc[e];
            ++e;
          }
      }
    } else if (GRAM) {
#pragma unroll
      for (int mi = 0; mi < NTG; ++mi)
#pragma unroll
        for (int nj = 0; nj < NTG; ++nj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = mi * 8 + g, j = nj * 8 + 2 * t4 + e;
            if (mi <= nj) {
              red[warp * dm_len + a.off_g + i + j * 16] = accg[mi][nj][e];
              if (mi < nj) red[warp * dm_len + a.off_g + j + i * 16] = accg[mi][nj][e];
            }
          }
      if constexpr (TG) {
        if (t4 == 0) {
#pragma unroll
          for (int c = 0; c < TN; ++c) {
            red[warp * dm_len + a.off_g + g + (8 + c) * 16] = tg[c];
            red[warp * dm_len + a.off_g + (8 + c) + g * 16] = tg[c];
          }
          if (g < NPAIR) {
            red[warp * dm_len + a.off_g + (8 + pa) + (8 + pb) * 16] = tgg;
            red[warp * dm_len + a.off_g + (8 + pb) + (8 + pa) * 16] = tgg;
          }
        }
      }
    }
    if (SK == SK_GAUSS) {
#pragma unroll
      for (int mi = 0; mi < MST; ++mi)
#pragma unroll
        for (int nj = 0; nj < NT; ++nj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = mi * 8 + g, j = nj * 8 + 2 * t4 + e;
            if (i < a.ld_s && j < 16) red[warp * dm_len + a.off_s + i + j * a.ld_s] = accs[mi][nj][e];
          }
    }
    ptx::named_bar_sync(1, NW * 32);
    double* part = a.partials + (size_t)blockIdx.x * a.part_len;
    for (int e = tid; e < dm_len; e += NW * 32) {
      double sum = 0.0;
      for (int w = 0; w < NW; ++w) sum += red[w * dm_len + e];
      part[e] = sum;
    }
    if (SK == SK_COUNT) {
      // every slot of the partial is written (the columns past K with zeros):
      // the cross-CTA tree reads the whole block
      for (int e = tid; e < mh * 16; e += NW * 32) {
        const int i = e % mh, j = e / mh;
        part[a.off_s + i + j * a.ld_s] = j < K ? cacc[i + j * mh] : 0.0;
      }
    }
  }

  // ---- cross-CTA reduction (fixed two-level tree: deterministic)
  if (!cta_tree_reduce(a.partials, a.part_len, a.sums, a.counter)) return;
  if (a.fused_finalize) finalize_dev(a.fin, reinterpret_cast<double*>(smem_raw));
}

}  // namespace bo
