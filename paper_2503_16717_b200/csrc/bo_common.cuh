// bo_common.cuh — shared device-side types for the block-orthogonalization
// kernels (status word, tiny-factor workspace layout, pass descriptors).
#pragma once
#include <cstdint>

namespace bo {

constexpr int kMaxK = 16;        // panel width bound of the streaming passes (s <= 15)
constexpr int kRld = 16;         // leading dimension of every K x K factor in the workspace
constexpr int kMaxPTile = 64;    // max projection columns per streaming pass
// Consumer warps per CTA (+ 1 producer warp).  Update passes use 8 so that
// the 16 eight-row groups of a 128-row tile split evenly (9 warps cap each
// thread at 168 registers, which those kernels fit); every other pass uses 7
// so that 8 warps share the SM and a thread may use up to 255 registers.
#ifndef BO_PRODUCER_WARP
#define BO_PRODUCER_WARP 1
#endif
#ifndef BO_NW_UPD
#define BO_NW_UPD 8
#endif
#ifndef BO_NW_OTHER
#define BO_NW_OTHER (BO_PRODUCER_WARP ? 7 : 8)
#endif
// Consumer warps per CTA.  Default: a dedicated producer warp + 7 consumers
// (8 warps: up to 255 registers a thread), 8 consumers for update passes (the
// 16 eight-row groups of a tile split evenly; 168 registers).  The
// producer-less variant (BO_PRODUCER_WARP=0: the last warp to release a stage
// issues its refill) measured 4% slower over the C2 sequence.
// Pre-solve passes (two row-solve warps + a U/S/R group): the consumer count
// of the projection (P2_QTX) and update (P2_UPD_*) kinds.  The update kinds
// use 2 + 8: two U/S/R warps on every SM sub-partition (11 warps, 186
// registers; they need 132).  Measured on the C2 sequence (scripts/ab_passes.sh):
// P2_UPD_GRAM_ST 3.92 -> 3.68 ms; 2 + 6 leaves two sub-partitions with one
// U/S/R warp and a solve warp, 4 + 8 starves the update of registers, and
// P2_QTX is best at 2 + 5 (2 + 4 wins only at p >= 44, 4 + 4 and 3 + 4 lose).
#ifndef BO_NW_PRE_QTX
#define BO_NW_PRE_QTX BO_NW_OTHER
#endif
#ifndef BO_NW_PRE_UPD
#define BO_NW_PRE_UPD 10
#endif
__host__ __device__ constexpr int consumer_warps(bool upd, bool pre_qtx = false, bool pre_upd = false) {
  return pre_qtx ? BO_NW_PRE_QTX : pre_upd ? BO_NW_PRE_UPD : upd ? BO_NW_UPD : BO_NW_OTHER;
}
__host__ __device__ constexpr int pass_threads(bool upd, bool pre_qtx = false, bool pre_upd = false) {
  return (consumer_warps(upd, pre_qtx, pre_upd) + BO_PRODUCER_WARP) * 32;
}
constexpr int kMaxStages = 24;
// warps per CTA of the tile-per-warp engine (bo_tpw.cuh): one per SM sub-partition
#ifndef BO_TPW_NW
#define BO_TPW_NW 4
#endif   // shared-memory stage ring depth bound

// Tile geometry.  A tile of T rows is staged as T / R sub-tiles of R <= 128
// rows; within a sub-tile an operand block is column-major with the padded
// column stride S = R + 4 (conflict-free DMMA fragment loads), and the
// sub-tiles of one operand block follow each other.  Element (c, r) of a block
// of P columns sits at (r / R) * P * S + c * S + r % R.  Every sub-tile is one
// 2-D TMA box of S rows, so one tensor map serves every T.
template <int T>
struct TileGeom {
  static constexpr int R = T < 128 ? T : 128;
  static constexpr int NSUB = T / R;
  static constexpr int S = R + 4;
};
__host__ __device__ inline int tile_sub_rows(int T) { return T < 128 ? T : 128; }
__host__ __device__ inline int tile_stride(int T) { return tile_sub_rows(T) + 4; }

struct StageLayout {
  int offV, offQ, offT, offC, stage;
};
__host__ __device__ inline int ru16(int x) { return (x + 15) & ~15; }
// Shared-memory stage layout (doubles): every operand block starts on a
// 128-byte boundary (TMA destination alignment).
// pad: operand blocks hold a multiple of 8 columns (zero padding for the MMA
// tiles); row-mode passes (no tensor-core reads) pack the columns tightly.
__host__ __device__ inline StageLayout stage_layout(int K, int ncolQ, int ncolT, bool count, int T, bool pad = true) {
  const int S = tile_stride(T), nsub = T / tile_sub_rows(T);
  StageLayout L;
  L.offV = 0;
  L.offQ = ru16((pad ? ((K + 7) & ~7) : K) * S * nsub);
  L.offT = L.offQ + ru16(((ncolQ + 7) & ~7) * S * nsub);
  L.offC = L.offT + ru16(((ncolT + 7) & ~7) * S * nsub);
  L.stage = L.offC + (count ? ru16(T / 2) : 0);
  return L;
}

// device status word (mirrors the reference exception set, errors.hpp:12-92)
struct DevStatus {
  int code;        // bo_code
  int pass;        // which pass raised it (for ledger reconstruction)
  long long step;  // 1-based Cholesky step / zero-diagonal index
  double pivot;
};

enum StatusCode : int {
  ST_OK = 0,
  ST_CHOLESKY = 1,
  ST_SINGULAR = 2,
};

// sketch payload kinds staged by the streaming passes
enum SketchStage : int { SK_NONE = 0, SK_GAUSS = 1, SK_COUNT = 2 };

// finalize micro-ops (bit mask), executed by one CTA after the cross-CTA /
// cross-rank reduction of a pass
enum FinOp : int {
  FIN_COPY_Q = 1 << 0,     // QTX block -> Cq (ld ldcq)
  FIN_CHOL = 1 << 1,       // GRAM block -> cholesky -> Rchol  (fails: ST_CHOLESKY)
  FIN_HH = 1 << 2,         // SK block (or Theta_g^T SK) -> Householder R -> Rhh (fails: ST_SINGULAR)
  FIN_PIP = 1 << 3,        // G = GRAM - QTX^T QTX before FIN_CHOL; QTX -> Cq
  FIN_COEFF = 1 << 4,      // coeffs = C1 + C2 * Rin ; rjj = Rchol * Rin   (bcgs2 push data)
  FIN_MULT = 1 << 5,       // rjj = Rchol * Rin (first panel)
  FIN_COPY_G = 1 << 6,     // GRAM block -> Gout (16 x 16)
  FIN_COPY_S = 1 << 7,     // SK block (after Theta_g) -> Sout (mh x K, ld mh)
  FIN_CHECK_DIAG = 1 << 8  // zero diagonal of Rin_check -> ST_SINGULAR
};

struct FinArgs {
  int ops;
  int K, p, mh, mc;        // panel width, QTX rows of this pass, sketch rows, count width (count-gauss)
  int p_total;             // rows of the full projection block (chunked passes), >= q_row_off + p
  int q_row_off;           // row offset of this pass's QTX block inside Cq
  int pass_id;
  double pivot_tol;
  const double* sums;      // reduced partials
  int off_q, ld_q;         // QTX block offset / ld inside sums
  int off_g;               // GRAM block offset (16 x 16)
  int off_s, ld_s;         // SK block offset / ld inside sums
  const double* theta_g;   // count-gauss dense stage, mc x mh (ld mc)
  double* Cq;              // FIN_COPY_Q / FIN_PIP destination
  int ldcq;
  double* Rchol;           // FIN_CHOL output (16 x 16)
  double* Rhh;             // FIN_HH output
  const double* C1;        // FIN_COEFF inputs
  const double* C2;
  int ldc;
  const double* Rin;       // inner R (16 x 16)
  double* coeffs;          // FIN_COEFF outputs (ld ldc)
  double* rjj;
  double* Gout;
  double* Sout;
  const double* Rcheck;
  DevStatus* status;
};

// one streaming pass over the local rows
struct PassArgs {
  long long nrows;
  int ntiles;
  int K;
  const double* V;
  long long ldv;
  const double* Q;
  long long ldq;
  int p;
  const double* Th;        // gaussian sketch rows (local rows x mh)
  long long ldth;
  const uint32_t* code;    // count sketch: bucket | sign bit (local rows)
  int mh;                  // sketch rows (gauss) / buckets of this pass (count)
  int bucket_lo;           // count: first bucket handled by this pass
  double* out;
  long long ldo;
  const double* Rpre0;     // first pre-TRSM factor (16 x 16)
  const double* Rpre1;     // second pre-TRSM factor
  const double* Rpost;     // post-update TRSM factor
  const double* Cm;        // update coefficients p x K (ld ldc)
  int ldc;
  double* partials;        // [grid][part_len]
  double* sums;            // [part_len]
  unsigned* counter;
  int part_len, off_q, ld_q, off_g, off_s, ld_s;
  int nstages;
  int gaw;                 // solve warps of a pre-solve projection pass (0: the build's default)
  int gw_active;           // U/S/R warps of a pre-solve projection pass (0: all the others)
  int nstages_v;           // panel-ring depth of the decoupled pre-solve passes (bo_pass.cuh DEC)
  int prefetch_tiles;      // L2 prefetch lookahead beyond the stage ring (tiles)
  int region0_dbl;         // doubles of shared region 0 (stage ring / reduction / finalize scratch)
  int dm_len;              // tensor-core partial length (excludes the count block)
  int fused_finalize;      // 1: last CTA runs FinArgs
  DevStatus* status;
  unsigned long long* phase_prof;  // diagnostic builds (-DBO_PHASE_PROF=1): [16 pass shapes][16 counters]
  FinArgs fin;
};

}  // namespace bo
