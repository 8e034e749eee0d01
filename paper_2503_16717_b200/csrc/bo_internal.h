// bo_internal.h — host-side objects behind the C ABI handles.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/bo_cuda.h"
#include "bo_common.cuh"

struct bo_ctx_s {
  int device = 0;
  unsigned long long* phase_prof = nullptr;  // diagnostic phase counters (bo_debug_phase_prof)
  int rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // halo exchanges of a sharded SpMV run here, overlapped with the interior
  // planes on `stream` (created lazily; ev_x: x ready, ev_halo: halos landed)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_x = nullptr, ev_halo = nullptr;
  void* nccl = nullptr;  // ncclComm_t
  // reductions go through the communicator (world > 1, or a size-1 NCCL
  // communicator created on request: the NCCL path on a single GPU)
  bool collective = false;
  bool has_comm = false;  // collectives through host callbacks (bo_ctx_create_comm)
  bo_comm_ops comm{};
  uint64_t n_global = 0, row_begin = 0, row_end = 0, n_local = 0, ld = 0;
  int num_sms = 0;
  size_t smem_optin = 0;
  // device workspace
  double* partials = nullptr;
  size_t partials_cap = 0;  // doubles
  double* sums = nullptr;
  size_t sums_cap = 0;
  unsigned* counter = nullptr;
  bo::DevStatus* status = nullptr;      // device
  bo::DevStatus* status_host = nullptr; // pinned
  double* tiny = nullptr;               // tiny-factor workspace (device)
  size_t tiny_cap = 0;
  double* tiny_host = nullptr;          // pinned mirror
  double* scratch[3] = {nullptr, nullptr, nullptr};  // ld x 16 tall scratch
  uint64_t launches = 0;
  uint64_t allreduces = 0;
  // profiling
  struct ProfRec {
    int kind, K, p, mh;
    uint64_t rows, bytes;
    cudaEvent_t e0, e1;
  };
  int profiling = 0;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  // sketch generator plan (seed-independent jump polynomials + chunk table,
  // device scratch for the per-build prefix and chunk windows)
  struct GenPlan {
    uint64_t key_total = 0;
    std::vector<std::pair<uint64_t, uint64_t>> key_segs;
    size_t nchunks = 0;
    size_t pre_off = 0;
    uint64_t* dev = nullptr;
    std::vector<uint64_t> prefix;
  } gen_plan;
  // one recycled tall sketch buffer (a Gaussian sketch is rebuilt every
  // restart cycle: cudaMalloc/cudaFree of ~1.4 GB each time would stall)
  void* spare_buf = nullptr;
  // one recycled basis slab and pinned snapshot area: a GMRES solve creates a
  // store of m + 1 columns (3.9 GB at 8e6 rows), and cudaMalloc / cudaFree /
  // cudaMallocHost of that every solve cost milliseconds
  double* spare_q = nullptr;
  size_t spare_q_bytes = 0;
  double* spare_snap = nullptr;
  size_t spare_bytes = 0;
  // stream-ordered pool for per-solve scratch (residual / panel vectors of a
  // GMRES solve, MPK and sketch temporaries): released memory stays reserved
  // (release threshold = max), so repeated solves allocate without a device
  // synchronisation or a page-mapping stall
  cudaMemPool_t pool = nullptr;
};

// scratch from the ctx pool, ordered on the ctx stream
inline cudaError_t ctx_alloc(bo_ctx_s* c, void** p, size_t bytes) {
  return cudaMallocFromPoolAsync(p, bytes, c->pool, c->stream);
}
inline void ctx_free(bo_ctx_s* c, void* p) {
  if (p) cudaFreeAsync(p, c->stream);
}

struct bo_sketch_s {
  bo_ctx ctx = nullptr;
  int kind = 0;
  uint64_t n = 0, mhat = 0, mc = 0;  // mc: count width (count / count_gauss)
  double* theta = nullptr;            // gaussian local rows (ld x mhat)
  uint64_t ldth = 0;
  size_t theta_bytes = 0;
  bool own_theta = true;
  uint32_t* code = nullptr;           // count codes (local rows)
  double* theta_g = nullptr;          // count_gauss dense stage (device, mc x mhat)
  std::vector<double> theta_g_host;
  // wide Count stages (bo_ops.cu count_apply_sorted): local rows sorted by
  // bucket (stable: ascending row within a bucket), sign in bit 31, bucket
  // offsets, and a device buffer for the bucket sums (mc x 16)
  uint32_t* perm = nullptr;
  uint32_t* boff = nullptr;
  double* cnt = nullptr;
};

struct bo_basis_s {
  bo_ctx ctx = nullptr;
  uint64_t cap = 0, cols = 0;
  double* q = nullptr;  // device slab ld x cap
  size_t q_bytes = 0;   // its allocation (a recycled slab may be larger)
  std::vector<double> r, c;  // host cap x cap
  std::vector<char> seeded;
  std::vector<uint64_t> bounds;
  uint64_t bp_lo = 0;
  std::vector<double> sk;  // sketched history sk_rows x sk_cols
  uint64_t sk_rows = 0, sk_cols = 0;
  uint64_t ledger[4] = {0, 0, 0, 0};
  // the arguments of the last push_panel (bo_basis_last_push: lets a host
  // BasisStore replay the push with the reference's own arithmetic)
  std::vector<double> last_proj, last_diag;
  uint64_t last_base = 0, last_k = 0;
  int last_overlap = 0;
  // Deferred mode (bo_bcgs2_enqueue / bo_basis_sync): the device runs the
  // enqueued calls back to back; each call's status word and output factors
  // are snapshotted into pinned slots, and the host-side bookkeeping
  // (push_panel, mark_seed, ledger) is replayed in program order at sync.
  // `cols` is speculative (the value after every pending call succeeds).
  struct Pending {
    int kind;  // 0: bcgs2 push, 1: mark_seed
    uint64_t col = 0, k = 0, cols_before = 0;
    bool overlap = false, first = false, rand = false;
    int slot = -1;
  };
  std::vector<Pending> pend;
  double* snap = nullptr;            // pinned [kSnapSlots][kSnapLen]
  int nsnap = 0;
  int deferred_code = 0;             // first failure drained by an accessor, reported by the next sync
  bo_status deferred_st{};
  uint64_t deferred_call = 0;
};

struct bo_op_s {
  bo_ctx ctx = nullptr;
  int kind = 0;  // 0 csr, 1 constant-coefficient stencil (Laplacian, convection-diffusion)
  double coef[7] = {0, 0, 0, 0, 0, 0, 0};  // stencil coefficients, ascending column order
  int dims = 0;
  uint64_t k = 0;
  uint64_t ncols = 0;
  int* row_ptr = nullptr;  // local CSR (int32 offsets / int32 local-or-global cols)
  int* col = nullptr;
  double* val = nullptr;
  uint64_t nnz = 0;
  double a_fro = 0.0;      // ||A||_F (global)
  // halo (world > 1): rows needed below/above the shard
  uint64_t halo_lo = 0, halo_hi = 0;
  uint64_t peer_need_lo = 0, peer_need_hi = 0;  // rows the neighbours need from us
  double* xext = nullptr;  // extended x: [halo_lo | local | halo_hi]
  double a_fro_local2 = 0.0;  // sum of squared values of this shard's rows
};

namespace bo {
namespace host {

//           name              NPRE UPD  NPOST QTX  GRAM  SK        STORE
#define BO_PASS_KINDS(X)                                               \
  X(QTX, 0, false, 0, true, false, SK_NONE, false)                     \
  X(QTX_GRAM, 0, false, 0, true, true, SK_NONE, false)                 \
  X(GRAM, 0, false, 0, false, true, SK_NONE, false)                    \
  X(SKG, 0, false, 0, false, false, SK_GAUSS, false)                   \
  X(SKC, 0, false, 0, false, false, SK_COUNT, false)                   \
  X(UPD_ST, 0, true, 0, false, false, SK_NONE, true)                   \
  X(UPD_GRAM_ST, 0, true, 0, false, true, SK_NONE, true)               \
  X(UPD_SKG_ST, 0, true, 0, false, false, SK_GAUSS, true)              \
  X(UPD_SKC_ST, 0, true, 0, false, false, SK_COUNT, true)              \
  X(P1_GRAM, 1, false, 0, false, true, SK_NONE, false)                 \
  X(P2_QTX, 2, false, 0, true, false, SK_NONE, false)                  \
  X(P2_UPD_GRAM_ST, 2, true, 0, false, true, SK_NONE, true)            \
  X(P1_ST, 1, false, 0, false, false, SK_NONE, true)                   \
  X(P2_ST, 2, false, 0, false, false, SK_NONE, true)                    \
  X(UPD_POST_ST, 0, true, 1, false, false, SK_NONE, true)              \
  X(P2_UPD_ST, 2, true, 0, false, false, SK_NONE, true)                \
  X(P1_QTX, 1, false, 0, true, false, SK_NONE, false)                  \
  X(P1_UPD_GRAM_ST, 1, true, 0, false, true, SK_NONE, true)            \
  X(P1_UPD_ST, 1, true, 0, false, false, SK_NONE, true)

enum PassKind {
#define X(nm, a, b, c, d, e, f, g) PK_##nm,
  BO_PASS_KINDS(X)
#undef X
      PK_COUNT
};
struct KindInfo {
  int npre;
  bool upd;
  int npost;
  bool qtx, gram;
  int sk;
  bool store;
};
inline const KindInfo kKindInfo[PK_COUNT] = {
#define X(nm, a, b, c, d, e, f, g) {a, b, c, d, e, f, g},
    BO_PASS_KINDS(X)
#undef X
};

struct PassReq {
  int kind;
  int K;
  const double* V;
  uint64_t ldv;
  const double* Q = nullptr;
  uint64_t ldq = 0;
  int p = 0;
  bo_sketch sk = nullptr;
  double* out = nullptr;
  uint64_t ldo = 0;
  const double* Rpre0 = nullptr;
  const double* Rpre1 = nullptr;
  const double* Rpost = nullptr;
  const double* Cm = nullptr;
  FinArgs fin{};
  int pass_id = 0;
  bool exact = false;  // bit-exact substitution (standalone apply_inv_upper only)
  int bucket_lo = 0;   // count sketch: first bucket of this pass (chunked bucket ranges)
  int bucket_n = 0;    // buckets in this pass (0 = all)
};


// tiny workspace layout (doubles) — all K x K factors have ld 16
// projection coefficient blocks (p x K) have ld LDC = 256 (p <= 255 basis columns)
constexpr int LDC = 256;
// The device status word and the factors a deferred call's host bookkeeping
// needs (Rin of a first panel; R_jj and the coefficients otherwise) lead the
// workspace contiguously, so a call's snapshot is ONE device-to-host copy.
constexpr int OFF_STATUS = 0, OFF_RIN = 8, OFF_RJJ = OFF_RIN + 256, OFF_COEF = OFF_RJJ + 256,
              OFF_R1 = OFF_COEF + LDC * 16, OFF_R2 = OFF_R1 + 256, OFF_R3 = OFF_R2 + 256, OFF_G = OFF_R3 + 256,
              OFF_R4 = OFF_G + 256, OFF_C1 = OFF_R4 + 512, OFF_C2 = OFF_C1 + LDC * 16, OFF_S = OFF_C2 + LDC * 16,
              TINY_LEN = OFF_S + 8192;
static_assert(sizeof(bo::DevStatus) <= OFF_RIN * sizeof(double), "status word slot");
// deferred-call snapshots (bo_bcgs2_enqueue): the leading workspace block
// [status | Rin | R_jj | coefficients], copied as one range
constexpr int kSnapSlots = 64, kSnapStatus = OFF_STATUS, kSnapRin = OFF_RIN, kSnapRjj = OFF_RJJ,
              kSnapCoef = OFF_COEF, kSnapLen = OFF_COEF + LDC * 16;

// NCCL, loaded lazily with dlopen (prefers the copy torch already mapped)
struct NcclUniqueId {  // ncclUniqueId (nccl.h:39)
  char internal[128];
};
struct NcclApi {
  void* h = nullptr;
  int (*GetUniqueId)(void* id) = nullptr;
  // ncclCommInitRank takes the 128-byte ncclUniqueId BY VALUE (nccl.h:171);
  // declaring it as a pointer would pass the address where NCCL reads the
  // struct from the stack
  int (*CommInitRank)(void** comm, int nranks, NcclUniqueId id, int rank) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  bool ok = false;
};
NcclApi& nccl();
constexpr int kNcclFloat64 = 8;  // ncclDouble
constexpr int kNcclUint64 = 5;   // ncclUint64
constexpr int kNcclSum = 0;

int set_st(bo_status* st, int code, long long index, double pivot, const char* fmt, ...);
// complete any deferred calls of the store (keeps their first error for bo_basis_sync)
int basis_drain(bo_basis b);
// return BO_CUDA with the error text from a bo_status*-returning function
#define CU(call)                                                                            \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return set_st(st, BO_CUDA, 0, 0.0, "CUDA error %s at %s:%d", cudaGetErrorString(e_), \
                    __FILE__, __LINE__);                                                    \
  } while (0)
#define TRY(expr)                 \
  do {                            \
    int rc_ = (expr);             \
    if (rc_ != BO_OK) return rc_; \
  } while (0)
void ok_st(bo_status* st);
int run_pass(bo_ctx ctx, PassReq& r, bo_status* st);        // splits p > 64 into chunks
int run_pass_single(bo_ctx ctx, PassReq& r, bo_status* st);
inline double* T_(bo_ctx ctx, int off) { return ctx->tiny + off; }
int reset_status(bo_ctx ctx, bo_status* st);
int fetch(bo_ctx ctx, bool tiny, bo_status* st);
int stage_input(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, int slot, const double** out,
                uint64_t* ldout, bo_status* st);
bool out_ok(bo_ctx ctx, const double* q, uint64_t ldq);
int dev_error(bo_ctx ctx, const char* chol_ctx, bo_status* st);
int dev_intra(bo_ctx ctx, const double* v, uint64_t ldv, int K, int intra, bo_sketch sk, double* q, uint64_t ldq,
              bo_status* st);
int dev_cholqr(bo_ctx ctx, const double* v, uint64_t ldv, int K, double* q, uint64_t ldq, int Rslot, int pass_id,
               bo_status* st);
int dev_project(bo_basis b, const double* v, uint64_t ldv, int K, uint64_t lo, uint64_t hi, double* vhat,
                uint64_t ldvh, int Cslot, int pass_id, bo_status* st);
int sketch_pass(bo_sketch sk, const double* v, uint64_t ldv, int K, int pass_id, int extra_ops, bo_status* st);
void push_panel_host(bo_basis b, uint64_t k, const double* proj, uint64_t ldp, const double* diag, uint64_t ldd,
                     bool overlap);
uint64_t derive_seed(uint64_t base, uint64_t stream);
// the context's collective transport (NCCL, or bo_comm_ops callbacks)
int comm_allreduce(bo_ctx ctx, double* buf, size_t n, bo_status* st);
// count_gauss dense stage for a sketch seed, drawn ahead on a host thread
void prefetch_theta_g(uint64_t seed, uint64_t mc, uint64_t mhat);
std::vector<double> take_theta_g(uint64_t seed, uint64_t mc, uint64_t mhat);
int comm_allgather_u64(bo_ctx ctx, const uint64_t* send, size_t n, uint64_t* recv, bo_status* st);
int comm_exchange(bo_ctx ctx, int nops, const bo_p2p_op* ops, bo_status* st, cudaStream_t s = nullptr);
int op_apply(bo_op op, const double* x, double* y, bo_status* st);
int sketch_to_host(bo_sketch th, const double* v, uint64_t ldv, int K, std::vector<double>& S, bo_status* st);
inline uint64_t round_up(uint64_t x, uint64_t m) { return (x + m - 1) / m * m; }

}  // namespace host
}  // namespace bo
