// bo_capi.cu — C ABI implementation: context, pass orchestration, sketches,
// intra-block and block orthogonalization (include/bo_cuda.h).
//
// Host code here only sequences device work; every tall (n-row) operation is
// a CUDA kernel (bo_pass.cuh, bo_sketch_gen.cuh, bo_spmv.cuh) and every tiny
// factorization runs on device inside the pass epilogue (bo_tiny.cuh).  The
// host mirrors BasisStore's small R/C bookkeeping exactly as the reference
// (proj/src/block_orth.cpp:10-153).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <future>
#include <map>
#include <mutex>
#include <random>
#include <set>
#include <unordered_map>

#include "bo_internal.h"
#include "bo_pass.cuh"
#include "bo_pass_inst.h"
#include "bo_sketch_gen.cuh"
#include "mt64_jump.h"

using namespace bo;
using namespace bo::host;

// ===========================================================================
// status helpers
// ===========================================================================
namespace bo {
namespace host {

int set_st(bo_status* st, int code, long long index, double pivot, const char* fmt, ...) {
  if (st) {
    st->code = code;
    st->index = index;
    st->pivot = pivot;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(st->msg, sizeof st->msg, fmt, ap);
    va_end(ap);
  }
  return code;
}
void ok_st(bo_status* st) {
  if (st) {
    st->code = BO_OK;
    st->index = 0;
    st->pivot = 0.0;
    st->msg[0] = 0;
  }
}


// ---------------------------------------------------------------------------
// NCCL, loaded lazily (prefer the copy torch already mapped)
// ---------------------------------------------------------------------------
NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      api.h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
      if (api.h) break;
    }
    if (!api.h)
      for (const char* nm : names) {
        api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        if (api.h) break;
      }
    if (!api.h) return;
    api.GetUniqueId = (int (*)(void*))dlsym(api.h, "ncclGetUniqueId");
    api.CommInitRank = (int (*)(void**, int, NcclUniqueId, int))dlsym(api.h, "ncclCommInitRank");
    api.AllReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(
        api.h, "ncclAllReduce");
    api.CommDestroy = (int (*)(void*))dlsym(api.h, "ncclCommDestroy");
    api.GetErrorString = (const char* (*)(int))dlsym(api.h, "ncclGetErrorString");
    api.Send = (int (*)(const void*, size_t, int, int, void*, cudaStream_t))dlsym(api.h, "ncclSend");
    api.Recv = (int (*)(void*, size_t, int, int, void*, cudaStream_t))dlsym(api.h, "ncclRecv");
    api.GroupStart = (int (*)())dlsym(api.h, "ncclGroupStart");
    api.GroupEnd = (int (*)())dlsym(api.h, "ncclGroupEnd");
    api.AllGather = (int (*)(const void*, void*, size_t, int, void*, cudaStream_t))dlsym(api.h, "ncclAllGather");
    api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.CommDestroy;
  });
  return api;
}

}  // namespace host
}  // namespace bo

// ===========================================================================
// pass kinds and dispatch
// ===========================================================================
namespace bo {
namespace host {


// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
  }();
  return fn;
}
// 2-D map over `cols` columns of `rows` doubles (leading dimension ld), box = S rows x cols
int make_tmap(CUtensorMap* m, const double* base, uint64_t rows, uint64_t cols, uint64_t ld, int S, bo_status* st) {
  std::memset(m, 0, sizeof *m);
  if (!base || cols == 0) return BO_OK;
  auto fn = encode_fn();
  if (!fn) return set_st(st, BO_CUDA, 0, 0.0, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {rows, cols};
  const cuuint64_t strides[1] = {ld * 8};
  const cuuint32_t box[2] = {(cuuint32_t)S, (cuuint32_t)cols};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_st(st, BO_CUDA, (long long)r, 0.0, "cuTensorMapEncodeTiled failed (%d): rows=%llu cols=%llu ld=%llu",
                  (int)r, (unsigned long long)rows, (unsigned long long)cols, (unsigned long long)ld);
  return BO_OK;
}

// The pass-kernel instantiations live in their own translation units
// (bo_pass_inst.cu, compiled once per (NT|KC, T) combination in parallel).
PassFn get_pass_fn(int nt, int T, int kind, bool exact, int K) {
  if (exact)  // standalone apply_inv_upper: bit-exact substitution (dense.cpp:166-186)
    return pass_fn_exact(nt);
  const KindInfo& ki = kKindInfo[kind];
  if (ki.npre > 0 || ki.npost > 0) {
    PassFn f = nullptr;
    if (T == 256) {
      if (K == 6) f = pass_fn_kc6_t256(kind);
      if (K == 11) f = pass_fn_kc11_t256(kind);
      if (K == 16) f = pass_fn_kc16_t256(kind);
      if (K == 13) f = pass_fn_kc13_t256(kind);
    } else if (T == 128) {
      if (K == 6) f = pass_fn_kc6_t128(kind);
      if (K == 11) f = pass_fn_kc11_t128(kind);
      if (K == 16) f = pass_fn_kc16_t128(kind);
      if (K == 13) f = pass_fn_kc13_t128(kind);
    } else {
      if (K == 6) f = pass_fn_kc6_t64(kind);
      if (K == 11) f = pass_fn_kc11_t64(kind);
      if (K == 16) f = pass_fn_kc16_t64(kind);
      if (K == 13) f = pass_fn_kc13_t64(kind);
    }
    if (f) return f;
  }
  if (nt == 1) return T == 256 ? pass_fn_nt1_t256(kind) : T == 128 ? pass_fn_nt1_t128(kind) : pass_fn_nt1_t64(kind);
  return T == 256 ? pass_fn_nt2_t256(kind) : T == 128 ? pass_fn_nt2_t128(kind) : pass_fn_nt2_t64(kind);
}

// launch one streaming pass (+ its reduction / finalize) on the ctx stream
int run_pass_single(bo_ctx ctx, PassReq& r, bo_status* st) {
  const KindInfo& ki = kKindInfo[r.kind];
  PassArgs a{};
  a.nrows = (long long)ctx->n_local;
  a.K = r.K;
  a.V = r.V;
  a.ldv = (long long)r.ldv;
  a.Q = r.Q;
  a.ldq = (long long)r.ldq;
  a.p = r.p;
  a.out = r.out;
  a.ldo = (long long)r.ldo;
  a.Rpre0 = r.Rpre0;
  a.Rpre1 = r.Rpre1;
  a.Rpost = r.Rpost;
  a.Cm = r.Cm;
  a.ldc = LDC;
  a.status = ctx->status;
  a.phase_prof = ctx->phase_prof;
  int mh = 0;
  if (ki.sk == SK_GAUSS) {
    a.Th = r.sk->theta;
    a.ldth = (long long)r.sk->ldth;
    mh = (int)r.sk->mhat;
  } else if (ki.sk == SK_COUNT) {
    a.code = r.sk->code;
    mh = r.bucket_n ? r.bucket_n : (int)r.sk->mc;
  }
  a.mh = mh;
  a.bucket_lo = r.bucket_lo;
  if (r.p > kMaxPTile) return set_st(st, BO_INVALID, 0, 0.0, "projection range of %d columns exceeds %d", r.p, kMaxPTile);
  if (r.K < 1 || r.K > kMaxK) return set_st(st, BO_INVALID, 0, 0.0, "panel width %d outside [1, %d]", r.K, kMaxK);
  if (ki.sk == SK_GAUSS && mh > 32) return set_st(st, BO_INVALID, 0, 0.0, "gaussian sketch of %d rows exceeds 32", mh);
  // partial layout [QTX][GRAM][SK]
  a.off_q = 0;
  a.ld_q = ki.qtx ? (int)round_up(std::max(r.p, 1), 8) : 0;
  a.off_g = a.off_q + a.ld_q * 16;
  a.off_s = a.off_g + (ki.gram ? 256 : 0);
  a.ld_s = ki.sk == SK_GAUSS ? (int)round_up(mh, 8) : (ki.sk == SK_COUNT ? mh : 0);
  a.part_len = a.off_s + a.ld_s * 16;
  const int dm_len = ki.sk == SK_COUNT ? a.off_s : a.part_len;
  if (a.part_len == 0) a.part_len = 1;

  const int nt = r.K <= 8 ? 1 : 2;
  const bool pre_qtx = ki.npre > 0 && ki.qtx, pre_upd = ki.npre > 0 && ki.upd;  // bo_pass.cuh consumer counts
  const size_t avail = std::min<size_t>(ctx->smem_optin, 227 * 1024) - 1024;  // static smem headroom
  // Tile choice: the largest tile (256 / 128 / 64 rows) whose stage ring is
  // at least double-buffered.  Per-tile synchronisation costs ~0.3-1 us
  // (ncu + T = 64 vs 128 sweeps), so larger tiles amortise it; the row-mode
  // Gram (ROWG) needs 128-row tiles; BO_TILE forces a size.
  static const int tile_env = [] {
    const char* e = getenv("BO_TILE");
    return e ? atoi(e) : 0;
  }();
  static const int tile_max = [] {
    const char* e = getenv("BO_MAX_TILE");
    return e ? atoi(e) : 256;
  }();
  // BO_TILE_PRE: force the tile of the pre-solve passes with a projection range only (diagnostic)
  static const int tile_pre = [] {
    const char* e = getenv("BO_TILE_PRE");
    return e ? atoi(e) : 0;
  }();
  int tile_env_k = (tile_pre && ki.npre > 0 && (ki.qtx || ki.upd)) ? tile_pre : tile_env;
  const bool rowg_kind = !r.exact && ki.npre > 0 && ki.gram && !ki.qtx && !ki.upd && ki.sk == SK_NONE &&
                         !ki.store && ki.npost == 0 && (r.K == 6 || r.K == 11);
  int T = 0, NS = 0;
  size_t region0 = 0, total = 0;
  // Pre-solve passes (bo_pass.cuh SPLIT) consume a tile in two hand-offs
  // (solve warps, then the U/S/R group), so they want a deeper ring than
  // double buffering; BO_NS_PRE sets the stage count they try for first.
  // A third stage helps only while the tile stays >= 128 rows (measured on the
  // C2 sequence, scripts/ab_passes.sh: P2_QTX p = 11 419 -> 373 us, p <= 33
  // P2_UPD_GRAM_ST -15 us; forcing 64-row tiles at p >= 44 lost 200 us each).
  static const int ns_pre = [] {
    const char* e = getenv("BO_NS_PRE");
    return e ? std::max(2, atoi(e)) : 3;
  }();
  // (a third stage for the other passes measured no better: QTX / UPD_SKG_ST
  // within +-2% at every p, sequence +0.3 ms at 3 stages)
  const int want_hi = (ki.npre > 0 && !rowg_kind) ? ns_pre : 2;
  // Decoupled rings (bo_pass.cuh DEC): pre-solve passes with a projection
  // range keep their panel tiles in a separate ring, vla tiles deeper than
  // the basis ring.  BO_DEC_RING=0 at build time restores joint stages.
  const bool dec_ok = BO_DEC_RING && BO_PRODUCER_WARP && ki.npre > 0 && (ki.qtx || ki.upd) && !r.exact;
  static const int vla = [] {
    const char* e = getenv("BO_VLA");
    return e ? std::max(1, atoi(e)) : 1;  // measured: 1 beats 2, 3 and 4
  }();
  static const int dec_env = [] {
    const char* e = getenv("BO_DEC");  // -1: never, 1: whenever eligible, 0 (default): when joint stages give <= 2
    return e ? atoi(e) : 0;
  }();
  int NSV = 0;
  auto choose = [&](bool dec) {
    T = 0;
    NS = NSV = 0;
    for (int want_ns : {want_hi, 2, 1}) {
      for (int tt : {256, 128, 64}) {
        if (T) break;
        if (want_ns > 2 && tt < 128 && !tile_env_k) continue;
        if (r.exact && tt != 64) continue;
        if (tile_env_k && tt != tile_env_k) continue;
        if (tt > tile_max) continue;
        if (rowg_kind && tt != 128 && !tile_env_k) continue;
        const int S = tile_stride(tt), nsub = tt / tile_sub_rows(tt);
        // row-mode Gram (bo_pass.cuh ROWG): unpadded stages, no X tile
        const bool rowg = rowg_kind && tt == 128;
        const StageLayout SL = stage_layout(r.K, (ki.qtx || ki.upd) ? r.p : 0, ki.sk == SK_GAUSS ? mh : 0,
                                            ki.sk == SK_COUNT, tt, !rowg);
        const size_t stage = (size_t)SL.stage * 8;
        // X tile.  The kernel only uses one for a post-solve without an update
        // (bo_pass.cuh XT && !XIN): update and pre-solve passes compute X in
        // place in the stage.  The reservation is kept for pre-solve passes as a
        // cap on their ring: releasing it lets them pick 256-row tiles and deeper
        // rings, which measured slower (P1_ST 227 -> 252 us, C2 sequence +0.4 ms).
        const bool xt = (ki.npre > 0 || ki.npost > 0) && !rowg && !(ki.upd && ki.npre == 0) && !dec;
        // row-major copies of the solve factors (bo_pass.cuh RFT) in K-specialised solve passes
        const bool rft = !r.exact && (ki.npre > 0 || ki.npost > 0) && (r.K == 6 || r.K == 11 || r.K == 13 || r.K == 16);
        const size_t fixed = (xt ? 2 * (size_t)nt * 8 * S * 8 * nsub : 0) + (3 * 256 + 48 + (rft ? 3 * 256 : 0)) * 8 +
                             (ki.sk == SK_COUNT ? (size_t)mh * r.K * 8 : 0) + 4 * kMaxStages * 8;
        const size_t need_red = (size_t)consumer_warps(ki.upd, pre_qtx, pre_upd) * dm_len * 8;
        const size_t need_fin = (1536 + (size_t)std::max(mh, 32) * 16 + 64) * 8;  // finalize_dev scratch
        if (avail <= fixed) continue;
        int ns = (int)std::min<size_t>(kMaxStages, (avail - fixed) / stage);
        size_t ring = (size_t)ns * stage;
        int nsv = 0;
        if (dec) {
          // basis ring of ns slots, panel ring of ns + vla slots
          const size_t vb = (size_t)SL.offQ * 8, qb = stage - vb;
          ns = avail - fixed > vla * vb ? (int)std::min<size_t>(kMaxStages - vla, (avail - fixed - vla * vb) / (qb + vb))
                                        : 0;
          nsv = ns + vla;
          ring = (size_t)ns * qb + (size_t)nsv * vb;
        }
        if (rowg) ns = ns / consumer_warps(false) * consumer_warps(false);  // one private sub-ring per warp
        if (ns < want_ns) continue;
        const size_t r0 = round_up(std::max({ring, need_red, need_fin}), 128);
        if (r0 + fixed > avail) continue;
        T = tt;
        NS = ns;
        NSV = nsv;
        region0 = r0;
        total = r0 + fixed;
      }
    }
  };
  // Decoupled rings (bo_pass.cuh DEC) where joint stages leave only a double
  // buffer: measured on the C2 sequence (scripts/ab_tail.sh), P2_QTX at
  // p = 44 / 55 734 / 810 -> 652 / 737 us and P2_UPD_GRAM_ST 883 / 939 -> 847 /
  // 908 us, while at p <= 33 (3-5 joint stages) they were 3-5% slower.
  // Narrow pre-solve passes (p <= 24): 256-row tiles with decoupled rings.
  // Their time is a per-tile cost, not bytes, so halving the
  // tile count pays: measured P1_QTX p = 11 / 22 391 / 455 -> 337 / 389 us,
  // P1_UPD_GRAM_ST 504 / 562 -> 463 / 512 us (wider ranges lose: one 256-row
  // basis slot only).
  static const int t256_maxp = [] {
    const char* e = getenv("BO_T256_MAXP");
    return e ? atoi(e) : 24;
  }();
  if (dec_ok && dec_env >= 0 && !tile_env_k && r.p <= t256_maxp) {
    tile_env_k = 256;
    choose(true);
    tile_env_k = 0;
    if (T && NS < 2) T = 0;
  }
  if (!T) choose(dec_ok && dec_env > 0);
  if (dec_ok && dec_env == 0 && T && NS <= 2 && NSV == 0) {
    const int T0 = T, NS0 = NS;
    const size_t r00 = region0, tot0 = total;
    choose(true);
    if (!T) T = T0, NS = NS0, NSV = 0, region0 = r00, total = tot0;
  }
  if (T == 0) return set_st(st, BO_INVALID, 0, 0.0, "pass does not fit in shared memory");
  if (total > avail) return set_st(st, BO_INVALID, 0, 0.0, "pass does not fit in shared memory (%zu bytes)", total);
  a.nstages = NS;
  a.nstages_v = NSV;
  {
    // one solve warp for single-solve projection passes with a wide basis
    // block (bo_pass.cuh gaw; measured on the C2 sequence, scripts/ab_tail.sh)
    static const int gaw_minp = [] {
      const char* e = getenv("BO_GAW1_MINP");
      return e ? atoi(e) : 25;
    }();
    a.gaw = (ki.npre == 1 && ki.qtx && T <= 128 && gaw_minp > 0 && r.p >= gaw_minp) ? 1 : 0;
    // narrow pre-solve projections: BO_QTX_GW_SMALLP=n contracts on n warps
    // (measured slower: p = 11 397 / 441 / 514 us with 5 / 4 / 3 warps, so the
    // pass is bound by latency, not by two warps sharing a DMMA pipe; off)
    static const int gw_small = [] {
      const char* e = getenv("BO_QTX_GW_SMALLP");
      return e ? atoi(e) : 0;
    }();
    a.gw_active = (ki.npre > 0 && ki.qtx && a.gaw == 0 && gw_small > 0 && r.p < gaw_minp) ? gw_small : 0;
  }
  {
    // bytes to keep in flight per SM (L2 prefetch + ring): loaded HBM latency
    // x per-SM bandwidth with margin (~5 us x 44 GB/s)
    static const long long pf_kb = [] {
      const char* e = getenv("BO_PF_KB");
      return e ? atoll(e) : 0LL;  // off: L2 prefetch measured slower than the ring alone
    }();
    const int ncols = r.K + ((ki.qtx || ki.upd) ? r.p : 0) + (ki.sk == SK_GAUSS ? mh : 0);
    const long long tile_bytes = (long long)T * (8LL * ncols + (ki.sk == SK_COUNT ? 4 : 0));
    const long long want = (pf_kb * 1024 + tile_bytes - 1) / tile_bytes - NS;
    a.prefetch_tiles = (int)std::max(0LL, std::min(64LL, want));
  }
  a.region0_dbl = (int)(region0 / 8);
  a.dm_len = dm_len;
  a.ntiles = (int)((ctx->n_local + T - 1) / T);
  const int grid = std::max(1, std::min(ctx->num_sms, a.ntiles));
  // workspace
  const size_t need_part = (size_t)grid * a.part_len;
  if (need_part > ctx->partials_cap) {
    if (ctx->partials) cudaFree(ctx->partials);
    ctx->partials_cap = need_part * 2;
    CU(cudaMalloc(&ctx->partials, ctx->partials_cap * 8));
  }
  if ((size_t)a.part_len > ctx->sums_cap) {
    if (ctx->sums) cudaFree(ctx->sums);
    ctx->sums_cap = (size_t)a.part_len * 2 + 1024;
    CU(cudaMalloc(&ctx->sums, ctx->sums_cap * 8));
  }
  a.partials = ctx->partials;
  a.sums = ctx->sums;
  a.counter = ctx->counter;
  // finalize descriptor
  FinArgs& f = r.fin;
  f.K = r.K;
  f.p = r.p;
  if (f.p_total == 0) f.p_total = r.p;
  f.mh = (ki.sk == SK_COUNT && r.sk && r.sk->theta_g) ? (int)r.sk->mhat : mh;
  f.mc = (ki.sk == SK_COUNT && r.sk) ? (int)r.sk->mc : 0;
  f.theta_g = (ki.sk == SK_COUNT && r.sk) ? r.sk->theta_g : nullptr;
  f.pass_id = r.pass_id;
  if (f.pivot_tol == 0.0) f.pivot_tol = 2.220446049250313e-16;
  f.sums = ctx->sums;
  f.off_q = a.off_q;
  f.ld_q = a.ld_q;
  f.off_g = a.off_g;
  f.off_s = a.off_s;
  f.ld_s = a.ld_s;
  f.status = ctx->status;
  if (f.ldcq == 0) f.ldcq = LDC;
  if (f.ldc == 0) f.ldc = LDC;
  a.fin = f;
  static const bool unfuse = getenv("BO_UNFUSE_FIN") != nullptr;  // diagnostics: finalize as its own kernel
  a.fused_finalize = (!ctx->collective && !unfuse) ? 1 : 0;

  PassFn fn = get_pass_fn(nt, T, r.kind, r.exact, r.K);
  static std::mutex mu;
  // the opt-in is a per-device function attribute: key the cache on (device, fn)
  static std::map<std::pair<int, const void*>, size_t> attr_set;
  {
    std::lock_guard<std::mutex> g(mu);
    const auto key = std::make_pair(ctx->device, (const void*)fn);
    auto it = attr_set.find(key);
    if (it == attr_set.end() || it->second < total) {
      CU(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)total));
      attr_set[key] = total;
    }
  }
  cudaEvent_t pe0 = nullptr, pe1 = nullptr;
  if (ctx->profiling) {
    while (ctx->ev_pool.size() < ctx->ev_used + 2) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      ctx->ev_pool.push_back(e);
    }
    pe0 = ctx->ev_pool[ctx->ev_used++];
    pe1 = ctx->ev_pool[ctx->ev_used++];
    CU(cudaEventRecord(pe0, ctx->stream));
  }
  CUtensorMap tmV, tmQ, tmT;
  {
    const int S = tile_stride(T);
    TRY(make_tmap(&tmV, r.V, ctx->n_local, r.K, r.ldv, S, st));
    TRY(make_tmap(&tmQ, (ki.qtx || ki.upd) ? r.Q : nullptr, ctx->n_local, r.p, r.ldq, S, st));
    TRY(make_tmap(&tmT, ki.sk == SK_GAUSS ? r.sk->theta : nullptr, ctx->n_local, mh,
                  ki.sk == SK_GAUSS ? r.sk->ldth : 0, S, st));
  }
  fn<<<grid, pass_threads(ki.upd, pre_qtx, pre_upd), total, ctx->stream>>>(a, tmV, tmQ, tmT);
  CU(cudaGetLastError());
  ctx->launches++;
  if (ctx->profiling) {
    CU(cudaEventRecord(pe1, ctx->stream));
    const int ncols = r.K + ((ki.qtx || ki.upd) ? r.p : 0) + (ki.sk == SK_GAUSS ? mh : 0);
    const uint64_t rows = ctx->n_local;
    const uint64_t bytes = rows * (8ull * ncols + (ki.sk == SK_COUNT ? 4ull : 0ull) + (ki.store ? 8ull * r.K : 0ull));
    ctx->prof.push_back({r.kind, r.K, r.p, mh, rows, bytes, pe0, pe1});
  }
  if (!a.fused_finalize) {
    // one all-reduce per pass that reduces (a ledger event); store-only passes have none
    if (ctx->collective && (ki.qtx || ki.gram || ki.sk != SK_NONE))
      TRY(comm_allreduce(ctx, ctx->sums, (size_t)a.part_len, st));
    if (f.ops) {
      const size_t fsm = (1536 + (size_t)std::max(f.mh, 32) * 16 + 64) * 8;
      if (fsm > 48 * 1024)
        CU(cudaFuncSetAttribute((const void*)finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));
      finalize_kernel<<<1, 256, fsm, ctx->stream>>>(f);
      CU(cudaGetLastError());
      ctx->launches++;
    }
  }
  return BO_OK;
}



// Projection ranges wider than one pass (64 columns) are split into column
// chunks: Q^T X chunk by chunk into the rows of Cq; X = V - Q C as a chain of
// partial updates through the output buffer, the last chunk carrying the
// pass's own reductions and finalize.
int run_pass(bo_ctx ctx, PassReq& r, bo_status* st) {
  const KindInfo& ki = kKindInfo[r.kind];
  if (!(ki.qtx || ki.upd) || r.p <= kMaxPTile) return run_pass_single(ctx, r, st);
  const int P = r.p;
  for (int c0 = 0; c0 < P; c0 += kMaxPTile) {
    const bool last = c0 + kMaxPTile >= P;
    PassReq q = r;
    q.Q = r.Q + (size_t)c0 * r.ldq;
    q.p = std::min(kMaxPTile, P - c0);
    q.fin.p_total = P;
    if (ki.qtx) {
      q.fin.q_row_off = c0;
      if (!last) {
        q.kind = ki.npre == 2 ? PK_P2_QTX : ki.npre == 1 ? PK_P1_QTX : PK_QTX;
        q.fin.ops = FIN_COPY_Q;
      }
    } else {
      q.Cm = r.Cm + c0;
      if (c0 > 0) {  // continue from the partial update stored by the previous chunk
        q.V = r.out;
        q.ldv = r.ldo;
        q.Rpre0 = q.Rpre1 = nullptr;
      }
      if (!last) {
        q.kind = (c0 == 0 && ki.npre == 2) ? PK_P2_UPD_ST : (c0 == 0 && ki.npre == 1) ? PK_P1_UPD_ST : PK_UPD_ST;
        q.fin.ops = 0;
        q.sk = nullptr;
      } else if (c0 > 0 && ki.npre > 0) {
        q.kind = PK_UPD_GRAM_ST;  // the pre-solve update kinds (P1/P2_UPD_GRAM_ST) minus their solve
      }
      if (!r.out) return set_st(st, BO_INVALID, 0, 0.0, "chunked update needs an output buffer");
    }
    TRY(run_pass_single(ctx, q, st));
  }
  return BO_OK;
}

// zero the device status word
// ---------------------------------------------------------------------------
// collective transport
// ---------------------------------------------------------------------------
int comm_allreduce(bo_ctx ctx, double* buf, size_t n, bo_status* st) {
  ctx->allreduces++;
  if (ctx->has_comm) {
    const int rc = ctx->comm.allreduce_sum_f64(ctx->comm.user, buf, n, ctx->stream);
    return rc ? set_st(st, BO_NCCL, rc, 0.0, "all-reduce callback failed (%d)", rc) : BO_OK;
  }
  NcclApi& nc = nccl();
  const int rc = nc.AllReduce(buf, buf, n, kNcclFloat64, kNcclSum, ctx->nccl, ctx->stream);
  return rc ? set_st(st, BO_NCCL, rc, 0.0, "ncclAllReduce failed: %s", nc.GetErrorString ? nc.GetErrorString(rc) : "?")
            : BO_OK;
}
int comm_allgather_u64(bo_ctx ctx, const uint64_t* send, size_t n, uint64_t* recv, bo_status* st) {
  if (ctx->has_comm) {
    const int rc = ctx->comm.allgather_u64(ctx->comm.user, send, n, recv, ctx->stream);
    return rc ? set_st(st, BO_NCCL, rc, 0.0, "all-gather callback failed (%d)", rc) : BO_OK;
  }
  NcclApi& nc = nccl();
  if (!nc.AllGather) return set_st(st, BO_NCCL, 0, 0.0, "ncclAllGather missing");
  const int rc = nc.AllGather(send, recv, n, kNcclUint64, ctx->nccl, ctx->stream);
  return rc ? set_st(st, BO_NCCL, rc, 0.0, "ncclAllGather failed (%d)", rc) : BO_OK;
}
int comm_exchange(bo_ctx ctx, int nops, const bo_p2p_op* ops, bo_status* st, cudaStream_t s) {
  if (nops == 0) return BO_OK;
  if (!s) s = ctx->stream;
  if (ctx->has_comm) {
    const int rc = ctx->comm.exchange_f64(ctx->comm.user, nops, ops, s);
    return rc ? set_st(st, BO_NCCL, rc, 0.0, "exchange callback failed (%d)", rc) : BO_OK;
  }
  NcclApi& nc = nccl();
  if (!nc.Send || !nc.Recv || !nc.GroupStart || !nc.GroupEnd) return set_st(st, BO_NCCL, 0, 0.0, "NCCL p2p missing");
  nc.GroupStart();
  for (int i = 0; i < nops; ++i) {
    if (ops[i].is_send)
      nc.Send(ops[i].buf, ops[i].count, kNcclFloat64, ops[i].peer, ctx->nccl, s);
    else
      nc.Recv(ops[i].buf, ops[i].count, kNcclFloat64, ops[i].peer, ctx->nccl, s);
  }
  const int rc = nc.GroupEnd();
  return rc ? set_st(st, BO_NCCL, rc, 0.0, "NCCL group send/recv failed (%d)", rc) : BO_OK;
}

int reset_status(bo_ctx ctx, bo_status* st) {
  CU(cudaMemsetAsync(ctx->status, 0, sizeof(DevStatus), ctx->stream));
  return BO_OK;
}
// fetch status + tiny workspace to host
int fetch(bo_ctx ctx, bool tiny, bo_status* st) {
  if (tiny)  // the status word leads the workspace: one copy
    CU(cudaMemcpyAsync(ctx->tiny_host, ctx->tiny, TINY_LEN * 8, cudaMemcpyDeviceToHost, ctx->stream));
  else
    CU(cudaMemcpyAsync(ctx->status_host, ctx->status, sizeof(DevStatus), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (tiny) std::memcpy(ctx->status_host, ctx->tiny_host + OFF_STATUS, sizeof(DevStatus));
  return BO_OK;
}

// Stage a tall input into 16-byte-aligned, ld%4==0 storage when the caller's is not.
int stage_input(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, int slot, const double** out,
                uint64_t* ldout, bo_status* st) {
  const uint64_t nl = ctx->n_local;
  if (((uintptr_t)v % 16) == 0 && ldv % 4 == 0 && ldv >= round_up(nl, 4)) {
    *out = v;
    *ldout = ldv;
    return BO_OK;
  }
  if (k > 16) return set_st(st, BO_INVALID, 0, 0.0, "panel too wide");
  CU(cudaMemcpy2DAsync(ctx->scratch[slot], ctx->ld * 8, v, ldv * 8, nl * 8, k, cudaMemcpyDeviceToDevice,
                       ctx->stream));
  *out = ctx->scratch[slot];
  *ldout = ctx->ld;
  return BO_OK;
}

// an output buffer the bulk store engine can write (else write scratch + copy)
bool out_ok(bo_ctx ctx, const double* q, uint64_t ldq) {
  return ((uintptr_t)q % 16) == 0 && ldq % 4 == 0 && ldq >= round_up(ctx->n_local, 4);
}

std::string chol_msg(const char* ctx_name, long long step) {
  char b[160];
  snprintf(b, sizeof b, "%s: nonpositive Cholesky pivot at step %lld", ctx_name, step);
  return b;
}
int dev_error(bo_ctx ctx, const char* chol_ctx, bo_status* st) {
  const DevStatus& d = *ctx->status_host;
  if (d.code == ST_CHOLESKY)
    return set_st(st, BO_CHOLESKY_BREAKDOWN, d.step, d.pivot, "%s", chol_msg(chol_ctx, d.step).c_str());
  if (d.code == ST_SINGULAR)
    return set_st(st, BO_SINGULAR_TRIANGULAR, d.step, 0.0,
                  "triangular factor is singular: zero diagonal at index %lld", d.step);
  return BO_OK;
}

}  // namespace host
}  // namespace bo

// ===========================================================================
// context
// ===========================================================================
extern "C" int bo_abi_version(void) { return BO_ABI_VERSION; }
extern "C" int bo_nccl_id_bytes(void) { return 128; }
extern "C" int bo_nccl_get_unique_id(void* out, bo_status* st) {
  NcclApi& nc = nccl();
  if (!nc.ok) return set_st(st, BO_NCCL, 0, 0.0, "NCCL library not available");
  int rc = nc.GetUniqueId(out);
  if (rc) return set_st(st, BO_NCCL, 0, 0.0, "ncclGetUniqueId failed (%d)", rc);
  ok_st(st);
  return BO_OK;
}

static int ctx_create_impl(int device, int rank, int world, const void* nccl_id, const bo_comm_ops* comm,
                           uint64_t n_global, uint64_t row_begin, uint64_t row_end, void* stream, bo_ctx* out,
                           bo_status* st);
extern "C" int bo_ctx_create(int device, int rank, int world, const void* nccl_id, uint64_t n_global,
                             uint64_t row_begin, uint64_t row_end, void* stream, bo_ctx* out,
                             bo_status* st) {
  return ctx_create_impl(device, rank, world, nccl_id, nullptr, n_global, row_begin, row_end, stream, out, st);
}
extern "C" int bo_ctx_create_comm(int device, int rank, int world, const bo_comm_ops* comm, uint64_t n_global,
                                  uint64_t row_begin, uint64_t row_end, void* stream, bo_ctx* out, bo_status* st) {
  ok_st(st);
  if (!comm || !comm->allreduce_sum_f64 || !comm->allgather_u64 || !comm->exchange_f64)
    return set_st(st, BO_INVALID, 0, 0.0, "bo_comm_ops needs allreduce_sum_f64, allgather_u64 and exchange_f64");
  return ctx_create_impl(device, rank, world, nullptr, comm, n_global, row_begin, row_end, stream, out, st);
}
static int ctx_create_impl(int device, int rank, int world, const void* nccl_id, const bo_comm_ops* comm,
                           uint64_t n_global, uint64_t row_begin, uint64_t row_end, void* stream, bo_ctx* out,
                           bo_status* st) {
  ok_st(st);
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_st(st, BO_CUDA, 0, 0.0, "no CUDA device available (the block-orthogonalization path has no CPU fallback)");
  if (device < 0 || device >= ndev) return set_st(st, BO_INVALID, 0, 0.0, "bad device %d", device);
  if (world < 1 || rank < 0 || rank >= world) return set_st(st, BO_INVALID, 0, 0.0, "bad rank/world");
  if (row_end < row_begin || row_end > n_global) return set_st(st, BO_INVALID, 0, 0.0, "bad row range");
  CU(cudaSetDevice(device));
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, device));
  // built for sm_100a only: arch-specific features do not carry to sm_103 / sm_11x / sm_12x
  if (prop.major != 10 || prop.minor != 0)
    return set_st(st, BO_CUDA, 0, 0.0, "device %s (sm_%d%d) is not sm_100 (library built for sm_100a only)",
                  prop.name, prop.major, prop.minor);
  bo_ctx c = new bo_ctx_s();
  c->device = device;
  c->rank = rank;
  c->world = world;
  c->n_global = n_global;
  c->row_begin = row_begin;
  c->row_end = row_end;
  c->n_local = row_end - row_begin;
  c->ld = round_up(std::max<uint64_t>(c->n_local, 1), 32);
  if (const char* e = getenv("BO_LD_PAD")) c->ld += round_up((uint64_t)atoll(e), 4);  // layout experiments
  c->num_sms = prop.multiProcessorCount;
  c->smem_optin = prop.sharedMemPerBlockOptin;
  if (stream) {
    c->stream = (cudaStream_t)stream;
  } else {
    CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  {
    cudaMemPoolProps pp{};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = device;
    CU(cudaMemPoolCreate(&c->pool, &pp));
    uint64_t keep = ~0ULL;
    CU(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  CU(cudaMalloc(&c->counter, bo::kMaxRedCounters * sizeof(unsigned)));
  CU(cudaMemset(c->counter, 0, bo::kMaxRedCounters * sizeof(unsigned)));

  CU(cudaMallocHost(&c->status_host, sizeof(DevStatus)));
  c->tiny_cap = TINY_LEN;
  CU(cudaMalloc(&c->tiny, TINY_LEN * 8));
  CU(cudaMemset(c->tiny, 0, TINY_LEN * 8));
  c->status = reinterpret_cast<DevStatus*>(c->tiny + OFF_STATUS);  // leads the workspace (one-copy snapshots)
  CU(cudaMallocHost(&c->tiny_host, TINY_LEN * 8));
  for (int i = 0; i < 3; ++i) {
    CU(cudaMalloc(&c->scratch[i], c->ld * 16 * 8));
    CU(cudaMemset(c->scratch[i], 0, c->ld * 16 * 8));
  }
  // the initial memsets ran on the legacy stream, which the non-blocking
  // ctx stream does not wait for
  CU(cudaDeviceSynchronize());
  if (comm) {
    c->has_comm = true;
    c->comm = *comm;
    c->collective = world > 1;
  } else if (world > 1 || nccl_id) {  // an id with world = 1: a size-1 communicator
    NcclApi& nc = nccl();
    if (!nc.ok) {
      bo_ctx_destroy(c);
      return set_st(st, BO_NCCL, 0, 0.0, "NCCL library not available");
    }
    NcclUniqueId id;
    std::memcpy(id.internal, nccl_id, sizeof id.internal);
    int rc = nc.CommInitRank(&c->nccl, world, id, rank);
    if (rc) {
      bo_ctx_destroy(c);
      return set_st(st, BO_NCCL, 0, 0.0, "ncclCommInitRank failed (%d)", rc);
    }
    c->collective = true;
  }
  *out = c;
  return BO_OK;
}

extern "C" int bo_ctx_destroy(bo_ctx c) {
  if (!c) return BO_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  if (c->nccl && nccl().ok) nccl().CommDestroy(c->nccl);
  cudaFree(c->partials);
  cudaFree(c->phase_prof);
  cudaFree(c->sums);
  cudaFree(c->counter);
  cudaFreeHost(c->status_host);
  cudaFree(c->tiny);
  cudaFreeHost(c->tiny_host);
  for (int i = 0; i < 3; ++i) cudaFree(c->scratch[i]);
  cudaFree(c->spare_buf);
  cudaFree(c->spare_q);
  if (c->spare_snap) cudaFreeHost(c->spare_snap);
  cudaFree(c->gen_plan.dev);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_x) cudaEventDestroy(c->ev_x);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  if (c->pool) cudaMemPoolDestroy(c->pool);
  delete c;
  return BO_OK;
}
extern "C" int bo_ctx_synchronize(bo_ctx c, bo_status* st) {
  ok_st(st);
  CU(cudaStreamSynchronize(c->stream));
  return BO_OK;
}
extern "C" uint64_t bo_ctx_local_rows(bo_ctx c) { return c->n_local; }
extern "C" uint64_t bo_ctx_ld(bo_ctx c) { return c->ld; }
extern "C" uint64_t bo_ctx_kernel_launches(bo_ctx c) { return c->launches; }
extern "C" uint64_t bo_ctx_allreduces(bo_ctx c) { return c->allreduces; }
extern "C" int bo_ctx_profile(bo_ctx c, int enable) {
  c->profiling = enable;
  if (enable) {
    c->prof.clear();
    c->ev_used = 0;
  }
  return BO_OK;
}
extern "C" int bo_ctx_profile_read(bo_ctx c, bo_prof_record* out, int max, int* count, bo_status* st) {
  ok_st(st);
  CU(cudaStreamSynchronize(c->stream));
  int m = 0;
  for (auto& r : c->prof) {
    if (m >= max) break;
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, r.e0, r.e1));
    out[m++] = {r.kind, r.K, r.p, r.mh, r.rows, r.bytes, ms};
  }
  if (count) *count = (int)c->prof.size();
  return BO_OK;
}
extern "C" const char* bo_pass_kind_name(int kind) {
  static const char* names[] = {
#define X(nm, a, b, c, d, e, f, g) #nm,
      BO_PASS_KINDS(X)
#undef X
  };
  return (kind >= 0 && kind < PK_COUNT) ? names[kind] : "?";
}

// ===========================================================================
// sketch
// ===========================================================================
namespace bo {
namespace host {
uint64_t derive_seed(uint64_t base, uint64_t stream) {  // rng.hpp:12-17
  uint64_t z = base + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// host Box-Muller stream (rng.hpp:37-49) for the tiny replicated count_gauss stage
struct HostRng {
  std::mt19937_64 gen;
  bool have = false;
  double spare = 0.0;
  explicit HostRng(uint64_t s) : gen(s) {}
  double normal() {
    if (have) {
      have = false;
      return spare;
    }
    const double u1 = (static_cast<double>(gen() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = static_cast<double>(gen() >> 11) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(a);
    have = true;
    return r * std::cos(a);
  }
};

// The count_gauss dense stage is drawn on the host with the reference's
// generator (bit-identical, ~15 ms for 7442 x 122).  The GMRES driver knows
// the next restart's seed, so it asks for that stage to be drawn on a host
// thread while the current restart runs on the GPU.
static std::vector<double> gen_theta_g(uint64_t seed, uint64_t mc, uint64_t mhat) {
  // (splitting the draw over host threads from jumped MT windows measured
  // 11-13 ms against 15 ms on 8 cores, plus ~25 ms of jump polynomials per
  // process: not worth it once the next restart's stage is prefetched)
  HostRng rg(derive_seed(seed, 1));
  const double scale = 1.0 / std::sqrt(double(mhat));
  std::vector<double> t(mc * mhat);
  for (uint64_t L = 0; L < mc * mhat; ++L) t[L] = scale * rg.normal();
  return t;
}
struct ThetaGJob {
  uint64_t seed, mc, mhat;
  std::future<std::vector<double>> fut;
};
static std::mutex g_tg_mu;
static std::vector<ThetaGJob> g_tg_jobs;

void prefetch_theta_g(uint64_t seed, uint64_t mc, uint64_t mhat) {
  std::lock_guard<std::mutex> g(g_tg_mu);
  for (auto& j : g_tg_jobs)
    if (j.seed == seed && j.mc == mc && j.mhat == mhat) return;
  if (g_tg_jobs.size() >= 2) g_tg_jobs.erase(g_tg_jobs.begin());  // (waits for a stale job to finish)
  g_tg_jobs.push_back({seed, mc, mhat, std::async(std::launch::async, gen_theta_g, seed, mc, mhat)});
}

std::vector<double> take_theta_g(uint64_t seed, uint64_t mc, uint64_t mhat) {
  std::future<std::vector<double>> f;
  {
    std::lock_guard<std::mutex> g(g_tg_mu);
    for (size_t k = 0; k < g_tg_jobs.size(); ++k)
      if (g_tg_jobs[k].seed == seed && g_tg_jobs[k].mc == mc && g_tg_jobs[k].mhat == mhat) {
        f = std::move(g_tg_jobs[k].fut);
        g_tg_jobs.erase(g_tg_jobs.begin() + k);
        break;
      }
  }
  return f.valid() ? f.get() : gen_theta_g(seed, mc, mhat);
}

struct Chunk {
  uint64_t J, len;
};

// generate draws [d0, d1) (both even) of the stream seeded with mt_seed
int gen_stream(bo_ctx ctx, uint64_t mt_seed, const std::vector<std::pair<uint64_t, uint64_t>>& segs,
               GenArgs ga, bo_status* st) {
  // chunking: about one chunk per SM over all segments, each a multiple of
  // 312 draws (mt_stream_kernel: one CTA per chunk)
  uint64_t total = 0;
  for (auto& s : segs) total += s.second - s.first;
  if (total == 0) return BO_OK;
  const uint64_t target = std::max<uint64_t>(312 * 16, round_up(total / (uint64_t)ctx->num_sms + 1, 312));
  auto& plan = ctx->gen_plan;
  if (plan.key_total != total || plan.key_segs != segs || !plan.dev) {
    // seed-independent part, cached per plan: chunk table + the set-bit
    // indices of every chunk's jump polynomial x^J mod phi
    std::vector<Chunk> chunks;
    for (auto& s : segs)
      for (uint64_t d = s.first; d < s.second; d += target) chunks.push_back({d, std::min(target, s.second - d)});
    const size_t nc = chunks.size();
    const int pw = bo::mt64::poly_words();
    std::vector<uint64_t> poly(pw), tab(2 * nc + nc + 1);
    // cache x^target first: every later chunk of a segment then costs one
    // multiplication mod phi (chained from its predecessor) instead of a full
    // square-and-multiply (~300 ms -> a few ms for a 148-chunk plan)
    bo::mt64::jump_poly(target, poly.data());
    std::vector<uint16_t> idx;
    idx.reserve(nc * 10240);
    for (size_t c = 0; c < nc; ++c) {
      bo::mt64::jump_poly(chunks[c].J, poly.data());
      tab[c] = chunks[c].J;
      tab[nc + c] = chunks[c].len;
      tab[2 * nc + c] = idx.size();
      for (int w = 0; w < pw; ++w)
        for (uint64_t b = poly[w]; b; b &= b - 1) idx.push_back((uint16_t)(w * 64 + __builtin_ctzll(b)));
    }
    tab[3 * nc] = idx.size();
    if (plan.dev) cudaFree(plan.dev);
    plan.dev = nullptr;
    const size_t words = tab.size() + (idx.size() + 3) / 4 + bo::mt64::prefix_words() + 2;
    CU(cudaMalloc((void**)&plan.dev, words * 8));
    CU(cudaMemcpyAsync(plan.dev, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(plan.dev + tab.size(), idx.data(), idx.size() * 2, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    plan.key_total = total;
    plan.key_segs = segs;
    plan.nchunks = nc;
    plan.pre_off = tab.size() + (idx.size() + 3) / 4;
    plan.pre_off += plan.pre_off & 1;  // 16-byte alignment for the vector prefix load
  }
  const size_t nc = plan.nchunks;
  uint64_t* dpre = plan.dev + plan.pre_off;
  // the seed-dependent stream prefix (20248 words of mt19937_64, ~0.1 ms host)
  plan.prefix.resize(bo::mt64::prefix_words());
  bo::mt64::prefix(mt_seed, plan.prefix.data());
  CU(cudaMemcpyAsync(dpre, plan.prefix.data(), plan.prefix.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  ga.prefix = dpre;
  ga.polys = nullptr;
  ga.chunk_J = plan.dev;
  ga.chunk_len = plan.dev + nc;
  ga.jidx_off = plan.dev + 2 * nc;
  ga.jidx = reinterpret_cast<const uint16_t*>(plan.dev + 3 * nc + 1);
  const size_t smem = (size_t)(kPrefixWords + 8 + kRing * kMtN + 2 * kRing) * 8;
  static std::mutex attr_mu;
  static std::set<int> attr_dev;  // per-device opt-in
  {
    std::lock_guard<std::mutex> g(attr_mu);
    if (!attr_dev.count(ctx->device)) {
      CU(cudaFuncSetAttribute((const void*)mt_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_dev.insert(ctx->device);
    }
  }
  mt_stream_kernel<<<(unsigned)nc, 1024, smem, ctx->stream>>>(ga);
  CU(cudaGetLastError());
  ctx->launches++;
  // the pageable prefix copy is staged by the driver; one sync keeps the
  // host vector valid (it is reused by the next build)
  CU(cudaStreamSynchronize(ctx->stream));
  return BO_OK;
}
}  // namespace host
}  // namespace bo

extern "C" int bo_sketch_build(bo_ctx ctx, int kind, uint64_t n, uint64_t shat, uint64_t seed, bo_sketch* out,
                               bo_status* st) {
  ok_st(st);
  *out = nullptr;
  if (n != ctx->n_global) return set_st(st, BO_INVALID, 0, 0.0, "sketch ambient dimension != ctx global rows");
  const uint64_t cols = shat + 1;
  bo_sketch s = new bo_sketch_s();
  s->ctx = ctx;
  s->kind = kind;
  s->n = n;
  uint64_t check = 0;
  switch (kind) {
    case BO_SKETCH_GAUSSIAN:
      s->mhat = 2 * cols;
      check = s->mhat;
      break;
    case BO_SKETCH_COUNT:
      s->mhat = 2 * cols * cols;
      s->mc = s->mhat;
      check = s->mhat;
      break;
    case BO_SKETCH_COUNT_GAUSS:
      s->mhat = 2 * cols;
      s->mc = 2 * cols * cols;
      check = s->mc;
      break;
    default:
      delete s;
      return set_st(st, BO_INVALID, 0, 0.0, "unknown sketch kind");
  }
  if (n <= check) {  // errors.hpp:45-49
    delete s;
    return set_st(st, BO_AMBIENT_TOO_SMALL, 0, 0.0, "ambient dimension n=%llu must exceed sketch size mhat=%llu",
                  (unsigned long long)n, (unsigned long long)check);
  }
  if (!bo::mt64::ready()) {
    delete s;
    return set_st(st, BO_INVALID, 0, 0.0, "MT19937-64 jump-ahead initialisation failed");
  }
  const uint64_t mt_seed = derive_seed(seed, 0);  // sketch.cpp:72
  GenArgs ga{};
  ga.n_global = n;
  ga.row_begin = ctx->row_begin;
  ga.row_end = ctx->row_end;
  const uint64_t nl = ctx->n_local;
  std::vector<std::pair<uint64_t, uint64_t>> segs;
  if (kind == BO_SKETCH_GAUSSIAN) {
    s->ldth = ctx->ld;
    const size_t bytes = std::max<uint64_t>(s->ldth * s->mhat, 1) * 8;
    if (ctx->spare_buf && ctx->spare_bytes >= bytes) {  // recycled from the previous cycle's sketch
      s->theta = (double*)ctx->spare_buf;
      s->theta_bytes = ctx->spare_bytes;
      ctx->spare_buf = nullptr;
      ctx->spare_bytes = 0;
    } else {
      cudaError_t e = cudaMalloc(&s->theta, bytes);
      if (e != cudaSuccess) {
        delete s;
        return set_st(st, BO_CUDA, 0, 0.0, "cudaMalloc(theta) failed: %s", cudaGetErrorString(e));
      }
      s->theta_bytes = bytes;
    }
    // every local row is generated; only the padding rows [n_local, ld) need zeros
    if (s->ldth > nl)
      cudaMemset2DAsync(s->theta + nl, s->ldth * 8, 0, (s->ldth - nl) * 8, s->mhat, ctx->stream);
    ga.kind = 0;
    ga.mhat = (int)s->mhat;
    ga.scale = 1.0 / std::sqrt(double(s->mhat));
    ga.theta = s->theta;
    ga.ldth = s->ldth;
    // column j needs normals [j n + a, j n + b) ; pairs start at even draws
    if (ctx->row_begin == 0 && ctx->row_end == n) {
      segs.push_back({0, round_up(n * s->mhat, 2)});
    } else {
      for (uint64_t j = 0; j < s->mhat; ++j) {
        const uint64_t lo = (j * n + ctx->row_begin) & ~1ULL;
        const uint64_t hi = round_up(j * n + ctx->row_end, 2);
        if (hi > lo) segs.push_back({lo, hi});
      }
    }
  } else {
    cudaError_t e = cudaMalloc(&s->code, round_up(std::max<uint64_t>(nl, 1), 32) * 4);
    if (e != cudaSuccess) {
      delete s;
      return set_st(st, BO_CUDA, 0, 0.0, "cudaMalloc(code) failed: %s", cudaGetErrorString(e));
    }
    cudaMemsetAsync(s->code, 0, round_up(std::max<uint64_t>(nl, 1), 32) * 4, ctx->stream);
    ga.kind = 1;
    ga.width = s->mc;
    ga.code = s->code;
    segs.push_back({2 * ctx->row_begin, 2 * ctx->row_end});
  }
  int rc = gen_stream(ctx, mt_seed, segs, ga, st);
  if (rc != BO_OK) {
    bo_sketch_destroy(s);
    return rc;
  }
  if (kind == BO_SKETCH_COUNT_GAUSS) {
    // dense stage mc x mhat from derive_seed(seed, 1) (sketch.cpp:91-95), replicated
    s->theta_g_host = bo::host::take_theta_g(seed, s->mc, s->mhat);
    cudaError_t e = cudaMalloc(&s->theta_g, s->theta_g_host.size() * 8);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(s->theta_g, s->theta_g_host.data(), s->theta_g_host.size() * 8, cudaMemcpyHostToDevice,
                          ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
      bo_sketch_destroy(s);
      return set_st(st, BO_CUDA, 0, 0.0, "count_gauss stage upload failed: %s", cudaGetErrorString(e));
    }
  }
  *out = s;
  return BO_OK;
}

extern "C" int bo_sketch_from_dense(bo_ctx ctx, const double* theta, uint64_t ld, uint64_t mhat, bo_sketch* out,
                                    bo_status* st) {
  ok_st(st);
  bo_sketch s = new bo_sketch_s();
  s->ctx = ctx;
  s->kind = BO_SKETCH_GAUSSIAN;
  s->n = ctx->n_global;
  s->mhat = mhat;
  s->ldth = ctx->ld;
  s->theta_bytes = std::max<uint64_t>(s->ldth * mhat, 1) * 8;
  CU(cudaMalloc(&s->theta, s->theta_bytes));
  CU(cudaMemsetAsync(s->theta, 0, s->ldth * mhat * 8, ctx->stream));
  CU(cudaMemcpy2DAsync(s->theta, s->ldth * 8, theta, ld * 8, ctx->n_local * 8, mhat, cudaMemcpyDeviceToDevice,
                       ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  *out = s;
  return BO_OK;
}

extern "C" int bo_sketch_destroy(bo_sketch s) {
  if (!s) return BO_OK;
  bo_ctx ctx = s->ctx;
  cudaStreamSynchronize(ctx->stream);
  if (s->own_theta && s->theta) {
    if (!ctx->spare_buf) {  // keep one buffer for the next build
      ctx->spare_buf = s->theta;
      ctx->spare_bytes = s->theta_bytes;
    } else if (ctx->spare_bytes < s->theta_bytes) {
      cudaFree(ctx->spare_buf);
      ctx->spare_buf = s->theta;
      ctx->spare_bytes = s->theta_bytes;
    } else {
      cudaFree(s->theta);
    }
  }
  cudaFree(s->code);
  cudaFree(s->theta_g);
  cudaFree(s->perm);
  cudaFree(s->boff);
  cudaFree(s->cnt);
  delete s;
  return BO_OK;
}
extern "C" uint64_t bo_sketch_size(bo_sketch s) { return s->mhat; }
extern "C" uint64_t bo_sketch_count_width(bo_sketch s) { return s->mc; }
extern "C" int bo_sketch_kind(bo_sketch s) { return s->kind; }

extern "C" int bo_sketch_dense_to_host(bo_sketch s, double* out, bo_status* st) {
  ok_st(st);
  if (!s->theta) return set_st(st, BO_INVALID, 0, 0.0, "sketch has no dense row stage");
  const uint64_t nl = s->ctx->n_local;
  CU(cudaStreamSynchronize(s->ctx->stream));
  CU(cudaMemcpy2D(out, nl * 8, s->theta, s->ldth * 8, nl * 8, s->mhat, cudaMemcpyDeviceToHost));
  return BO_OK;
}
extern "C" int bo_sketch_count_to_host(bo_sketch s, uint32_t* buckets, double* signs, bo_status* st) {
  ok_st(st);
  if (!s->code) return set_st(st, BO_INVALID, 0, 0.0, "sketch has no count stage");
  const uint64_t nl = s->ctx->n_local;
  std::vector<uint32_t> c(nl);
  CU(cudaMemcpyAsync(c.data(), s->code, nl * 4, cudaMemcpyDeviceToHost, s->ctx->stream));
  CU(cudaStreamSynchronize(s->ctx->stream));
  for (uint64_t i = 0; i < nl; ++i) {
    if (buckets) buckets[i] = c[i] & 0x7fffffffu;
    if (signs) signs[i] = (c[i] & 0x80000000u) ? -1.0 : 1.0;
  }
  return BO_OK;
}
extern "C" int bo_sketch_gauss_stage_to_host(bo_sketch s, double* out, bo_status* st) {
  ok_st(st);
  if (s->theta_g_host.empty()) return set_st(st, BO_INVALID, 0, 0.0, "sketch has no count_gauss stage");
  std::memcpy(out, s->theta_g_host.data(), s->theta_g_host.size() * 8);
  return BO_OK;
}

namespace bo {
namespace host {
int sketch_pass(bo_sketch sk, const double* v, uint64_t ldv, int K, int pass_id, int extra_ops, bo_status* st) {
  bo_ctx ctx = sk->ctx;
  PassReq r{};
  r.kind = sk->kind == BO_SKETCH_GAUSSIAN ? PK_SKG : PK_SKC;
  r.K = K;
  r.V = v;
  r.ldv = ldv;
  r.sk = sk;
  r.pass_id = pass_id;
  r.fin.ops = FIN_COPY_S | extra_ops;
  r.fin.Sout = T_(ctx, OFF_S);
  r.fin.Rhh = T_(ctx, OFF_R1);
  return run_pass(ctx, r, st);
}
}  // namespace host
}  // namespace bo

extern "C" int bo_sketch_apply(bo_sketch sk, const double* v, uint64_t ldv, uint64_t k, double* out,
                               uint64_t ledger[4], bo_status* st) {
  ok_st(st);
  bo_ctx ctx = sk->ctx;
  CU(cudaSetDevice(ctx->device));
  const double* vv;
  uint64_t lv;
  TRY(stage_input(ctx, v, ldv, k, 0, &vv, &lv, st));
  std::vector<double> S;
  TRY(sketch_to_host(sk, vv, lv, (int)k, S, st));
  std::memcpy(out, S.data(), sk->mhat * k * 8);
  if (ledger) ledger[BO_LEDGER_SKETCH]++;
  return BO_OK;
}

// ===========================================================================
// dense / intra-orth
// ===========================================================================
namespace bo {
namespace host {
void copy_factor_host(const double* src16, int K, double* dst /* K x K */) {
  for (int j = 0; j < K; ++j)
    for (int i = 0; i < K; ++i) dst[i + j * K] = src16[i + j * 16];
}

// cholqr on device: G -> R (slot Rslot) -> store Q (when q != nullptr)
int dev_cholqr(bo_ctx ctx, const double* v, uint64_t ldv, int K, double* q, uint64_t ldq, int Rslot, int pass_id,
               bo_status* st) {
  PassReq g{};
  g.kind = PK_GRAM;
  g.K = K;
  g.V = v;
  g.ldv = ldv;
  g.pass_id = pass_id;
  g.fin.ops = FIN_CHOL;
  g.fin.Rchol = T_(ctx, Rslot);
  TRY(run_pass(ctx, g, st));
  if (q) {
    PassReq w{};
    w.kind = PK_P1_ST;
    w.K = K;
    w.V = v;
    w.ldv = ldv;
    w.out = q;
    w.ldo = ldq;
    w.Rpre0 = T_(ctx, Rslot);
    w.pass_id = pass_id + 1;
    TRY(run_pass(ctx, w, st));
  }
  return BO_OK;
}

// intra-block factorization of V (n x K) per IntraKind, writing Q to q:
// cholqr2: gram->R1, trsm(R1)+gram->R2 (Rin = R2 R1), trsm(R1,R2)->store
// rand   : sketch->Rs(R1), trsm(R1)+gram->Rc(R2) (Rin = Rc Rs), trsm(R1,R2)->store
// pass ids 1, 2 (+3 store); Rin in OFF_RIN
int dev_intra(bo_ctx ctx, const double* v, uint64_t ldv, int K, int intra, bo_sketch sk, double* q, uint64_t ldq,
              bo_status* st) {
  if (intra == BO_INTRA_CHOLQR2) {
    PassReq g{};
    g.kind = PK_GRAM;
    g.K = K;
    g.V = v;
    g.ldv = ldv;
    g.pass_id = 1;
    g.fin.ops = FIN_CHOL;
    g.fin.Rchol = T_(ctx, OFF_R1);
    TRY(run_pass(ctx, g, st));
  } else {
    TRY(sketch_pass(sk, v, ldv, K, 1, FIN_HH, st));
  }
  PassReq g2{};
  g2.kind = PK_P1_GRAM;
  g2.K = K;
  g2.V = v;
  g2.ldv = ldv;
  g2.Rpre0 = T_(ctx, OFF_R1);
  g2.pass_id = 2;
  g2.fin.ops = FIN_CHOL | FIN_MULT;
  g2.fin.Rchol = T_(ctx, OFF_R2);
  g2.fin.Rin = T_(ctx, OFF_R1);
  g2.fin.rjj = T_(ctx, OFF_RIN);
  TRY(run_pass(ctx, g2, st));
  if (q) {
    // Two solves here, not one with Rin = R2 R1 (as bcgs2's P4 / P5 do): this
    // Q is final, and the second solve is what re-orthogonalises it (measured:
    // the product factor gave ||I - Q^T Q|| 1.3e-11 against the reference's
    // 1.7e-13 for CholQR2 at cond 1e6)
    PassReq w{};
    w.kind = PK_P2_ST;
    w.K = K;
    w.V = v;
    w.ldv = ldv;
    w.out = q;
    w.ldo = ldq;
    w.Rpre0 = T_(ctx, OFF_R1);
    w.Rpre1 = T_(ctx, OFF_R2);
    w.pass_id = 3;
    TRY(run_pass(ctx, w, st));
  }
  return BO_OK;
}

int write_out(bo_ctx ctx, double* q, uint64_t ldq, int K, double** target, uint64_t* ldt) {
  if (out_ok(ctx, q, ldq)) {
    *target = q;
    *ldt = ldq;
  } else {
    *target = ctx->scratch[2];
    *ldt = ctx->ld;
  }
  return BO_OK;
}
int finish_out(bo_ctx ctx, double* q, uint64_t ldq, int K, double* target, bo_status* st) {
  if (target != q)
    CU(cudaMemcpy2DAsync(q, ldq * 8, target, ctx->ld * 8, ctx->n_local * 8, K, cudaMemcpyDeviceToDevice,
                         ctx->stream));
  return BO_OK;
}
}  // namespace host
}  // namespace bo

extern "C" int bo_gram(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, double* g, uint64_t ledger[4],
                       bo_status* st) {
  ok_st(st);
  CU(cudaSetDevice(ctx->device));
  const double* vv;
  uint64_t lv;
  TRY(stage_input(ctx, v, ldv, k, 0, &vv, &lv, st));
  TRY(reset_status(ctx, st));
  PassReq r{};
  r.kind = PK_GRAM;
  r.K = (int)k;
  r.V = vv;
  r.ldv = lv;
  r.fin.ops = FIN_COPY_G;
  r.fin.Gout = T_(ctx, OFF_G);
  TRY(run_pass(ctx, r, st));
  TRY(fetch(ctx, true, st));
  copy_factor_host(ctx->tiny_host + OFF_G, (int)k, g);
  if (ledger) ledger[BO_LEDGER_GRAM]++;
  return BO_OK;
}

extern "C" int bo_apply_inv_upper(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, const double* r, double* x,
                                  uint64_t ldx, bo_status* st) {
  ok_st(st);
  CU(cudaSetDevice(ctx->device));
  for (uint64_t j = 0; j < k; ++j)
    if (r[j + j * k] == 0.0)
      return set_st(st, BO_SINGULAR_TRIANGULAR, (long long)j, 0.0,
                    "triangular factor is singular: zero diagonal at index %llu", (unsigned long long)j);
  const double* vv;
  uint64_t lv;
  TRY(stage_input(ctx, v, ldv, k, 0, &vv, &lv, st));
  double* h = ctx->tiny_host + OFF_R4;
  for (int e = 0; e < 256; ++e) h[e] = 0.0;
  for (uint64_t j = 0; j < k; ++j)
    for (uint64_t i = 0; i <= j; ++i) h[i + j * 16] = r[i + j * k];
  CU(cudaMemcpyAsync(T_(ctx, OFF_R4), h, 256 * 8, cudaMemcpyHostToDevice, ctx->stream));
  TRY(reset_status(ctx, st));
  double* tgt;
  uint64_t ldt;
  write_out(ctx, x, ldx, (int)k, &tgt, &ldt);
  PassReq w{};
  w.kind = PK_P1_ST;
  w.K = (int)k;
  w.V = vv;
  w.ldv = lv;
  w.out = tgt;
  w.ldo = ldt;
  w.Rpre0 = T_(ctx, OFF_R4);
  w.exact = true;
  TRY(run_pass(ctx, w, st));
  TRY(finish_out(ctx, x, ldx, (int)k, tgt, st));
  CU(cudaStreamSynchronize(ctx->stream));
  return BO_OK;
}

extern "C" int bo_cholqr(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, double* q, uint64_t ldq, double* r,
                         uint64_t ledger[4], bo_status* st) {
  ok_st(st);
  CU(cudaSetDevice(ctx->device));
  const double* vv;
  uint64_t lv;
  TRY(stage_input(ctx, v, ldv, k, 0, &vv, &lv, st));
  TRY(reset_status(ctx, st));
  double* tgt;
  uint64_t ldt;
  write_out(ctx, q, ldq, (int)k, &tgt, &ldt);
  TRY(dev_cholqr(ctx, vv, lv, (int)k, tgt, ldt, OFF_R1, 1, st));
  TRY(fetch(ctx, true, st));
  if (ledger) ledger[BO_LEDGER_GRAM]++;
  TRY(dev_error(ctx, "cholqr", st));
  TRY(finish_out(ctx, q, ldq, (int)k, tgt, st));
  CU(cudaStreamSynchronize(ctx->stream));
  if (r) copy_factor_host(ctx->tiny_host + OFF_R1, (int)k, r);
  return BO_OK;
}

namespace bo {
namespace host {
int intra_api(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, int intra, bo_sketch sk, double* q,
              uint64_t ldq, double* r, uint64_t ledger[4], bo_status* st) {
  ok_st(st);
  CU(cudaSetDevice(ctx->device));
  if (intra == BO_INTRA_RAND_CHOLQR && !sk)
    return set_st(st, BO_INVALID, 0, 0.0, "rand_cholqr intra-orthogonalization needs a sketch operator");
  const double* vv;
  uint64_t lv;
  TRY(stage_input(ctx, v, ldv, k, 0, &vv, &lv, st));
  TRY(reset_status(ctx, st));
  double* tgt;
  uint64_t ldt;
  write_out(ctx, q, ldq, (int)k, &tgt, &ldt);
  TRY(dev_intra(ctx, vv, lv, (int)k, intra, sk, tgt, ldt, st));
  TRY(fetch(ctx, true, st));
  const DevStatus& d = *ctx->status_host;
  if (ledger) {
    // cholqr2: gram, gram ; rand_cholqr: sketch, gram (intra_orth.cpp:21-39)
    const int upto = d.code ? d.pass : 2;
    if (upto >= 1) ledger[intra == BO_INTRA_CHOLQR2 ? BO_LEDGER_GRAM : BO_LEDGER_SKETCH]++;
    if (upto >= 2) ledger[BO_LEDGER_GRAM]++;
  }
  TRY(dev_error(ctx, "cholqr", st));
  TRY(finish_out(ctx, q, ldq, (int)k, tgt, st));
  CU(cudaStreamSynchronize(ctx->stream));
  if (r) copy_factor_host(ctx->tiny_host + OFF_RIN, (int)k, r);
  return BO_OK;
}
}  // namespace host
}  // namespace bo

extern "C" int bo_cholqr2(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, double* q, uint64_t ldq, double* r,
                          uint64_t ledger[4], bo_status* st) {
  return intra_api(ctx, v, ldv, k, BO_INTRA_CHOLQR2, nullptr, q, ldq, r, ledger, st);
}
extern "C" int bo_rand_cholqr(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, bo_sketch sk, double* q,
                              uint64_t ldq, double* r, uint64_t ledger[4], bo_status* st) {
  return intra_api(ctx, v, ldv, k, BO_INTRA_RAND_CHOLQR, sk, q, ldq, r, ledger, st);
}

// ===========================================================================
// BasisStore
// ===========================================================================
extern "C" int bo_basis_create(bo_ctx ctx, uint64_t capacity, bo_basis* out, bo_status* st) {
  ok_st(st);
  *out = nullptr;
  CU(cudaSetDevice(ctx->device));
  bo_basis b = new bo_basis_s();
  b->ctx = ctx;
  b->cap = capacity;
  const size_t qbytes = std::max<uint64_t>(ctx->ld * capacity, 1) * 8;
  if (ctx->spare_q && ctx->spare_q_bytes >= qbytes) {  // recycled from a destroyed store
    b->q = ctx->spare_q;
    b->q_bytes = ctx->spare_q_bytes;
    ctx->spare_q = nullptr;
  } else {
    cudaError_t e = cudaMalloc(&b->q, qbytes);
    if (e != cudaSuccess) {
      delete b;
      return set_st(st, BO_CUDA, 0, 0.0, "cudaMalloc(basis) failed: %s", cudaGetErrorString(e));
    }
    b->q_bytes = qbytes;
  }
  cudaMemsetAsync(b->q, 0, ctx->ld * capacity * 8, ctx->stream);
  if (ctx->spare_snap) {
    b->snap = ctx->spare_snap;
    ctx->spare_snap = nullptr;
  }
  b->r.assign(capacity * capacity, 0.0);
  b->c.assign(capacity * capacity, 0.0);
  b->seeded.assign(capacity, 0);
  *out = b;
  return BO_OK;
}
extern "C" int bo_basis_destroy(bo_basis b) {
  if (!b) return BO_OK;
  basis_drain(b);
  bo_ctx ctx = b->ctx;
  cudaStreamSynchronize(ctx->stream);
  if (b->snap) {
    if (!ctx->spare_snap) ctx->spare_snap = b->snap;  // keep one pinned snapshot area
    else cudaFreeHost(b->snap);
  }
  if (!ctx->spare_q || ctx->spare_q_bytes < b->q_bytes) {  // keep the larger slab for the next store
    if (ctx->spare_q) cudaFree(ctx->spare_q);
    ctx->spare_q = b->q;
    ctx->spare_q_bytes = b->q_bytes;
  } else {
    cudaFree(b->q);
  }
  delete b;
  return BO_OK;
}
extern "C" int bo_basis_reset(bo_basis b) {
  basis_drain(b);
  b->deferred_code = 0;
  b->cols = 0;
  std::fill(b->r.begin(), b->r.end(), 0.0);
  std::fill(b->c.begin(), b->c.end(), 0.0);
  std::fill(b->seeded.begin(), b->seeded.end(), 0);
  b->bounds.clear();
  b->bp_lo = 0;
  b->sk.clear();
  b->sk_rows = b->sk_cols = 0;
  for (auto& l : b->ledger) l = 0;
  return BO_OK;
}
extern "C" uint64_t bo_basis_cols(bo_basis b) { return b->cols; }
extern "C" uint64_t bo_basis_capacity(bo_basis b) { return b->cap; }
extern "C" double* bo_basis_q_device(bo_basis b, uint64_t* ld) {
  if (ld) *ld = b->ctx->ld;
  return b->q;
}
extern "C" int bo_basis_ledger(bo_basis b, uint64_t out[4]) {
  basis_drain(b);
  std::memcpy(out, b->ledger, sizeof b->ledger);
  return BO_OK;
}
extern "C" int bo_basis_r_copy(bo_basis b, double* out) {  // block_orth.cpp:33-38
  basis_drain(b);
  for (uint64_t j = 0; j < b->cols; ++j)
    for (uint64_t i = 0; i < b->cols; ++i) out[i + j * b->cols] = i <= j ? b->r[i + j * b->cap] : 0.0;
  return BO_OK;
}
extern "C" double bo_basis_r_entry(bo_basis b, uint64_t i, uint64_t j) {
  basis_drain(b);
  return b->r[i + j * b->cap];
}
extern "C" int bo_basis_c_copy(bo_basis b, double* out) {
  basis_drain(b);
  for (uint64_t j = 0; j < b->cols; ++j)
    for (uint64_t i = 0; i < b->cols; ++i) out[i + j * b->cols] = b->c[i + j * b->cap];
  return BO_OK;
}
extern "C" int bo_basis_mark_seed(bo_basis b, uint64_t col) {  // block_orth.cpp:40-45
  if (col >= b->cols) return BO_INVALID;
  if (!b->pend.empty()) {  // after the enqueued calls, in program order (bo_basis_sync)
    bo_basis_s::Pending op;
    op.kind = 1;
    op.col = col;
    b->pend.push_back(op);
    return BO_OK;
  }
  for (uint64_t i = 0; i < b->cap; ++i) b->c[i + col * b->cap] = 0.0;
  b->c[col + col * b->cap] = 1.0;
  b->seeded[col] = 1;
  return BO_OK;
}
extern "C" int bo_basis_is_seed(bo_basis b, uint64_t col) {
  basis_drain(b);
  return col < b->cap && b->seeded[col];
}
extern "C" int bo_basis_input_coeff_col(bo_basis b, uint64_t k, uint64_t len, double* out) {  // :47-52
  basis_drain(b);
  const std::vector<double>& src = bo_basis_is_seed(b, k) ? b->c : b->r;
  for (uint64_t i = 0; i < len; ++i) out[i] = src[i + k * b->cap];
  return BO_OK;
}
extern "C" int bo_basis_begin_big_panel(bo_basis b, uint64_t sketch_rows, int overlap) {  // :54-57
  basis_drain(b);
  b->bp_lo = b->cols - ((overlap && b->cols > 0) ? 1 : 0);
  b->sk.clear();
  b->sk_rows = sketch_rows;
  b->sk_cols = 0;
  return BO_OK;
}
extern "C" uint64_t bo_basis_big_panel_lo(bo_basis b) { return b->bp_lo; }
extern "C" uint64_t bo_basis_num_boundaries(bo_basis b) {
  basis_drain(b);
  return b->bounds.size();
}
extern "C" int bo_basis_boundaries(bo_basis b, uint64_t* out) {
  basis_drain(b);
  for (size_t i = 0; i < b->bounds.size(); ++i) out[i] = b->bounds[i];
  return BO_OK;
}
extern "C" uint64_t bo_basis_sketched(bo_basis b, double* out, uint64_t* rows) {
  basis_drain(b);
  if (rows) *rows = b->sk_rows;
  if (out && !b->sk.empty()) std::memcpy(out, b->sk.data(), b->sk.size() * 8);
  return b->sk_cols;
}
extern "C" int bo_basis_cols_to_host(bo_basis b, uint64_t lo, uint64_t hi, double* out, bo_status* st) {
  ok_st(st);
  TRY(basis_drain(b));
  bo_ctx ctx = b->ctx;
  if (hi < lo || hi > b->cap) return set_st(st, BO_INVALID, 0, 0.0, "bad column range");
  CU(cudaStreamSynchronize(ctx->stream));
  if (hi > lo)
    CU(cudaMemcpy2D(out, ctx->n_local * 8, b->q + lo * ctx->ld, ctx->ld * 8, ctx->n_local * 8, hi - lo,
                    cudaMemcpyDeviceToHost));
  return BO_OK;
}

extern "C" int bo_basis_last_push(bo_basis b, uint64_t* base, uint64_t* k, int* overlap, double* proj,
                                  double* diag) {
  basis_drain(b);
  if (base) *base = b->last_base;
  if (k) *k = b->last_k;
  if (overlap) *overlap = b->last_overlap;
  if (proj) std::copy(b->last_proj.begin(), b->last_proj.end(), proj);
  if (diag) std::copy(b->last_diag.begin(), b->last_diag.end(), diag);
  return BO_OK;
}

extern "C" int bo_basis_import(bo_basis b, uint64_t cols, const double* q_host, uint64_t ldq, const double* r,
                               const double* c, const unsigned char* seeded, const uint64_t* bounds,
                               uint64_t nbounds, bo_status* st) {
  ok_st(st);
  TRY(basis_drain(b));
  bo_ctx ctx = b->ctx;
  if (cols > b->cap) return set_st(st, BO_INVALID, 0, 0.0, "import: %llu columns exceed the capacity %llu",
                                   (unsigned long long)cols, (unsigned long long)b->cap);
  if (cols > 0 && ldq < ctx->n_local) return set_st(st, BO_INVALID, 0, 0.0, "import: ldq < local rows");
  // on the ctx stream: a pageable cudaMemcpy on the legacy stream may return
  // before its DMA lands, and the non-blocking ctx stream would not wait for it
  // (the reference driver's every-restart import raced its first pass)
  if (cols > 0)
    CU(cudaMemcpy2DAsync(b->q, ctx->ld * 8, q_host, ldq * 8, ctx->n_local * 8, cols, cudaMemcpyHostToDevice,
                         ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  const uint64_t cap = b->cap;
  std::fill(b->r.begin(), b->r.end(), 0.0);
  std::fill(b->c.begin(), b->c.end(), 0.0);
  std::fill(b->seeded.begin(), b->seeded.end(), 0);
  for (uint64_t j = 0; j < cols; ++j) {
    for (uint64_t i = 0; i < cols; ++i) {
      b->r[i + j * cap] = r[i + j * cols];
      if (c) b->c[i + j * cap] = c[i + j * cols];
    }
    b->seeded[j] = seeded ? seeded[j] : 0;
  }
  b->bounds.assign(bounds, bounds + nbounds);
  b->cols = cols;
  return BO_OK;
}

namespace bo {
namespace host {
// push_panel bookkeeping (block_orth.cpp:57-98) — Q columns are already in the slab
// proj: base x k (ld ldp), diag: k x k (ld ldd)
void push_panel_host(bo_basis b, uint64_t k, const double* proj, uint64_t ldp, const double* diag, uint64_t ldd,
                     bool overlap) {
  const uint64_t cap = b->cap;
  const uint64_t base = overlap ? b->cols - 1 : b->cols;
  b->last_base = base;
  b->last_k = k;
  b->last_overlap = overlap ? 1 : 0;
  b->last_proj.assign(base * k, 0.0);
  b->last_diag.assign(k * k, 0.0);
  for (uint64_t j = 0; j < k; ++j) {
    for (uint64_t i = 0; i < base; ++i) b->last_proj[i + j * base] = proj[i + j * ldp];
    for (uint64_t i = 0; i <= j; ++i) b->last_diag[i + j * k] = diag[i + j * ldd];
  }
  if (overlap) {  // fold_overlap_column (block_orth.cpp:59-73)
    const uint64_t k0 = b->cols - 1;
    const double scale = diag[0];
    const double r_diag = b->r[k0 + k0 * cap];
    for (uint64_t i = 0; i < k0; ++i) b->r[i + k0 * cap] += r_diag * proj[i];
    b->r[k0 + k0 * cap] = r_diag * scale;
    if (b->seeded[k0]) {
      const double c_diag = b->c[k0 + k0 * cap];
      for (uint64_t i = 0; i < k0; ++i) b->c[i + k0 * cap] += c_diag * proj[i];
      b->c[k0 + k0 * cap] = c_diag * scale;
    }
  }
  for (uint64_t j = 0; j < k; ++j) {
    const uint64_t g = base + j;
    if (!(overlap && j == 0)) {
      for (uint64_t i = 0; i < base; ++i) b->r[i + g * cap] = proj[i + j * ldp];
      for (uint64_t i = 0; i <= j; ++i) b->r[base + i + g * cap] = diag[i + j * ldd];
    }
  }
  b->bounds.push_back(base);
  b->cols = base + k;
}
}  // namespace host
}  // namespace bo

// ===========================================================================
// bcgs_project_range / bcgs2
// ===========================================================================
namespace bo {
namespace host {
// P1: C = Q^T V (slot Cslot) ; P2: Vhat = V - Q C (stored)
int dev_project(bo_basis b, const double* v, uint64_t ldv, int K, uint64_t lo, uint64_t hi, double* vhat,
                uint64_t ldvh, int Cslot, int pass_id, bo_status* st) {
  bo_ctx ctx = b->ctx;
  const int p = (int)(hi - lo);
  PassReq r1{};
  r1.kind = PK_QTX;
  r1.K = K;
  r1.V = v;
  r1.ldv = ldv;
  r1.Q = b->q + lo * ctx->ld;
  r1.ldq = ctx->ld;
  r1.p = p;
  r1.pass_id = pass_id;
  r1.fin.ops = FIN_COPY_Q;
  r1.fin.Cq = T_(ctx, Cslot);
  TRY(run_pass(ctx, r1, st));
  PassReq r2{};
  r2.kind = PK_UPD_ST;
  r2.K = K;
  r2.V = v;
  r2.ldv = ldv;
  r2.Q = r1.Q;
  r2.ldq = ctx->ld;
  r2.p = p;
  r2.Cm = T_(ctx, Cslot);
  r2.out = vhat;
  r2.ldo = ldvh;
  r2.pass_id = pass_id;
  return run_pass(ctx, r2, st);
}
}  // namespace host
}  // namespace bo

extern "C" int bo_bcgs_project_range(bo_basis b, const double* v, uint64_t ldv, uint64_t k, uint64_t lo, uint64_t hi,
                                     double* vhat, uint64_t ldvh, double* coeffs, bo_status* st) {
  ok_st(st);
  TRY(basis_drain(b));
  bo_ctx ctx = b->ctx;
  CU(cudaSetDevice(ctx->device));
  if (lo > hi || hi > b->cols) return set_st(st, BO_INVALID, 0, 0.0, "bad projection range");
  const double* vv;
  uint64_t lv;
  TRY(stage_input(ctx, v, ldv, k, 0, &vv, &lv, st));
  double* tgt;
  uint64_t ldt;
  write_out(ctx, vhat, ldvh, (int)k, &tgt, &ldt);
  if (hi == lo) {  // no reduce: vhat = v
    CU(cudaMemcpy2DAsync(vhat, ldvh * 8, vv, lv * 8, ctx->n_local * 8, k, cudaMemcpyDeviceToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return BO_OK;
  }
  TRY(reset_status(ctx, st));
  TRY(dev_project(b, vv, lv, (int)k, lo, hi, tgt, ldt, OFF_C1, 1, st));
  TRY(finish_out(ctx, vhat, ldvh, (int)k, tgt, st));
  TRY(fetch(ctx, true, st));
  b->ledger[BO_LEDGER_PROJECTION]++;
  const uint64_t p = hi - lo;
  if (coeffs)
    for (uint64_t j = 0; j < k; ++j)
      for (uint64_t i = 0; i < p; ++i) coeffs[i + j * p] = ctx->tiny_host[OFF_C1 + i + j * LDC];
  return BO_OK;
}

namespace bo {
namespace host {
// pinned snapshot of one enqueued call: its status word and the tiny factors
// its host bookkeeping needs (Rin for a first panel; coefficients and R_jj)
int snapshot(bo_basis b, bo_basis_s::Pending& op, bo_status* st) {
  bo_ctx ctx = b->ctx;
  if (!b->snap) CU(cudaMallocHost((void**)&b->snap, (size_t)kSnapSlots * kSnapLen * 8));
  op.slot = b->nsnap++;
  double* sn = b->snap + (size_t)op.slot * kSnapLen;
  // one copy of [status | Rin] (first panel) or [status | Rin | R_jj | coefficients]
  const size_t len = op.first ? (size_t)OFF_RJJ : (size_t)kSnapLen;
  CU(cudaMemcpyAsync(sn, ctx->tiny + OFF_STATUS, len * 8, cudaMemcpyDeviceToHost, ctx->stream));
  b->pend.push_back(op);
  b->cols = op.cols_before - (op.overlap ? 1 : 0) + op.k;  // speculative: as if the call succeeds
  return BO_OK;
}

int basis_drain(bo_basis b) {
  if (b->pend.empty()) return BO_OK;
  bo_status tmp;
  uint64_t failed = 0;
  const uint64_t before = b->deferred_code ? b->deferred_call : 0;
  const int rc = bo_basis_sync(b, &failed, &tmp);
  if (rc == BO_CUDA || rc == BO_NCCL) return rc;
  if (rc != BO_OK && !b->deferred_code) {
    b->deferred_code = rc;
    b->deferred_st = tmp;
    b->deferred_call = before + failed;
  }
  return BO_OK;
}
}  // namespace host
}  // namespace bo

// bcgs2 (block_orth.cpp:207-226), enqueued: the passes and a snapshot of the
// call's status word and output factors go on the stream; the host bookkeeping
// is replayed by bo_basis_sync.  No host wait.
extern "C" int bo_bcgs2_enqueue(bo_basis b, const double* v, uint64_t ldv, uint64_t k, int intra, bo_sketch theta,
                                int overlap, bo_status* st) {
  ok_st(st);
  bo_ctx ctx = b->ctx;
  CU(cudaSetDevice(ctx->device));
  const int K = (int)k;
  const bool eff_overlap = overlap && b->cols > 0;
  const uint64_t hi = b->cols - (eff_overlap ? 1 : 0);
  const uint64_t base = hi;  // push_panel base == hi in both cases
  if (base + k > b->cap) return set_st(st, BO_INVALID, 0, 0.0, "basis capacity exceeded");
  if (intra == BO_INTRA_RAND_CHOLQR && !theta)
    return set_st(st, BO_INVALID, 0, 0.0, "rand_cholqr intra-orthogonalization needs a sketch operator");
  if (intra != BO_INTRA_CHOLQR2 && intra != BO_INTRA_RAND_CHOLQR)
    return set_st(st, BO_INVALID, 0, 0.0, "unknown intra kind");
  const double* vv;
  uint64_t lv;
  if (b->pend.size() >= (size_t)kSnapSlots) TRY(basis_drain(b));  // bounded queue
  TRY(stage_input(ctx, v, ldv, k, 0, &vv, &lv, st));
  double* qout = b->q + base * ctx->ld;
  if (b->pend.empty()) TRY(reset_status(ctx, st));  // sticky across a batch: later calls skip after a failure
  const bool rand = intra == BO_INTRA_RAND_CHOLQR;
  bo_basis_s::Pending op;
  op.kind = 0;
  op.k = k;
  op.cols_before = b->cols;
  op.overlap = eff_overlap;
  op.rand = rand;

  if (hi == 0) {  // first panel: intra only (block_orth.cpp:212-215)
    TRY(dev_intra(ctx, vv, lv, K, intra, theta, qout, ctx->ld, st));
    op.first = true;
    TRY(snapshot(b, op, st));
    return BO_OK;
  }

  const int p = (int)hi;
  double* vhat = ctx->scratch[1];
  const double* Q = b->q;
  // P1: C1 = Q^T V
  PassReq r1{};
  r1.kind = PK_QTX;
  r1.K = K;
  r1.V = vv;
  r1.ldv = lv;
  r1.Q = Q;
  r1.ldq = ctx->ld;
  r1.p = p;
  r1.pass_id = 1;
  r1.fin.ops = FIN_COPY_Q;
  r1.fin.Cq = T_(ctx, OFF_C1);
  TRY(run_pass(ctx, r1, st));
  // P2: Vhat = V - Q C1 ; G1 = Vhat^T Vhat -> R1  |  S = Theta^T Vhat -> Rs (R1)
  PassReq r2{};
  r2.kind = rand ? (theta->kind == BO_SKETCH_GAUSSIAN ? PK_UPD_SKG_ST : PK_UPD_SKC_ST) : PK_UPD_GRAM_ST;
  r2.K = K;
  r2.V = vv;
  r2.ldv = lv;
  r2.Q = Q;
  r2.ldq = ctx->ld;
  r2.p = p;
  r2.Cm = T_(ctx, OFF_C1);
  r2.out = vhat;
  r2.ldo = ctx->ld;
  r2.sk = rand ? theta : nullptr;
  r2.pass_id = 2;
  if (rand) {
    r2.fin.ops = FIN_HH;
    r2.fin.Rhh = T_(ctx, OFF_R1);
  } else {
    r2.fin.ops = FIN_CHOL;
    r2.fin.Rchol = T_(ctx, OFF_R1);
  }
  TRY(run_pass(ctx, r2, st));
  // P3: Y = Vhat R1^-1 ; G = Y^T Y -> R2 ; Rin = R2 R1
  PassReq r3{};
  r3.kind = PK_P1_GRAM;
  r3.K = K;
  r3.V = vhat;
  r3.ldv = ctx->ld;
  r3.Rpre0 = T_(ctx, OFF_R1);
  r3.pass_id = 3;
  r3.fin.ops = FIN_CHOL | FIN_MULT;
  r3.fin.Rchol = T_(ctx, OFF_R2);
  r3.fin.Rin = T_(ctx, OFF_R1);
  r3.fin.rjj = T_(ctx, OFF_RIN);
  TRY(run_pass(ctx, r3, st));
  // P4: Qhat = Vhat R1^-1 R2^-1 ; C2 = Q^T Qhat.  With the product factor
  // (default) the row solve is Vhat Rin^-1, Rin = R2 R1 (P3's FIN_MULT):
  // one triangular solve per row instead of two.  The reference solves twice
  // (intra_orth.cpp:28-39); the single solve differs from it by rounding
  // amplified by cond(R1) (the problem's own sensitivity; P5/P6 re-
  // orthogonalise), and halves the FP64 solve work of the two solve warps,
  // which share their sub-partitions' FP64 pipe with the DMMA contraction.
  static const bool pre_product = [] {
    const char* e = getenv("BO_PRE_PRODUCT");
    return e ? atoi(e) != 0 : true;
  }();
  PassReq r4{};
  r4.kind = pre_product ? PK_P1_QTX : PK_P2_QTX;
  r4.K = K;
  r4.V = vhat;
  r4.ldv = ctx->ld;
  r4.Q = Q;
  r4.ldq = ctx->ld;
  r4.p = p;
  r4.Rpre0 = pre_product ? T_(ctx, OFF_RIN) : T_(ctx, OFF_R1);
  r4.Rpre1 = pre_product ? nullptr : T_(ctx, OFF_R2);
  r4.pass_id = 4;
  r4.fin.ops = FIN_COPY_Q;
  r4.fin.Cq = T_(ctx, OFF_C2);
  TRY(run_pass(ctx, r4, st));
  // P5: Z = Qhat - Q C2 (in place over Vhat) ; G3 = Z^T Z -> R3 ; coeffs, rjj
  PassReq r5{};
  r5.kind = pre_product ? PK_P1_UPD_GRAM_ST : PK_P2_UPD_GRAM_ST;
  r5.K = K;
  r5.V = vhat;
  r5.ldv = ctx->ld;
  r5.Q = Q;
  r5.ldq = ctx->ld;
  r5.p = p;
  r5.Rpre0 = pre_product ? T_(ctx, OFF_RIN) : T_(ctx, OFF_R1);
  r5.Rpre1 = pre_product ? nullptr : T_(ctx, OFF_R2);
  r5.Cm = T_(ctx, OFF_C2);
  r5.out = vhat;
  r5.ldo = ctx->ld;
  r5.pass_id = 5;
  r5.fin.ops = FIN_CHOL | FIN_COEFF;
  r5.fin.Rchol = T_(ctx, OFF_R3);
  r5.fin.C1 = T_(ctx, OFF_C1);
  r5.fin.C2 = T_(ctx, OFF_C2);
  r5.fin.Rin = T_(ctx, OFF_RIN);
  r5.fin.coeffs = T_(ctx, OFF_COEF);
  r5.fin.rjj = T_(ctx, OFF_RJJ);
  TRY(run_pass(ctx, r5, st));
  // P6: Q_out = Z R3^-1 written in place into the basis slab
  PassReq r6{};
  r6.kind = PK_P1_ST;
  r6.K = K;
  r6.V = vhat;
  r6.ldv = ctx->ld;
  r6.Rpre0 = T_(ctx, OFF_R3);
  r6.out = qout;
  r6.ldo = ctx->ld;
  r6.pass_id = 6;
  TRY(run_pass(ctx, r6, st));
  TRY(snapshot(b, op, st));
  return BO_OK;
}

// Complete the store's enqueued calls in program order: ledger events,
// push_panel bookkeeping and deferred mark_seeds, up to the first failing
// call, whose error is returned (*failed = its index among the enqueued
// calls).  Calls after it were no-ops on the device (sticky status) and are
// dropped, so the store is left as the sequential API would leave it.
extern "C" int bo_basis_sync(bo_basis b, uint64_t* failed, bo_status* st) {
  ok_st(st);
  if (failed) *failed = 0;
  if (b->pend.empty()) {
    const int code = b->deferred_code;
    if (code) {
      if (st) *st = b->deferred_st;
      if (failed) *failed = b->deferred_call;
      b->deferred_code = 0;
    }
    return code;
  }
  bo_ctx ctx = b->ctx;
  CU(cudaStreamSynchronize(ctx->stream));
  std::vector<bo_basis_s::Pending> ops;
  ops.swap(b->pend);
  b->nsnap = 0;
  b->cols = ops.front().cols_before;
  int rc = BO_OK;
  uint64_t call = 0;
  for (const bo_basis_s::Pending& op : ops) {
    if (op.kind == 1) {  // deferred mark_seed (block_orth.cpp:40-45)
      for (uint64_t i = 0; i < b->cap; ++i) b->c[i + op.col * b->cap] = 0.0;
      b->c[op.col + op.col * b->cap] = 1.0;
      b->seeded[op.col] = 1;
      continue;
    }
    DevStatus d;
    std::memcpy(&d, b->snap + (size_t)op.slot * kSnapLen + kSnapStatus, sizeof d);
    const double* sn = b->snap + (size_t)op.slot * kSnapLen;
    // ledger: the reduce events the call reached (block_orth.cpp:212-221)
    if (op.first) {
      const int upto = d.code ? d.pass : 2;
      if (upto >= 1) b->ledger[op.rand ? BO_LEDGER_SKETCH : BO_LEDGER_GRAM]++;
      if (upto >= 2) b->ledger[BO_LEDGER_GRAM]++;
    } else {
      const int upto = d.code ? d.pass : 5;
      if (upto >= 1) b->ledger[BO_LEDGER_PROJECTION]++;
      if (upto >= 2) b->ledger[op.rand ? BO_LEDGER_SKETCH : BO_LEDGER_GRAM]++;
      if (upto >= 3) b->ledger[BO_LEDGER_GRAM]++;
      if (upto >= 4) b->ledger[BO_LEDGER_PROJECTION]++;
      if (upto >= 5) b->ledger[BO_LEDGER_GRAM]++;
    }
    if (d.code != ST_OK) {
      *ctx->status_host = d;
      rc = dev_error(ctx, "cholqr", st);
      if (failed) *failed = call;
      break;
    }
    if (op.first)
      push_panel_host(b, op.k, nullptr, 1, sn + kSnapRin, 16, op.overlap);
    else
      push_panel_host(b, op.k, sn + kSnapCoef, LDC, sn + kSnapRjj, 16, op.overlap);
    ++call;
  }
  {
    bo_status t2;
    const int r2 = reset_status(ctx, &t2);
    if (r2 != BO_OK) {
      if (st) *st = t2;
      return r2;
    }
  }
  return rc;
}

// bcgs2 with the reference's synchronous contract: enqueue, then sync
extern "C" int bo_bcgs2(bo_basis b, const double* v, uint64_t ldv, uint64_t k, int intra, bo_sketch theta,
                        int overlap, bo_status* st) {
  TRY(basis_drain(b));
  const int rc = bo_bcgs2_enqueue(b, v, ldv, k, intra, theta, overlap, st);
  if (rc != BO_OK) {
    bo_status tmp;
    bo_basis_sync(b, nullptr, &tmp);  // drop what was enqueued
    return rc;
  }
  return bo_basis_sync(b, nullptr, st);
}

extern "C" int bo_mt64_jump_window(uint64_t seed, uint64_t J, uint64_t* out312) {
  if (!bo::mt64::ready()) return BO_INVALID;
  bo::mt64::jump_window_host(seed, J, out312);
  return BO_OK;
}

// Diagnostic: per-phase cycle counters of the pass kernels (only a library
// built with -DBO_PHASE_PROF=1 fills them).  Copies the 16 x 16 counters to
// out (when non-null) and zeroes them; the first call allocates them.
extern "C" int bo_debug_phase_prof(bo_ctx ctx, unsigned long long* out) {
  if (!ctx) return BO_INVALID;
  if (!ctx->phase_prof) {
    if (cudaMalloc(&ctx->phase_prof, 256 * sizeof(unsigned long long)) != cudaSuccess) return BO_CUDA;
  } else if (out) {
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return BO_CUDA;
    if (cudaMemcpy(out, ctx->phase_prof, 256 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
      return BO_CUDA;
  }
  if (cudaMemsetAsync(ctx->phase_prof, 0, 256 * sizeof(unsigned long long), ctx->stream) != cudaSuccess)
    return BO_CUDA;
  return BO_OK;
}

// Diagnostic / CPU test hook: the count_gauss dense stage for a sketch seed
// (mc x mhat, column-major), drawn exactly as bo_sketch_build draws it.
extern "C" int bo_debug_count_gauss_stage(uint64_t seed, uint64_t mc, uint64_t mhat, double* out) {
  const std::vector<double> t = bo::host::gen_theta_g(seed, mc, mhat);
  std::memcpy(out, t.data(), t.size() * 8);
  return BO_OK;
}
