// blkorth_gpu.hpp — header-only C++ adapter that re-presents the C ABI
// (bo_cuda.h) with the reference blkorth signatures and exception types, so a
// maintainer of /root/reference/proj can switch the solver's orthogonalization
// / operator calls to the GPU with minimal edits.
//
//   reference (namespace blkorth)                      adapter (blkorth::gpu)
//   SketchOperator::build(kind, n, shat, seed)  sketch.hpp:28   SketchOperator::build(ctx, ...)
//   SketchOperator::apply(v, ledger)            sketch.hpp:40   SketchOperator::apply(panel, ledger)
//   cholqr / cholqr2 / rand_cholqr              intra_orth.hpp:19-28
//   recursive_cholqr                            intra_orth.hpp:50
//   BasisStore                                  block_orth.hpp:27-102
//   bcgs_project_range / bcgs2 / bcgs_pip / rand_bcgs_preproc / two_stage_*
//                                               block_orth.hpp:111-169
//   mpk / spmv                                  gmres.hpp:65, sparse.hpp:49
//   sstep_gmres_solve                           gmres.hpp:92
// Tall arguments are DevicePanel views (device pointer, leading dimension,
// columns) of this rank's row shard instead of host DenseMatrix objects.
#pragma once

#include <array>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "bo_cuda.h"
#if defined(BLKORTH_GPU_REFERENCE_TYPES)
#include "blkorth/dense.hpp"
#include "blkorth/errors.hpp"
#endif

namespace blkorth {
namespace gpu {

// CUDA / NCCL faults are not numerical breakdowns: they derive from
// std::runtime_error only, so the reference driver's `catch (const Error&)`
// (gmres.cpp:429-435) never routes them into recover_panel.
struct DeviceError : std::runtime_error {
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

#if defined(BLKORTH_GPU_REFERENCE_TYPES)
// ---- built against /root/reference/proj/include: the reference's own types.
// Every library status is rethrown as the reference exception, constructed
// with the reference's arguments, so what() is the reference text
// (errors.hpp:12-92) and `catch (const blkorth::Error&)` sees it.
using ::blkorth::AllColumnsDiscarded;
using ::blkorth::AmbientTooSmall;
using ::blkorth::BannerError;
using ::blkorth::CholeskyBreakdown;
using ::blkorth::Error;
using ::blkorth::InvalidScheme;
using ::blkorth::ParseError;
using ::blkorth::RankDeficient;
using ::blkorth::ReduceLedger;
using ::blkorth::ReducePhase;
using ::blkorth::SingularTriangular;
using ::blkorth::UpperTriangular;
using ::blkorth::ZeroMatrix;

inline std::string after(const std::string& m, const std::string& prefix) {
  return m.compare(0, prefix.size(), prefix) == 0 ? m.substr(prefix.size()) : m;
}

inline void check(int rc, const bo_status& st) {
  if (rc == BO_OK) return;
  const std::string m(st.msg);
  switch (rc) {
    case BO_CHOLESKY_BREAKDOWN: {  // "<context>: nonpositive Cholesky pivot at step <k>"
      const std::size_t at = m.find(": nonpositive Cholesky pivot");
      throw CholeskyBreakdown((std::size_t)st.index, at == std::string::npos ? m : m.substr(0, at));
    }
    case BO_SINGULAR_TRIANGULAR: throw SingularTriangular((std::size_t)st.index);
    case BO_AMBIENT_TOO_SMALL: {
      unsigned long long n = 0, mh = 0;
      std::sscanf(st.msg, "ambient dimension n=%llu must exceed sketch size mhat=%llu", &n, &mh);
      throw AmbientTooSmall((std::size_t)n, (std::size_t)mh);
    }
    case BO_ALL_COLUMNS_DISCARDED: throw AllColumnsDiscarded();
    case BO_RANK_DEFICIENT: throw RankDeficient(m);
    case BO_ZERO_MATRIX: throw ZeroMatrix();
    case BO_INVALID: throw InvalidScheme(m);
    case BO_PARSE_ERROR: {
      const std::string tail = after(m, "parse error at line ");
      const std::size_t colon = tail.find(": ");
      throw ParseError((std::size_t)st.index, colon == std::string::npos ? tail : tail.substr(colon + 2));
    }
    case BO_BANNER_ERROR: throw BannerError(after(m, "unsupported MatrixMarket banner: "));
    default: throw DeviceError(m);
  }
}
#else
// ---- standalone: exceptions mirroring proj/include/blkorth/errors.hpp ------
struct Error : std::runtime_error {
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct CholeskyBreakdown : Error {
  CholeskyBreakdown(const std::string& m, std::size_t s) : Error(m), step_(s) {}
  std::size_t step() const noexcept { return step_; }
  std::size_t step_;
};
struct SingularTriangular : Error {
  SingularTriangular(const std::string& m, std::size_t i) : Error(m), index_(i) {}
  std::size_t index() const noexcept { return index_; }
  std::size_t index_;
};
struct AmbientTooSmall : Error { using Error::Error; };
struct RankDeficient : Error { using Error::Error; };
struct AllColumnsDiscarded : Error { using Error::Error; };
struct ZeroMatrix : Error { using Error::Error; };
struct InvalidScheme : Error { using Error::Error; };
struct ParseError : Error { using Error::Error; };
struct BannerError : Error { using Error::Error; };

inline void check(int rc, const bo_status& st) {
  if (rc == BO_OK) return;
  const std::string m(st.msg);
  switch (rc) {
    case BO_CHOLESKY_BREAKDOWN: throw CholeskyBreakdown(m, (std::size_t)st.index);
    case BO_SINGULAR_TRIANGULAR: throw SingularTriangular(m, (std::size_t)st.index);
    case BO_AMBIENT_TOO_SMALL: throw AmbientTooSmall(m);
    case BO_ALL_COLUMNS_DISCARDED: throw AllColumnsDiscarded(m);
    case BO_RANK_DEFICIENT: throw RankDeficient(m);
    case BO_ZERO_MATRIX: throw ZeroMatrix(m);
    case BO_INVALID: throw InvalidScheme(m);
    case BO_PARSE_ERROR: throw ParseError(m);
    case BO_BANNER_ERROR: throw BannerError(m);
    default: throw DeviceError(m);
  }
}

// ReduceLedger (dense.hpp:97-119)
enum class ReducePhase : int { projection = 0, gram = 1, sketch = 2, norm = 3 };
struct ReduceLedger {
  std::array<uint64_t, 4> counts{};
  void record(ReducePhase p) { ++counts[(int)p]; }
  uint64_t count(ReducePhase p) const { return counts[(int)p]; }
  uint64_t total() const { return counts[0] + counts[1] + counts[2] + counts[3]; }
};
#endif

// The C ABI counts ledger events in a uint64_t[4]; LedgerIO lends one to a call
// and records the events it added into the caller's ReduceLedger.
class LedgerIO {
 public:
  explicit LedgerIO(ReduceLedger& l) : l_(l) {
    for (int p = 0; p < 4; ++p) c_[p] = c0_[p] = l.count((ReducePhase)p);
  }
  ~LedgerIO() {
    for (int p = 0; p < 4; ++p)
      for (uint64_t d = c0_[p]; d < c_[p]; ++d) l_.record((ReducePhase)p);
  }
  uint64_t* data() { return c_; }

 private:
  ReduceLedger& l_;
  uint64_t c_[4], c0_[4];
};

enum class SketchKind { gaussian = BO_SKETCH_GAUSSIAN, count = BO_SKETCH_COUNT, count_gauss = BO_SKETCH_COUNT_GAUSS };
enum class IntraKind { cholqr2 = BO_INTRA_CHOLQR2, rand_cholqr = BO_INTRA_RAND_CHOLQR };
enum class PreprocKind { bcgs_pip = BO_PREPROC_PIP, rand_bcgs = BO_PREPROC_RAND_BCGS };

// a column-major device view of this rank's rows
struct DevicePanel {
  double* data = nullptr;
  uint64_t ld = 0;
  uint64_t cols = 0;
};

// small host results (column-major)
struct HostMatrix {
  uint64_t rows = 0, cols = 0;
  std::vector<double> a;
  double operator()(uint64_t i, uint64_t j) const { return a[i + j * rows]; }
};

class Context {
 public:
  // one GPU owning rows [row_begin, row_end) of an n-row problem
  Context(uint64_t n, int device = 0, int rank = 0, int world = 1, const void* nccl_id = nullptr,
          uint64_t row_begin = 0, uint64_t row_end = UINT64_MAX, void* stream = nullptr) {
    bo_status st{};
    if (row_end == UINT64_MAX) row_end = n;
    check(bo_ctx_create(device, rank, world, nccl_id, n, row_begin, row_end, stream, &h_, &st), st);
  }
  ~Context() { bo_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  bo_ctx get() const { return h_; }
  uint64_t local_rows() const { return bo_ctx_local_rows(h_); }
  uint64_t ld() const { return bo_ctx_ld(h_); }

 private:
  bo_ctx h_ = nullptr;
};

class SketchOperator {
 public:
  static SketchOperator build(Context& c, SketchKind kind, uint64_t n, uint64_t shat, uint64_t seed) {
    SketchOperator s;
    bo_status st{};
    check(bo_sketch_build(c.get(), (int)kind, n, shat, seed, &s.h_, &st), st);
    return s;
  }
  SketchOperator(SketchOperator&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  ~SketchOperator() { bo_sketch_destroy(h_); }
  uint64_t sketch_size() const { return bo_sketch_size(h_); }
  HostMatrix apply(const DevicePanel& v, ReduceLedger& ledger) const {
    HostMatrix out{sketch_size(), v.cols, std::vector<double>(sketch_size() * v.cols)};
    bo_status st{};
    check(bo_sketch_apply(h_, v.data, v.ld, v.cols, out.a.data(), LedgerIO(ledger).data(), &st), st);
    return out;
  }
  bo_sketch get() const { return h_; }

 private:
  SketchOperator() = default;
  bo_sketch h_ = nullptr;
};

struct QrResult {
  DevicePanel q;   // written into the caller's output panel
  HostMatrix r;
};

inline QrResult cholqr(Context& c, const DevicePanel& v, DevicePanel q, ReduceLedger& ledger) {
  QrResult o{q, {v.cols, v.cols, std::vector<double>(v.cols * v.cols)}};
  bo_status st{};
  check(bo_cholqr(c.get(), v.data, v.ld, v.cols, q.data, q.ld, o.r.a.data(), LedgerIO(ledger).data(), &st), st);
  return o;
}
inline QrResult cholqr2(Context& c, const DevicePanel& v, DevicePanel q, ReduceLedger& ledger) {
  QrResult o{q, {v.cols, v.cols, std::vector<double>(v.cols * v.cols)}};
  bo_status st{};
  check(bo_cholqr2(c.get(), v.data, v.ld, v.cols, q.data, q.ld, o.r.a.data(), LedgerIO(ledger).data(), &st), st);
  return o;
}
inline QrResult rand_cholqr(Context& c, const DevicePanel& v, const SketchOperator& theta, DevicePanel q,
                            ReduceLedger& ledger) {
  QrResult o{q, {v.cols, v.cols, std::vector<double>(v.cols * v.cols)}};
  bo_status st{};
  check(bo_rand_cholqr(c.get(), v.data, v.ld, v.cols, theta.get(), q.data, q.ld, o.r.a.data(), LedgerIO(ledger).data(),
                       &st),
        st);
  return o;
}

class BasisStore {
 public:
  BasisStore(Context& c, uint64_t capacity) {
    bo_status st{};
    check(bo_basis_create(c.get(), capacity, &h_, &st), st);
  }
  ~BasisStore() { bo_basis_destroy(h_); }
  BasisStore(const BasisStore&) = delete;
  uint64_t cols() const { return bo_basis_cols(h_); }
  ReduceLedger ledger() const {
    ReduceLedger l;
    uint64_t c[4];
    bo_basis_ledger(h_, c);
    for (int p = 0; p < 4; ++p)
      for (uint64_t d = 0; d < c[p]; ++d) l.record((ReducePhase)p);
    return l;
  }
  DevicePanel basis() const {
    uint64_t ld = 0;
    double* p = bo_basis_q_device(h_, &ld);
    return {p, ld, cols()};
  }
  HostMatrix r_copy() const {
    HostMatrix m{cols(), cols(), std::vector<double>(cols() * cols())};
    bo_basis_r_copy(h_, m.a.data());
    return m;
  }
  double r_entry(uint64_t i, uint64_t j) const { return bo_basis_r_entry(h_, i, j); }
  void mark_seed(uint64_t col) { bo_basis_mark_seed(h_, col); }
  std::vector<double> input_coeff_col(uint64_t k, uint64_t len) const {
    std::vector<double> v(len);
    bo_basis_input_coeff_col(h_, k, len, v.data());
    return v;
  }
  void begin_big_panel(uint64_t sketch_rows, bool overlap = false) {
    bo_basis_begin_big_panel(h_, sketch_rows, overlap);
  }
  uint64_t big_panel_lo() const { return bo_basis_big_panel_lo(h_); }
  bo_basis get() const { return h_; }

 private:
  bo_basis h_ = nullptr;
};

inline void bcgs2(BasisStore& s, const DevicePanel& v, IntraKind intra, const SketchOperator* theta = nullptr,
                  bool overlap = false) {
  bo_status st{};
  check(bo_bcgs2(s.get(), v.data, v.ld, v.cols, (int)intra, theta ? theta->get() : nullptr, overlap, &st), st);
}
inline void bcgs_pip(BasisStore& s, const DevicePanel& v, bool overlap = false) {
  bo_status st{};
  check(bo_bcgs_pip(s.get(), v.data, v.ld, v.cols, overlap, &st), st);
}
inline void rand_bcgs_preproc(BasisStore& s, const DevicePanel& v, const SketchOperator& theta, bool overlap = false) {
  bo_status st{};
  check(bo_rand_bcgs_preproc(s.get(), v.data, v.ld, v.cols, theta.get(), overlap, &st), st);
}
inline void two_stage_panel(BasisStore& s, const DevicePanel& v, PreprocKind pre, const SketchOperator* theta,
                            bool overlap = false) {
  bo_status st{};
  check(bo_two_stage_panel(s.get(), v.data, v.ld, v.cols, (int)pre, theta ? theta->get() : nullptr, overlap, &st),
        st);
}
struct TwoStageStats {
  double preproc_condition = 0.0, sketched_orth_error = 0.0;
};
inline TwoStageStats two_stage_finish(BasisStore& s, PreprocKind pre, bool reorthogonalize = true,
                                      bool record_condition = false) {
  double stats[2] = {0, 0};
  bo_status st{};
  check(bo_two_stage_finish(s.get(), (int)pre, reorthogonalize, record_condition, stats, &st), st);
  return {stats[0], stats[1]};
}

class Operator {  // CsrMatrix rows of this shard, or the matrix-free Laplacian
 public:
  static Operator laplace(Context& c, int dims, uint64_t k) {
    Operator o;
    bo_status st{};
    check(bo_op_laplace(c.get(), dims, k, &o.h_, &st), st);
    return o;
  }
  static Operator csr(Context& c, uint64_t ncols, const std::vector<int64_t>& row_ptr,
                      const std::vector<int64_t>& col, const std::vector<double>& val) {
    Operator o;
    bo_status st{};
    check(bo_op_csr(c.get(), ncols, row_ptr.data(), col.data(), val.data(), &o.h_, &st), st);
    return o;
  }
  Operator(Operator&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  ~Operator() { bo_op_destroy(h_); }
  void spmv(const double* x, double* y) const {
    bo_status st{};
    check(bo_spmv(h_, x, y, &st), st);
  }
  void mpk(const double* v0, uint64_t s, DevicePanel v) const {
    bo_status st{};
    check(bo_mpk(h_, v0, s, v.data, v.ld, &st), st);
  }
  bo_op get() const { return h_; }

 private:
  Operator() = default;
  bo_op h_ = nullptr;
};

// SolverConfig / SolveReport (gmres.hpp:26-61)
inline bo_solve_report sstep_gmres_solve(const Operator& a, const double* b, const double* x0,
                                         const bo_solver_config& cfg, double* x) {
  bo_solve_report rep{};
  bo_status st{};
  check(bo_sstep_gmres(a.get(), b, x0, &cfg, x, &rep, &st), st);
  return rep;
}

}  // namespace gpu
}  // namespace blkorth
