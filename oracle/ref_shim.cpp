// ref_shim.cpp — C ABI over the UNMODIFIED reference library, compiled from
// its own sources under /root/reference/proj into oracle/_ref/ (see
// oracle/Makefile).  TEST INFRASTRUCTURE ONLY: used to pin the C oracle
// bit-for-bit and as the reference CPU arm of bench.py.  Signatures mirror
// oracle.h (prefix ref_ instead of orc_), so the same Python harness drives
// both.
#include <cstdio>
#include <cstring>
#include <exception>
#include <optional>
#include <string>
#include <vector>

#include "blkorth/block_orth.hpp"
#include "blkorth/cost_model.hpp"
#include "blkorth/dense.hpp"
#include "blkorth/errors.hpp"
#include "blkorth/gmres.hpp"
#include "blkorth/intra_orth.hpp"
#include "blkorth/metrics.hpp"
#include "blkorth/problems.hpp"
#include "blkorth/rng.hpp"
#include "blkorth/sketch.hpp"
#include "blkorth/sparse.hpp"

extern "C" {
#include "oracle.h"
}

using namespace blkorth;

namespace {
thread_local orc_status g_st;

int code_of(const Error& e) {
  if (dynamic_cast<const CholeskyBreakdown*>(&e)) return ORC_CHOLESKY_BREAKDOWN;
  if (dynamic_cast<const SingularTriangular*>(&e)) return ORC_SINGULAR_TRIANGULAR;
  if (dynamic_cast<const AmbientTooSmall*>(&e)) return ORC_AMBIENT_TOO_SMALL;
  if (dynamic_cast<const AllColumnsDiscarded*>(&e)) return ORC_ALL_COLUMNS_DISCARDED;
  if (dynamic_cast<const RankDeficient*>(&e)) return ORC_RANK_DEFICIENT;
  if (dynamic_cast<const ZeroMatrix*>(&e)) return ORC_ZERO_MATRIX;
  return ORC_INVALID;
}
int fail(const Error& e) {
  g_st.code = code_of(e);
  g_st.index = 0;
  if (auto* c = dynamic_cast<const CholeskyBreakdown*>(&e)) g_st.index = (long long)c->step();
  if (auto* s = dynamic_cast<const SingularTriangular*>(&e)) g_st.index = (long long)s->index();
  std::snprintf(g_st.msg, sizeof g_st.msg, "%s", e.what());
  return g_st.code;
}
void clear() {
  g_st.code = 0;
  g_st.index = 0;
  g_st.pivot = 0;
  g_st.msg[0] = 0;
}
DenseMatrix to_dense(const double* v, size_t n, size_t k) {
  DenseMatrix m(n, k);
  if (n * k) std::memcpy(m.data(), v, n * k * sizeof(double));
  return m;
}
void from_dense(const DenseMatrix& m, double* out) {
  if (m.rows() * m.cols()) std::memcpy(out, m.data(), m.rows() * m.cols() * sizeof(double));
}
void from_upper(const UpperTriangular& r, double* out) {
  const size_t k = r.dim();
  for (size_t j = 0; j < k; ++j)
    for (size_t i = 0; i < k; ++i) out[i + j * k] = r(i, j);
}
UpperTriangular to_upper(const double* r, size_t k) {
  UpperTriangular u(k);
  for (size_t i = 0; i < k; ++i)
    for (size_t j = i; j < k; ++j) u.at(i, j) = r[i + j * k];
  return u;
}
void ledger_add(const ReduceLedger& l, uint64_t* led) {
  if (!led) return;
  for (int p = 0; p < 4; ++p) led[p] += l.count(static_cast<ReducePhase>(p));
}
SketchKind kind_of(int k) {
  return k == 0 ? SketchKind::gaussian : (k == 1 ? SketchKind::count : SketchKind::count_gauss);
}
}  // namespace

extern "C" {

const orc_status* ref_last_status(void) { return &g_st; }
uint64_t ref_derive_seed(uint64_t base, uint64_t stream) { return derive_seed(base, stream); }

/* raw std::mt19937_64 + Rng transforms */
void ref_rng_draws(uint64_t seed, size_t count, uint64_t* out) {
  Rng r(seed);
  for (size_t i = 0; i < count; ++i) out[i] = r.next_u64();
}
void ref_rng_normals(uint64_t seed, size_t count, double* out) {
  Rng r(seed);
  for (size_t i = 0; i < count; ++i) out[i] = r.normal();
}

/* dense kernels */
void ref_gram(const double* v, size_t n, size_t k, double* g) {
  ReduceLedger l;
  from_dense(gram(to_dense(v, n, k), l), g);
}
size_t ref_cholesky(const double* g, size_t k, double tol, double* r, double* pivot) {
  CholeskyOutcome o = cholesky(to_dense(g, k, k), tol);
  from_upper(o.factor, r);
  if (pivot) *pivot = o.failed_pivot;
  return o.failed_at;
}
void ref_householder_qr(const double* v, size_t n, size_t k, double* q, double* r) {
  QrFactorization f = householder_qr(to_dense(v, n, k));
  from_dense(f.q, q);
  from_upper(f.r, r);
}
int ref_apply_inv_upper(const double* v, size_t n, size_t k, const double* r, double* x) {
  clear();
  try {
    from_dense(apply_inv_upper(to_dense(v, n, k), to_upper(r, k)), x);
  } catch (const Error& e) {
    return fail(e);
  }
  return 0;
}

/* sketch */
void* ref_sketch_build(int kind, size_t n, size_t shat, uint64_t seed) {
  clear();
  try {
    return new SketchOperator(SketchOperator::build(kind_of(kind), n, shat, seed));
  } catch (const Error& e) {
    fail(e);
    return nullptr;
  }
}
void ref_sketch_free(void* s) { delete static_cast<SketchOperator*>(s); }
size_t ref_sketch_size(void* s) { return static_cast<SketchOperator*>(s)->sketch_size(); }
void ref_sketch_dense(void* s, double* out, size_t* rows, size_t* cols) {
  const DenseMatrix& d = static_cast<SketchOperator*>(s)->dense_stage();
  if (rows) *rows = d.rows();
  if (cols) *cols = d.cols();
  if (out) from_dense(d, out);
}
size_t ref_sketch_count(void* s, uint32_t* bucket, double* sign) {
  const CsrMatrix& c = static_cast<SketchOperator*>(s)->count_stage();
  for (size_t i = 0; i < c.nrows(); ++i) {
    const size_t k = c.row_ptr()[i];
    if (bucket) bucket[i] = (uint32_t)c.col_idx()[k];
    if (sign) sign[i] = c.values()[k];
  }
  return c.nrows();
}
void ref_sketch_apply(void* s, const double* v, size_t n, size_t k, double* out) {
  ReduceLedger l;
  from_dense(static_cast<SketchOperator*>(s)->apply(to_dense(v, n, k), l), out);
}

/* intra-orth */
int ref_cholqr(const double* v, size_t n, size_t k, double* q, double* r, uint64_t* led) {
  clear();
  ReduceLedger l;
  try {
    QrResult o = cholqr(to_dense(v, n, k), l);
    from_dense(o.q, q);
    from_upper(o.r, r);
  } catch (const Error& e) {
    ledger_add(l, led);
    return fail(e);
  }
  ledger_add(l, led);
  return 0;
}
int ref_cholqr2(const double* v, size_t n, size_t k, double* q, double* r, uint64_t* led) {
  clear();
  ReduceLedger l;
  try {
    QrResult o = cholqr2(to_dense(v, n, k), l);
    from_dense(o.q, q);
    from_upper(o.r, r);
  } catch (const Error& e) {
    ledger_add(l, led);
    return fail(e);
  }
  ledger_add(l, led);
  return 0;
}
int ref_rand_cholqr(const double* v, size_t n, size_t k, void* th, double* q, double* r, uint64_t* led) {
  clear();
  ReduceLedger l;
  try {
    QrResult o = rand_cholqr(to_dense(v, n, k), *static_cast<SketchOperator*>(th), l);
    from_dense(o.q, q);
    from_upper(o.r, r);
  } catch (const Error& e) {
    ledger_add(l, led);
    return fail(e);
  }
  ledger_add(l, led);
  return 0;
}
int ref_recursive_cholqr(const double* v, size_t n, size_t k, double* q, double* coeffs, size_t* kept,
                         size_t* nkept, size_t* disc, double* disc_norm, size_t* ndisc, size_t* depth,
                         uint64_t* led) {
  clear();
  ReduceLedger l;
  try {
    RecursiveQr o = recursive_cholqr(to_dense(v, n, k), l);
    from_dense(o.q, q);
    std::memset(coeffs, 0, k * k * sizeof(double));
    for (size_t j = 0; j < k; ++j)
      for (size_t i = 0; i < o.coeffs.rows(); ++i) coeffs[i + j * k] = o.coeffs(i, j);
    for (size_t i = 0; i < o.kept.size(); ++i) kept[i] = o.kept[i];
    *nkept = o.kept.size();
    for (size_t i = 0; i < o.discarded.size(); ++i) {
      disc[i] = o.discarded[i];
      disc_norm[i] = o.discard_norm[i];
    }
    *ndisc = o.discarded.size();
    *depth = o.depth;
  } catch (const Error& e) {
    ledger_add(l, led);
    return fail(e);
  }
  ledger_add(l, led);
  return 0;
}

/* block-orth */
struct RefBasis {
  BasisStore s;
  RefBasis(size_t n, size_t cap) : s(n, cap) {}
};
void* ref_basis_new(size_t n, size_t cap) { return new RefBasis(n, cap); }
void ref_basis_free(void* b) { delete static_cast<RefBasis*>(b); }
size_t ref_basis_cols(void* b) { return static_cast<RefBasis*>(b)->s.cols(); }
void ref_basis_get(void* bb, double* q /* n x cols */, double* r /* cols x cols */, uint64_t* led) {
  BasisStore& s = static_cast<RefBasis*>(bb)->s;
  if (q) from_dense(s.basis_copy(), q);
  if (r) from_dense(s.r_copy(), r);
  if (led)
    for (int p = 0; p < 4; ++p) led[p] = s.ledger().count(static_cast<ReducePhase>(p));
}
void ref_basis_input_coeff_col(void* bb, size_t k, size_t len, double* out) {
  auto v = static_cast<RefBasis*>(bb)->s.input_coeff_col(k, len);
  std::memcpy(out, v.data(), len * sizeof(double));
}
void ref_basis_mark_seed(void* bb, size_t col) { static_cast<RefBasis*>(bb)->s.mark_seed(col); }
void ref_basis_begin_big_panel(void* bb, size_t rows, int overlap) {
  static_cast<RefBasis*>(bb)->s.begin_big_panel(rows, overlap != 0);
}
size_t ref_basis_big_panel_lo(void* bb) { return static_cast<RefBasis*>(bb)->s.big_panel_lo(); }
size_t ref_basis_sketched(void* bb, double* out, size_t* rows) {
  const DenseMatrix& d = static_cast<RefBasis*>(bb)->s.sketched();
  if (rows) *rows = d.rows();
  if (out) from_dense(d, out);
  return d.cols();
}
void ref_bcgs_project_range(void* bb, const double* v, size_t n, size_t k, size_t lo, size_t hi, double* vhat,
                            double* coeffs) {
  ProjectResult pr = bcgs_project_range(static_cast<RefBasis*>(bb)->s, to_dense(v, n, k), lo, hi);
  from_dense(pr.vhat, vhat);
  if (coeffs) from_dense(pr.coeffs, coeffs);
}
int ref_bcgs2(void* bb, const double* v, size_t n, size_t k, int intra, void* th, int overlap) {
  clear();
  try {
    bcgs2(static_cast<RefBasis*>(bb)->s, to_dense(v, n, k), intra == 0 ? IntraKind::cholqr2 : IntraKind::rand_cholqr,
          static_cast<SketchOperator*>(th), overlap != 0);
  } catch (const Error& e) {
    return fail(e);
  }
  return 0;
}
int ref_bcgs_pip(void* bb, const double* v, size_t n, size_t k, int overlap) {
  clear();
  try {
    bcgs_pip(static_cast<RefBasis*>(bb)->s, to_dense(v, n, k), overlap != 0);
  } catch (const Error& e) {
    return fail(e);
  }
  return 0;
}
int ref_rand_bcgs_preproc(void* bb, const double* v, size_t n, size_t k, void* th, int overlap) {
  clear();
  try {
    rand_bcgs_preproc(static_cast<RefBasis*>(bb)->s, to_dense(v, n, k), *static_cast<SketchOperator*>(th),
                      overlap != 0);
  } catch (const Error& e) {
    return fail(e);
  }
  return 0;
}
int ref_two_stage_panel(void* bb, const double* v, size_t n, size_t k, int preproc, void* th, int overlap) {
  clear();
  try {
    two_stage_panel(static_cast<RefBasis*>(bb)->s, to_dense(v, n, k),
                    preproc == 0 ? PreprocKind::bcgs_pip : PreprocKind::rand_bcgs, static_cast<SketchOperator*>(th),
                    overlap != 0);
  } catch (const Error& e) {
    return fail(e);
  }
  return 0;
}
int ref_two_stage_finish(void* bb, int preproc, int reorth, int record, double* stats) {
  clear();
  try {
    TwoStageOptions o;
    o.reorthogonalize = reorth != 0;
    o.record_condition = record != 0;
    TwoStageStats s = two_stage_finish(static_cast<RefBasis*>(bb)->s,
                                       preproc == 0 ? PreprocKind::bcgs_pip : PreprocKind::rand_bcgs, o);
    if (stats) {
      stats[0] = s.preproc_condition;
      stats[1] = s.sketched_orth_error;
    }
  } catch (const Error& e) {
    return fail(e);
  }
  return 0;
}

/* problems / sparse */
void ref_gen_glued(size_t n, size_t np, size_t w, double kp, double kg, uint64_t seed, double* v) {
  from_dense(gen_glued(n, np, w, kp, kg, seed), v);
}
struct RefCsr {
  CsrMatrix a;
};
void* ref_laplace(size_t k, int dims) { return new RefCsr{dims == 2 ? laplace_2d(k) : laplace_3d(k)}; }
void* ref_csr_from_triplets(size_t nr, size_t nc, size_t nt, const size_t* r, const size_t* c, const double* v) {
  std::vector<CsrMatrix::Triplet> t(nt);
  for (size_t i = 0; i < nt; ++i) t[i] = {r[i], c[i], v[i]};
  return new RefCsr{CsrMatrix::from_triplets(nr, nc, std::move(t))};
}
/* read_matrix_market (sparse.cpp:88-136): NULL + message on a thrown Error */
void* ref_mm_read(const char* path, char* msg, size_t msg_len) {
  try {
    return new RefCsr{read_matrix_market(path)};
  } catch (const Error& e) {
    std::snprintf(msg, msg_len, "%s", e.what());
    return nullptr;
  }
}
int ref_mm_write(const char* path, void* a, char* msg, size_t msg_len) {
  try {
    write_matrix_market(path, static_cast<RefCsr*>(a)->a);
    return 0;
  } catch (const Error& e) {
    std::snprintf(msg, msg_len, "%s", e.what());
    return 1;
  }
}
void ref_csr_free(void* a) { delete static_cast<RefCsr*>(a); }
size_t ref_csr_info(void* a, size_t* nrows, size_t* ncols) {
  const CsrMatrix& m = static_cast<RefCsr*>(a)->a;
  if (nrows) *nrows = m.nrows();
  if (ncols) *ncols = m.ncols();
  return m.nnz();
}
void ref_csr_arrays(void* a, size_t* row_ptr, size_t* col, double* val) {
  const CsrMatrix& m = static_cast<RefCsr*>(a)->a;
  std::memcpy(row_ptr, m.row_ptr().data(), (m.nrows() + 1) * sizeof(size_t));
  std::memcpy(col, m.col_idx().data(), m.nnz() * sizeof(size_t));
  std::memcpy(val, m.values().data(), m.nnz() * sizeof(double));
}
void ref_spmv(void* a, const double* x, double* y) {
  const CsrMatrix& m = static_cast<RefCsr*>(a)->a;
  auto r = spmv(m, std::span<const double>(x, m.ncols()));
  std::memcpy(y, r.data(), r.size() * sizeof(double));
}
void ref_mpk(void* a, const double* v0, size_t s, double* v) {
  const CsrMatrix& m = static_cast<RefCsr*>(a)->a;
  from_dense(mpk(m, std::span<const double>(v0, m.nrows()), s), v);
}

/* s-step GMRES: same config/report structs as the C oracle */
int ref_sstep_gmres(void* a, const double* b, const double* x0, const orc_solver_config* cfg, double* x,
                    orc_solve_report* rep) {
  clear();
  std::memset(rep, 0, sizeof *rep);
  const CsrMatrix& m = static_cast<RefCsr*>(a)->a;
  SolverConfig c;
  c.n = cfg->n;
  c.m = cfg->m;
  c.s = cfg->s;
  c.shat = cfg->shat;
  c.scheme = static_cast<Scheme>(cfg->scheme);
  c.sketch = kind_of(cfg->sketch);
  c.rel_tol = cfg->rel_tol;
  c.max_restarts = cfg->max_restarts;
  c.seed = cfg->seed;
  c.reorthogonalize = cfg->reorthogonalize != 0;
  try {
    SolveResult r = sstep_gmres_solve(m, std::span<const double>(b, m.nrows()), std::span<const double>(x0, m.nrows()), c);
    std::memcpy(x, r.x.data(), r.x.size() * sizeof(double));
    const SolveReport& s = r.report;
    rep->converged = s.converged;
    rep->breakdown = s.breakdown;
    rep->happy_breakdown = s.happy_breakdown;
    std::snprintf(rep->breakdown_detail, sizeof rep->breakdown_detail, "%s", s.breakdown_detail.c_str());
    rep->restarts = s.restarts;
    rep->iterations = s.iterations;
    rep->initial_residual = s.initial_residual;
    rep->final_relres = s.final_relres;
    rep->reduce[0] = s.reduce_projection;
    rep->reduce[1] = s.reduce_gram;
    rep->reduce[2] = s.reduce_sketch;
    rep->reduce[3] = s.reduce_norm;
    rep->reduce_total = s.reduce_total;
    rep->nhist = std::min<size_t>(s.restart_relres.size(), 256);
    for (size_t i = 0; i < rep->nhist; ++i) {
      rep->relres[i] = s.restart_relres[i];
      rep->lsq[i] = s.restart_lsq_residual[i];
      rep->orth[i] = s.restart_orth_error[i];
      rep->arnoldi[i] = s.restart_arnoldi_resid[i];
    }
  } catch (const Error& e) {
    return fail(e);
  }
  return 0;
}

// cost_model.cpp:38-111 (eval_cost): out[5] = flops_total, flops_second,
// latency, volume, storage; scheme 0..4 = standard, sstep, sketch_eq_s,
// sketch_between, sketch_eq_m
int ref_eval_cost(int scheme, int64_t n, int64_t m, int64_t s, int64_t shat, int64_t mhat, int64_t* out) {
  try {
    CostQuery q;
    q.scheme = static_cast<CostScheme>(scheme);
    q.n = n;
    q.m = m;
    q.s = s;
    q.shat = shat;
    q.mhat = mhat;
    const CostResult r = eval_cost(q);
    out[0] = r.flops_total;
    out[1] = r.flops_second;
    out[2] = r.latency;
    out[3] = r.volume;
    out[4] = r.storage;
  } catch (const Error& e) {
    return fail(e);
  }
  return 0;
}

}  // extern "C"
