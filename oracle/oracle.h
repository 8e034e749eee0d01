/*
 * oracle.h — CPU restatement of the reference block-orthogonalization path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA product
 * path in paper_2503_16717_b200/; only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product
 * path never links, loads or falls back to it.
 *
 * Every routine is a plain-C restatement of the reference algorithm in
 * /root/reference/proj (cited as file:line), with the same element-level
 * semantics: sequential row-order sums, zero-coefficient skips, true division,
 * no FMA contraction (build with -ffp-contract=off).  Its outputs are pinned
 * bit-for-bit against the reference itself compiled from its own sources into
 * oracle/_ref/ (see oracle/Makefile and tests/test_oracle_vs_ref.py) and
 * against the golden values in tests/golden/.
 *
 * Matrices are column-major doubles with leading dimension == rows.
 */
#ifndef BO_ORACLE_H
#define BO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: identical numbering to include/bo_cuda.h */
enum {
  ORC_OK = 0,
  ORC_CHOLESKY_BREAKDOWN = 1,
  ORC_SINGULAR_TRIANGULAR = 2,
  ORC_AMBIENT_TOO_SMALL = 3,
  ORC_ALL_COLUMNS_DISCARDED = 4,
  ORC_RANK_DEFICIENT = 5,
  ORC_INVALID = 6,
  ORC_ZERO_MATRIX = 7
};

typedef struct {
  int code;
  long long index;   /* failed step (1-based) / zero-diagonal index */
  double pivot;
  char msg[512];     /* == the reference exception what() text */
} orc_status;

/* last error of the calling thread */
const orc_status* orc_last_status(void);

/* ---------------- rng (proj/include/blkorth/rng.hpp) ---------------- */
uint64_t orc_derive_seed(uint64_t base, uint64_t stream);
typedef struct orc_rng orc_rng;
orc_rng* orc_rng_new(uint64_t seed);
void orc_rng_free(orc_rng* r);
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_uniform_open(orc_rng* r);
double orc_rng_normal(orc_rng* r);
uint64_t orc_rng_uniform_index(orc_rng* r, uint64_t n);
double orc_rng_sign(orc_rng* r);

/* ---------------- dense (proj/src/dense.cpp) ---------------- */
/* upper-triangular factors are passed as dense k x k column-major with the
 * strict lower part zero (storage differs from the packed UpperTriangular,
 * values are identical) */
void orc_gram(const double* v, size_t n, size_t k, double* g /* k*k */);
/* test-only: sum the tall dot products of gram / transpose_times in `chunks`
 * contiguous runs (0 / 1: the reference's sequential order) */
void orc_set_sum_chunks(size_t chunks);
void orc_transpose_times(const double* a, size_t n, size_t ca, const double* b, size_t cb,
                         double* c /* ca*cb */);
void orc_times(const double* a, size_t n, size_t ca, const double* b, size_t cb,
               double* c /* n*cb */);
void orc_subtract_product(double* b, size_t n, size_t cb, const double* q, size_t cq,
                          const double* c);
/* returns failed_at (0 = ok), failed pivot in *pivot; r is k*k upper */
size_t orc_cholesky(const double* g, size_t k, double rel_pivot_tol, double* r,
                    double* pivot);
void orc_householder_qr(const double* v, size_t n, size_t k, double* q /* n*k */,
                        double* r /* k*k */);
int orc_apply_inv_upper(const double* v, size_t n, size_t k, const double* r,
                        double* x /* n*k, may alias v */);
void orc_multiply_upper(const double* t, const double* r, size_t k, double* out);

/* ---------------- sketch (proj/src/sketch.cpp) ---------------- */
enum { ORC_SK_GAUSSIAN = 0, ORC_SK_COUNT = 1, ORC_SK_COUNT_GAUSS = 2 };
typedef struct orc_sketch orc_sketch;
orc_sketch* orc_sketch_build(int kind, size_t n, size_t shat, uint64_t seed); /* NULL + status on error */
orc_sketch* orc_sketch_from_dense(const double* theta, size_t n, size_t mhat);
void orc_sketch_free(orc_sketch* s);
size_t orc_sketch_size(const orc_sketch* s);
size_t orc_sketch_count_width(const orc_sketch* s);
int orc_sketch_kind(const orc_sketch* s);
/* dense stage: gaussian n x mhat; count_gauss mhat_count x mhat */
const double* orc_sketch_dense(const orc_sketch* s, size_t* rows, size_t* cols);
/* count stage: bucket per row and sign per row (NULL for gaussian) */
const uint32_t* orc_sketch_buckets(const orc_sketch* s);
const double* orc_sketch_signs(const orc_sketch* s);
void orc_sketch_apply(const orc_sketch* s, const double* v, size_t n, size_t k,
                      double* out /* mhat*k */);

/* ---------------- intra-orth (proj/src/intra_orth.cpp) ---------------- */
typedef uint64_t orc_ledger[4]; /* projection, gram, sketch, norm */
int orc_cholqr(const double* v, size_t n, size_t k, double* q, double* r, orc_ledger led);
int orc_cholqr2(const double* v, size_t n, size_t k, double* q, double* r, orc_ledger led);
int orc_rand_cholqr(const double* v, size_t n, size_t k, const orc_sketch* th, double* q,
                    double* r, orc_ledger led);
/* recursive CholQR; q n*kept (caller buffer n*k), coeffs kept*k (caller k*k, ld=k),
 * kept/discarded index lists, discard norms.  Returns status. */
int orc_recursive_cholqr(const double* v, size_t n, size_t k, double* q, double* coeffs,
                         size_t* kept, size_t* nkept, size_t* disc, double* disc_norm,
                         size_t* ndisc, size_t* depth, orc_ledger led);

/* ---------------- block-orth (proj/src/block_orth.cpp) ---------------- */
typedef struct orc_basis orc_basis;
orc_basis* orc_basis_new(size_t n, size_t cap);
void orc_basis_free(orc_basis* b);
size_t orc_basis_cols(const orc_basis* b);
const double* orc_basis_q(const orc_basis* b);   /* n x cap */
const double* orc_basis_r(const orc_basis* b);   /* cap x cap */
const double* orc_basis_c(const orc_basis* b);   /* cap x cap */
void orc_basis_ledger(const orc_basis* b, uint64_t out[4]);
void orc_basis_mark_seed(orc_basis* b, size_t col);
int orc_basis_is_seed(const orc_basis* b, size_t col);
void orc_basis_input_coeff_col(const orc_basis* b, size_t k, size_t len, double* out);
void orc_basis_begin_big_panel(orc_basis* b, size_t sketch_rows, int overlap);
size_t orc_basis_big_panel_lo(const orc_basis* b);
size_t orc_basis_sketched(const orc_basis* b, const double** data, size_t* rows);
size_t orc_basis_num_boundaries(const orc_basis* b);
void orc_basis_boundaries(const orc_basis* b, size_t* out);
void orc_basis_push_panel(orc_basis* b, const double* qblock, size_t k, const double* proj,
                          const double* diag, int overlap);

/* project v (n x k) against columns [lo,hi): vhat (n*k) and coeffs ((hi-lo)*k) */
void orc_bcgs_project_range(orc_basis* b, const double* v, size_t k, size_t lo, size_t hi,
                            double* vhat, double* coeffs);
enum { ORC_INTRA_CHOLQR2 = 0, ORC_INTRA_RAND_CHOLQR = 1 };
int orc_bcgs2(orc_basis* b, const double* v, size_t k, int intra, const orc_sketch* th,
              int overlap);
int orc_bcgs_pip(orc_basis* b, const double* v, size_t k, int overlap);
int orc_rand_bcgs_preproc(orc_basis* b, const double* v, size_t k, const orc_sketch* th,
                          int overlap);
enum { ORC_PRE_PIP = 0, ORC_PRE_RAND_BCGS = 1 };
int orc_two_stage_panel(orc_basis* b, const double* v, size_t k, int preproc,
                        const orc_sketch* th, int overlap);
/* stats[0] = preproc condition, stats[1] = sketched orth error (when record) */
int orc_two_stage_finish(orc_basis* b, int preproc, int reorthogonalize, int record,
                         double* stats);

/* ---------------- metrics (proj/src/metrics.cpp semantics, Eigen-free) ------- */
double orc_orthogonality_error(const double* q, size_t n, size_t k);
/* singular values descending, count min(rows, cols) */
void orc_singular_values(const double* m, size_t rows, size_t cols, double* sv);
double orc_condition_number(const double* v, size_t n, size_t k); /* NaN + status on error */

/* ---------------- sparse + problems (proj/src/sparse.cpp, problems.cpp) ------ */
typedef struct {
  size_t nrows, ncols, nnz;
  size_t* row_ptr;
  size_t* col_idx;
  double* values;
} orc_csr;
orc_csr* orc_csr_from_triplets(size_t nrows, size_t ncols, size_t nt, const size_t* rows,
                               const size_t* cols, const double* vals);
void orc_csr_free(orc_csr* a);
orc_csr* orc_laplace_2d(size_t k);
orc_csr* orc_laplace_3d(size_t k);
void orc_spmv(const orc_csr* a, const double* x, double* y);
void orc_mpk(const orc_csr* a, const double* v0, size_t s, double* v /* n*(s+1) */);
void orc_gen_glued(size_t n, size_t np, size_t w, double kp, double kg, uint64_t seed,
                   double* v /* n*np*w */);

/* ---------------- s-step GMRES (proj/src/gmres.cpp) ---------------- */
enum {
  ORC_BCGS2_CHOLQR2 = 0,
  ORC_BCGS2_RANDCHOLQR = 1,
  ORC_TWOSTAGE_PIP = 2,
  ORC_TWOSTAGE_RANDBCGS = 3,
  ORC_STANDARD_CGS2 = 4
};
typedef struct {
  size_t n, m, s, shat;
  int scheme;
  int sketch;
  double rel_tol;
  size_t max_restarts;
  uint64_t seed;
  int reorthogonalize;
  int diagnostics; /* 1 = compute orth error / arnoldi residual per restart */
} orc_solver_config;

typedef struct {
  int converged, breakdown, happy_breakdown;
  char breakdown_detail[512];
  size_t restarts, iterations;
  double initial_residual, final_relres;
  uint64_t reduce[4];
  uint64_t reduce_total;
  size_t nhist;
  double relres[256], lsq[256], orth[256], arnoldi[256];
} orc_solve_report;

int orc_sstep_gmres(const orc_csr* a, const double* b, const double* x0,
                    const orc_solver_config* cfg, double* x, orc_solve_report* rep);

/* tiny host helpers shared with the GMRES port */
int orc_solve_upper_right(const double* b, size_t p, size_t q, const double* u, double* x);
double orc_solve_lsq(const double* h, size_t p, size_t q, double gamma, double* y);

#ifdef __cplusplus
}
#endif
#endif
