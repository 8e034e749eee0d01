/*
 * bo_cuda.h — C ABI of the B200-native block-orthogonalization hot path.
 *
 * This is the drop-in boundary for the reference library blkorth
 * (/root/reference/proj).  The reference has no FFI layer: its path is a set
 * of C++ free functions and classes (proj/include/blkorth/*.hpp) called by
 * sstep_gmres_solve (proj/src/gmres.cpp:270-512).  Each entry point below is
 * the C-ABI replacement of one reference interface (cited per function); the
 * C++ adapter include/blkorth_gpu.hpp re-presents them with the reference
 * signatures and exception types, and INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Matrices are column-major doubles.  Tall arguments (n rows) are DEVICE
 *    pointers to this rank's row shard [row_begin, row_end) with leading
 *    dimension ld >= round_up(n_local, 4) and ld % 4 == 0 (16-byte aligned
 *    columns for the bulk-copy engine); other layouts are accepted and
 *    re-staged on the device.  Small results go to HOST buffers.
 *  - Every function returns a bo_code and, when `st` is non-NULL, fills it;
 *    st->msg equals the reference exception what() text
 *    (proj/include/blkorth/errors.hpp:12-92).
 *  - One host thread per bo_ctx; one bo_ctx per GPU (one process per GPU).
 *  - Every reduction is deterministic (fixed CTA order); with world > 1 the
 *    partial sums are combined with one NCCL all-reduce per reference ledger
 *    event (ReduceLedger, proj/include/blkorth/dense.hpp:97-119).
 *  - There is no CPU fallback: without a usable sm_100 GPU every call fails
 *    with BO_CUDA.
 */
#ifndef BO_CUDA_H
#define BO_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BO_ABI_VERSION 1

typedef enum {
  BO_OK = 0,
  BO_CHOLESKY_BREAKDOWN = 1,     /* errors.hpp:20 CholeskyBreakdown */
  BO_SINGULAR_TRIANGULAR = 2,    /* errors.hpp:32 SingularTriangular */
  BO_AMBIENT_TOO_SMALL = 3,      /* errors.hpp:45 AmbientTooSmall */
  BO_ALL_COLUMNS_DISCARDED = 4,  /* errors.hpp:59 AllColumnsDiscarded */
  BO_RANK_DEFICIENT = 5,         /* errors.hpp:53 RankDeficient */
  BO_INVALID = 6,                /* errors.hpp:71 InvalidScheme / bad arguments */
  BO_ZERO_MATRIX = 7,            /* errors.hpp:65 ZeroMatrix */
  BO_CUDA = 8,                   /* CUDA runtime failure / no GPU */
  BO_NCCL = 9,                   /* NCCL / collective transport failure */
  BO_PARSE_ERROR = 10,           /* errors.hpp:77 ParseError (MatrixMarket) */
  BO_BANNER_ERROR = 11           /* errors.hpp:88 BannerError (MatrixMarket) */
} bo_code;

typedef struct {
  int code;          /* bo_code */
  long long index;   /* Cholesky step (1-based) or zero-diagonal index */
  double pivot;      /* offending pivot (CholeskyOutcome::failed_pivot) */
  char msg[256];     /* reference what() text */
} bo_status;

/* reduce ledger phases, ReducePhase (dense.hpp:97) */
enum { BO_LEDGER_PROJECTION = 0, BO_LEDGER_GRAM = 1, BO_LEDGER_SKETCH = 2, BO_LEDGER_NORM = 3 };
/* SketchKind (sketch.hpp:12) */
enum { BO_SKETCH_GAUSSIAN = 0, BO_SKETCH_COUNT = 1, BO_SKETCH_COUNT_GAUSS = 2 };
/* IntraKind (block_orth.hpp:119) */
enum { BO_INTRA_CHOLQR2 = 0, BO_INTRA_RAND_CHOLQR = 1 };
/* PreprocKind (block_orth.hpp:140) */
enum { BO_PREPROC_PIP = 0, BO_PREPROC_RAND_BCGS = 1 };
/* Scheme (gmres.hpp:15) */
enum {
  BO_BCGS2_CHOLQR2 = 0,
  BO_BCGS2_RANDCHOLQR = 1,
  BO_TWOSTAGE_PIP = 2,
  BO_TWOSTAGE_RANDBCGS = 3,
  BO_STANDARD_CGS2 = 4
};

typedef struct bo_ctx_s* bo_ctx;
typedef struct bo_basis_s* bo_basis;
typedef struct bo_sketch_s* bo_sketch;
typedef struct bo_op_s* bo_op;

/* ------------------------------------------------------------------ ctx -- */
int bo_abi_version(void);
/* NCCL unique id for world > 1 (rank 0 creates it, all ranks pass it in) */
int bo_nccl_id_bytes(void);
int bo_nccl_get_unique_id(void* out, bo_status* st);
/* One context per GPU.  n_global rows are split into contiguous row shards;
 * this rank owns [row_begin, row_end).  nccl_id may be NULL when world == 1.
 * stream: a cudaStream_t to run on (NULL = a private stream). */
int bo_ctx_create(int device, int rank, int world, const void* nccl_id, uint64_t n_global,
                  uint64_t row_begin, uint64_t row_end, void* stream, bo_ctx* out,
                  bo_status* st);
/* Host-provided collective transport (MPI, gloo, a serving runtime ...) in
 * place of NCCL.  All buffers are device memory of this context; each call
 * must be ordered after the work already queued on `stream` and complete
 * (or be queued on `stream`) before it returns.  Return 0 on success. */
typedef struct {
  int peer;       /* rank */
  int is_send;    /* 1 send buf to peer, 0 receive into buf from peer */
  double* buf;
  uint64_t count; /* doubles */
} bo_p2p_op;
typedef struct {
  void* user;
  /* in-place sum over all ranks of count doubles (the ledger's logical all-reduce) */
  int (*allreduce_sum_f64)(void* user, double* buf, uint64_t count, void* stream);
  /* recv[r * count + i] = send_r[i] for every rank r */
  int (*allgather_u64)(void* user, const uint64_t* send, uint64_t count, uint64_t* recv, void* stream);
  /* one group of point-to-point transfers (matrix-powers halo exchange) */
  int (*exchange_f64)(void* user, int nops, const bo_p2p_op* ops, void* stream);
} bo_comm_ops;
/* as bo_ctx_create, with collectives through `comm` (copied) instead of NCCL */
int bo_ctx_create_comm(int device, int rank, int world, const bo_comm_ops* comm, uint64_t n_global,
                       uint64_t row_begin, uint64_t row_end, void* stream, bo_ctx* out, bo_status* st);
int bo_ctx_destroy(bo_ctx ctx);
int bo_ctx_synchronize(bo_ctx ctx, bo_status* st);
uint64_t bo_ctx_local_rows(bo_ctx ctx);
/* leading dimension the library uses for its own tall buffers */
uint64_t bo_ctx_ld(bo_ctx ctx);
/* number of device kernels this context has launched (instrumentation) */
uint64_t bo_ctx_kernel_launches(bo_ctx ctx);
/* physical all-reduces issued (world > 1) */
uint64_t bo_ctx_allreduces(bo_ctx ctx);
/* Per-launch profiling of the streaming passes with CUDA events on the ctx
 * stream (bench.py roofline).  enable != 0 clears and starts recording. */
typedef struct {
  int kind;          /* pass kind id (bo_pass_kind_name) */
  int k, p, mh;      /* panel width, projection columns, sketch rows */
  uint64_t rows;     /* local rows streamed */
  uint64_t bytes;    /* HBM bytes the pass must move (reads + writes) */
  float ms;          /* device time of the launch */
} bo_prof_record;
int bo_ctx_profile(bo_ctx ctx, int enable);
int bo_ctx_profile_read(bo_ctx ctx, bo_prof_record* out, int max, int* count, bo_status* st);
const char* bo_pass_kind_name(int kind);

/* -------------------------------------------------------------- sketch -- */
/* SketchOperator::build (sketch.hpp:28, sketch.cpp:66-99).  The Count
 * (bucket, sign) stream is bit-identical to the reference's mt19937_64 draws
 * for the same seed; it is regenerated on the GPU with MT19937-64 jump-ahead
 * (each rank generates only its rows). */
int bo_sketch_build(bo_ctx ctx, int kind, uint64_t n, uint64_t shat, uint64_t seed,
                    bo_sketch* out, bo_status* st);
/* SketchOperator::from_dense (sketch.hpp:31): theta is this rank's row shard
 * (device, n_local x mhat, ld) */
int bo_sketch_from_dense(bo_ctx ctx, const double* theta, uint64_t ld, uint64_t mhat,
                         bo_sketch* out, bo_status* st);
int bo_sketch_destroy(bo_sketch sk);
uint64_t bo_sketch_size(bo_sketch sk);        /* sketch_size() */
uint64_t bo_sketch_count_width(bo_sketch sk); /* count stage width (count / count_gauss) */
int bo_sketch_kind(bo_sketch sk);
/* local rows of the dense Gaussian stage to host (n_local x mhat, ld n_local) */
int bo_sketch_dense_to_host(bo_sketch sk, double* out, bo_status* st);
/* local rows of the count stage: bucket and +-1 sign per row */
int bo_sketch_count_to_host(bo_sketch sk, uint32_t* buckets, double* signs, bo_status* st);
/* count_gauss dense stage (mc x mhat) to host */
int bo_sketch_gauss_stage_to_host(bo_sketch sk, double* out, bo_status* st);
/* SketchOperator::apply (sketch.cpp:110-126): out = Theta^T V (host, mhat x k).
 * ledger (may be NULL) gets +1 sketch. */
int bo_sketch_apply(bo_sketch sk, const double* v, uint64_t ldv, uint64_t k, double* out,
                    uint64_t ledger[4], bo_status* st);

/* ---------------------------------------------------------- intra-orth -- */
/* cholqr / cholqr2 / rand_cholqr (intra_orth.hpp:19-28).  q: device n_local x k
 * (may alias v), r: host k x k column-major upper.  ledger may be NULL. */
int bo_cholqr(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, double* q, uint64_t ldq,
              double* r, uint64_t ledger[4], bo_status* st);
int bo_cholqr2(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, double* q, uint64_t ldq,
               double* r, uint64_t ledger[4], bo_status* st);
int bo_rand_cholqr(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, bo_sketch theta,
                   double* q, uint64_t ldq, double* r, uint64_t ledger[4], bo_status* st);
/* recursive_cholqr (intra_orth.hpp:50): q device n_local x kept; coeffs host
 * k x k (rows >= kept zero); kept/discarded host index arrays (length >= k). */
int bo_recursive_cholqr(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, double* q,
                        uint64_t ldq, double* coeffs, uint64_t* kept, uint64_t* nkept,
                        uint64_t* discarded, double* discard_norm, uint64_t* ndiscarded,
                        uint64_t* depth, uint64_t ledger[4], bo_status* st);
/* gram (dense.cpp:10): g host k x k ; apply_inv_upper (dense.cpp:166) */
int bo_gram(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, double* g,
            uint64_t ledger[4], bo_status* st);
int bo_apply_inv_upper(bo_ctx ctx, const double* v, uint64_t ldv, uint64_t k, const double* r,
                       double* x, uint64_t ldx, bo_status* st);

/* --------------------------------------------------------- block-orth -- */
/* BasisStore(n, capacity) (block_orth.hpp:27-102): device Q slab + host R/C */
int bo_basis_create(bo_ctx ctx, uint64_t capacity, bo_basis* out, bo_status* st);
/* The context keeps the largest destroyed slab (and one pinned snapshot area)
 * for the next store it creates, as a GMRES solve creates an (m+1)-column
 * store per call; they are freed with the context. */
int bo_basis_destroy(bo_basis b);
int bo_basis_reset(bo_basis b); /* back to an empty store, ledger zeroed */
uint64_t bo_basis_cols(bo_basis b);
uint64_t bo_basis_capacity(bo_basis b);
/* device pointer to the Q slab (n_local x capacity, ld) */
double* bo_basis_q_device(bo_basis b, uint64_t* ld);
int bo_basis_ledger(bo_basis b, uint64_t out[4]);
/* r_copy(): cols x cols (host, column-major) ; c: seed-coefficient matrix */
int bo_basis_r_copy(bo_basis b, double* out);
double bo_basis_r_entry(bo_basis b, uint64_t i, uint64_t j);
int bo_basis_c_copy(bo_basis b, double* out);
int bo_basis_mark_seed(bo_basis b, uint64_t col);
int bo_basis_is_seed(bo_basis b, uint64_t col);
int bo_basis_input_coeff_col(bo_basis b, uint64_t k, uint64_t len, double* out);
int bo_basis_begin_big_panel(bo_basis b, uint64_t sketch_rows, int overlap);
uint64_t bo_basis_big_panel_lo(bo_basis b);
uint64_t bo_basis_num_boundaries(bo_basis b);
int bo_basis_boundaries(bo_basis b, uint64_t* out);
/* sketched history of the current big panel (rows x cols, host) */
uint64_t bo_basis_sketched(bo_basis b, double* out, uint64_t* rows);
/* local rows of basis columns [lo, hi) to host (n_local x (hi-lo)) */
int bo_basis_cols_to_host(bo_basis b, uint64_t lo, uint64_t hi, double* out, bo_status* st);
/* the arguments of the store's last push_panel (block_orth.cpp:76-98): base
 * (= p), k, overlap, proj (base x k, ld base) and diag (k x k upper, ld k), so
 * a host BasisStore can replay the push with the reference's own arithmetic */
int bo_basis_last_push(bo_basis b, uint64_t* base, uint64_t* k, int* overlap, double* proj, double* diag);
/* load a host BasisStore's state (first cols columns of Q, this rank's rows,
 * ld ldq; R and C cols x cols column-major; seed flags; panel boundaries) so
 * device calls continue from it (the reverse of bo_basis_last_push) */
int bo_basis_import(bo_basis b, uint64_t cols, const double* q_host, uint64_t ldq, const double* r,
                    const double* c, const unsigned char* seeded, const uint64_t* bounds, uint64_t nbounds,
                    bo_status* st);

/* bcgs_project_range (block_orth.hpp:111): vhat device, coeffs host (hi-lo) x k */
int bo_bcgs_project_range(bo_basis b, const double* v, uint64_t ldv, uint64_t k, uint64_t lo,
                          uint64_t hi, double* vhat, uint64_t ldvh, double* coeffs,
                          bo_status* st);
/* bcgs2 (block_orth.hpp:123-124) — the north_star unit of work */
int bo_bcgs2(bo_basis b, const double* v, uint64_t ldv, uint64_t k, int intra, bo_sketch theta,
             int overlap, bo_status* st);
/* Deferred bcgs2: the same call enqueued on the context stream without a host
 * wait (the panel must stay valid until it has run).  Enqueue several (and
 * bo_basis_mark_seed between them), then bo_basis_sync: the calls run back to
 * back on the device, and the host bookkeeping (push_panel, mark_seed, ledger)
 * is replayed in program order up to the first failing call, whose error (the
 * text bo_bcgs2 would have returned) comes back with *failed = its index
 * among the enqueued calls.  Calls after a failure are no-ops on the device
 * and are dropped, so the store ends exactly where the synchronous API would
 * have thrown.  bo_basis_cols is the speculative count (all calls succeed);
 * every other basis accessor completes the pending calls first (an error they
 * meet is kept for the next bo_basis_sync). */
int bo_bcgs2_enqueue(bo_basis b, const double* v, uint64_t ldv, uint64_t k, int intra, bo_sketch theta,
                     int overlap, bo_status* st);
int bo_basis_sync(bo_basis b, uint64_t* failed, bo_status* st);
/* bcgs_pip (block_orth.hpp:130), rand_bcgs_preproc (:137) */
int bo_bcgs_pip(bo_basis b, const double* v, uint64_t ldv, uint64_t k, int overlap,
                bo_status* st);
int bo_rand_bcgs_preproc(bo_basis b, const double* v, uint64_t ldv, uint64_t k,
                         bo_sketch theta, int overlap, bo_status* st);
/* two_stage_panel (block_orth.hpp:157), two_stage_finish (:163).
 * stats[0] preproc condition, stats[1] sketched orth error (record != 0) */
int bo_two_stage_panel(bo_basis b, const double* v, uint64_t ldv, uint64_t k, int preproc,
                       bo_sketch theta, int overlap, bo_status* st);
int bo_two_stage_finish(bo_basis b, int preproc, int reorthogonalize, int record,
                        double* stats, bo_status* st);

/* ------------------------------------------------------------ operator -- */
/* CsrMatrix rows of this shard (sparse.hpp:16): row_ptr (n_local+1, local
 * offsets), col (global column ids) and val, host arrays. */
int bo_op_csr(bo_ctx ctx, uint64_t ncols, const int64_t* row_ptr, const int64_t* col,
              const double* val, bo_op* out, bo_status* st);
/* matrix-free 2D 5-point / 3D 7-point Laplacian on a k^dims grid
 * (problems.cpp:65-113), bit-identical to spmv on the CSR of laplace_2d/3d */
int bo_op_laplace(bo_ctx ctx, int dims, uint64_t k, bo_op* out, bo_status* st);
/* matrix-free constant-coefficient 5-point (2D) / 7-point (3D) stencil on a
 * k^dims grid; coeffs (2*dims+1) in ascending column order, 3D: (i-1, j-1,
 * l-1, self, l+1, j+1, i+1).  Bit-identical to spmv on the CSR that
 * CsrMatrix::from_triplets (sparse.cpp:13-42) builds from the same entries.
 * Config 5's nonsymmetric convection-diffusion operator (absent from the
 * reference, SURVEY finding 4) is coeffs = (-1-w, -1-w, -1-w, 6, -1+w, -1+w, -1+w). */
int bo_op_stencil(bo_ctx ctx, int dims, uint64_t k, const double* coeffs, bo_op* out, bo_status* st);
int bo_op_destroy(bo_op op);
/* MatrixMarket ingestion (sparse.cpp:88-136 read_matrix_market, :138-152
 * write_matrix_market): "matrix coordinate real general|symmetric"; the CSR
 * is what CsrMatrix::from_triplets builds (sorted, duplicates summed,
 * symmetric entries mirrored).  Errors: BO_PARSE_ERROR / BO_BANNER_ERROR with
 * the reference what() text.  Host-only: no GPU needed.  Feed the rows of a
 * shard to bo_op_csr. */
typedef struct bo_csr_host_s* bo_csr_host;
int bo_mm_read(const char* path, bo_csr_host* out, bo_status* st);
int bo_csr_host_info(bo_csr_host h, uint64_t* nrows, uint64_t* ncols, uint64_t* nnz);
int bo_csr_host_arrays(bo_csr_host h, int64_t* row_ptr, int64_t* col, double* val);
int bo_csr_host_destroy(bo_csr_host h);
int bo_mm_write(const char* path, uint64_t nrows, uint64_t ncols, const int64_t* row_ptr, const int64_t* col,
                const double* val, bo_status* st);
/* Raw FP64 panel cache for C2 inputs: a
 * 312-byte header (magic "BOPC0001", rows, cols, SHA-256 of the payload, a
 * 256-byte generator description) followed by rows x cols doubles,
 * column-major.  Write hashes the host block (ld >= rows) and writes through a
 * temporary file; read fills a host block and fails with BO_INVALID on a size
 * or digest mismatch.  Host only.  bo_sha256: the same digest of any buffer. */
int bo_panel_cache_write(const char* path, const double* a, uint64_t rows, uint64_t cols, uint64_t ld,
                         const char* desc, char sha_hex[65], bo_status* st);
int bo_panel_cache_info(const char* path, uint64_t* rows, uint64_t* cols, char sha_hex[65], char desc[256],
                        bo_status* st);
int bo_panel_cache_read(const char* path, double* a, uint64_t rows, uint64_t cols, uint64_t ld, bo_status* st);
int bo_sha256(const void* data, uint64_t len, char hex_out[65]);
/* Cost model (cost_model.hpp:9-39, cost_model.cpp:38-111): exact integer
 * per-restart-cycle flops (both orthogonalization passes), latency (global
 * reduces), volume and storage of the tabulated schemes.  shat is forced to
 * 1 / s / m for standard / sstep and sketch_eq_s / sketch_eq_m; mhat <= 0
 * selects 2(shat+1).  Errors: BO_INVALID with the reference's InvalidScheme
 * text.  Host only. */
enum { BO_COST_STANDARD = 0, BO_COST_SSTEP = 1, BO_COST_SKETCH_EQ_S = 2, BO_COST_SKETCH_BETWEEN = 3,
       BO_COST_SKETCH_EQ_M = 4 };
typedef struct {
  int64_t flops_total, flops_second, latency, volume, storage;
} bo_cost_result;
int bo_cost_eval(int scheme, int64_t n, int64_t m, int64_t s, int64_t shat, int64_t mhat, bo_cost_result* out,
                 bo_status* st);
/* gen_glued (problems.cpp:21-61): the glued test matrix n x (num_panels *
 * panel_width), bit-identical to the reference for the same arguments (the
 * config-2 input).  n must be the context's global row count;
 * the rank's rows [row_begin, row_end) go to out (device, column-major, ld
 * ldo).  Gaussian drawn on the host with glibc as rng.hpp:37-49 does; the
 * Householder QR's row-order dot products run on the device. */
int bo_gen_glued(bo_ctx ctx, uint64_t n, uint64_t num_panels, uint64_t panel_width, double kappa_panel,
                 double kappa_global, uint64_t seed, double* out, uint64_t ldo, bo_status* st);
/* spmv (sparse.cpp:51-63): y = A x (local rows; x is the local shard, halo
 * exchanged internally when world > 1) */
int bo_spmv(bo_op op, const double* x, double* y, bo_status* st);
/* mpk (gmres.cpp:48-58): V(:,0) = v0, V(:,j+1) = A V(:,j); V device n_local x (s+1) */
int bo_mpk(bo_op op, const double* v0, uint64_t s, double* v, uint64_t ldv, bo_status* st);

/* ---------------------------------------------------------- s-step GMRES -- */
typedef struct {
  uint64_t n, m, s, shat;
  int scheme, sketch;
  double rel_tol;
  uint64_t max_restarts;
  uint64_t seed;
  int reorthogonalize;
  int diagnostics; /* 1: per-restart ||I-Q^TQ|| and Arnoldi residual (cycle_diagnostics) */
} bo_solver_config;

typedef struct {
  int converged, breakdown, happy_breakdown;
  char breakdown_detail[256];
  uint64_t restarts, iterations;
  double initial_residual, final_relres;
  uint64_t reduce[4];
  uint64_t reduce_total;
  uint64_t nhist;
  double relres[256], lsq[256], orth[256], arnoldi[256];
  /* phase timings (ms, device events): sketch build, mpk, block orth, small dense
   * + x update, true residual, diagnostics */
  double t_sketch, t_mpk, t_orth, t_update, t_residual, t_diag;
  /* device time (CUDA events on the ctx stream) from the first restart
   * cycle's start to the last one's end: solver setup / teardown excluded */
  double t_cycles;
} bo_solve_report;

/* sstep_gmres_solve (gmres.hpp:92, gmres.cpp:270-512): b, x0, x device shards */
int bo_sstep_gmres(bo_op op, const double* b, const double* x0, const bo_solver_config* cfg,
                   double* x, bo_solve_report* rep, bo_status* st);

/* ------------------------------------------------------ host utilities -- */
/* MT19937-64 jump-ahead check (host only, no GPU): window g[J..J+311] of the
 * untempered stream of std::mt19937_64(seed) after its first twist. */
int bo_mt64_jump_window(uint64_t seed, uint64_t J, uint64_t* out312);

#ifdef __cplusplus
}
#endif
#endif
