/*
 * oracle.c — CPU restatement of the reference block-orthogonalization path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Never linked into the product.
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared (oracle/Makefile).
 *
 * Each function cites the reference routine it restates.  Element-level
 * semantics follow the reference exactly: sequential sums
 * in row order starting from +0.0, zero-coefficient skips, true division,
 * no FMA.
 */
#include "oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* status                                                                   */
/* ------------------------------------------------------------------------ */
static _Thread_local orc_status g_status;

const orc_status* orc_last_status(void) { return &g_status; }

static int set_status(int code, long long index, double pivot, const char* fmt, ...) {
  g_status.code = code;
  g_status.index = index;
  g_status.pivot = pivot;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_status.msg, sizeof g_status.msg, fmt, ap);
  va_end(ap);
  return code;
}
static void clear_status(void) {
  g_status.code = ORC_OK;
  g_status.index = 0;
  g_status.pivot = 0.0;
  g_status.msg[0] = 0;
}
/* errors.hpp:20-25  CholeskyBreakdown(step, context) */
static int err_cholesky(size_t step, const char* ctx) {
  return set_status(ORC_CHOLESKY_BREAKDOWN, (long long)step, 0.0,
                    "%s: nonpositive Cholesky pivot at step %zu", ctx, step);
}
/* errors.hpp:32-36 */
static int err_singular(size_t idx) {
  return set_status(ORC_SINGULAR_TRIANGULAR, (long long)idx, 0.0,
                    "triangular factor is singular: zero diagonal at index %zu", idx);
}

static double* dalloc(size_t n) {
  double* p = (double*)calloc(n ? n : 1, sizeof(double));
  if (!p) abort();
  return p;
}
static double* ddup(const double* s, size_t n) {
  double* p = dalloc(n);
  if (n) memcpy(p, s, n * sizeof(double));
  return p;
}
#define AT(m, ld, i, j) ((m)[(size_t)(i) + (size_t)(j) * (size_t)(ld)])

/* ------------------------------------------------------------------------ */
/* rng — proj/include/blkorth/rng.hpp:12-64                                 */
/* ------------------------------------------------------------------------ */
/* rng.hpp:12-17 splitmix64 */
uint64_t orc_derive_seed(uint64_t base, uint64_t stream) {
  uint64_t z = base + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* std::mt19937_64 (ISO C++ [rand.eng.mers], parameters of mt19937_64) */
#define MT_N 312
#define MT_M 156
struct orc_rng {
  uint64_t mt[MT_N];
  size_t idx;
  int have_spare;
  double spare;
};

static void mt_seed(struct orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (size_t i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + i;
  r->idx = MT_N;
}
static void mt_twist(struct orc_rng* r) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  for (size_t i = 0; i < MT_N; ++i) {
    uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % MT_N] & LM);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->idx = 0;
}
static uint64_t mt_next(struct orc_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

orc_rng* orc_rng_new(uint64_t seed) {
  orc_rng* r = (orc_rng*)calloc(1, sizeof *r);
  mt_seed(r, seed);
  return r;
}
void orc_rng_free(orc_rng* r) { free(r); }
uint64_t orc_rng_next_u64(orc_rng* r) { return mt_next(r); }
/* rng.hpp:29 */
double orc_rng_uniform(orc_rng* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:32-34 */
double orc_rng_uniform_open(orc_rng* r) {
  return ((double)(mt_next(r) >> 11) + 1.0) * 0x1.0p-53;
}
/* rng.hpp:37-49 Box-Muller with a cached spare */
double orc_rng_normal(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  const double u1 = orc_rng_uniform_open(r);
  const double u2 = orc_rng_uniform(r);
  const double rr = sqrt(-2.0 * log(u1));
  const double a = 6.283185307179586476925286766559 * u2;
  r->spare = rr * sin(a);
  r->have_spare = 1;
  return rr * cos(a);
}
/* rng.hpp:52-55 multiply-shift */
uint64_t orc_rng_uniform_index(orc_rng* r, uint64_t n) {
  unsigned __int128 wide = (unsigned __int128)mt_next(r) * n;
  return (uint64_t)(wide >> 64);
}
/* rng.hpp:58 */
double orc_rng_sign(orc_rng* r) { return (mt_next(r) & 1ULL) ? 1.0 : -1.0; }

/* ------------------------------------------------------------------------ */
/* dense — proj/src/dense.cpp                                               */
/* ------------------------------------------------------------------------ */
/* Tall dot products of gram / transpose_times.  Chunks 0 or 1 (the default)
 * is the reference's sequential row sum, exactly.  Chunks c > 1 is a
 * TEST-ONLY perturbation (orc_set_sum_chunks): rows split into c contiguous
 * runs, each summed in order, the run sums added in order -- the same
 * algorithm with another summation order, whose effect on an output measures
 * the reference's own sensitivity to reordering, the yardstick
 * for the GPU's tree-ordered sums. */
static size_t g_sum_chunks = 0;
void orc_set_sum_chunks(size_t chunks) { g_sum_chunks = chunks; }
static double tall_dot(const double* a, const double* b, size_t n) {
  if (g_sum_chunks <= 1) {
    double s = 0.0;
    for (size_t r = 0; r < n; ++r) s += a[r] * b[r];
    return s;
  }
  double tot = 0.0;
  for (size_t q = 0; q < g_sum_chunks; ++q) {
    const size_t lo = n * q / g_sum_chunks, hi = n * (q + 1) / g_sum_chunks;
    double s = 0.0;
    for (size_t r = lo; r < hi; ++r) s += a[r] * b[r];
    tot += s;
  }
  return tot;
}

/* dense.cpp:10-26 (ledger recorded by callers) */
void orc_gram(const double* v, size_t n, size_t k, double* g) {
  for (size_t j = 0; j < k; ++j)
    for (size_t i = 0; i <= j; ++i) {
      const double s = tall_dot(v + i * n, v + j * n, n);
      AT(g, k, i, j) = s;
      AT(g, k, j, i) = s;
    }
}
static void gram_led(const double* v, size_t n, size_t k, double* g, orc_ledger led) {
  orc_gram(v, n, k, g);
  led[1]++;
}

/* dense.cpp:28-42 */
void orc_transpose_times(const double* a, size_t n, size_t ca, const double* b, size_t cb,
                         double* c) {
  for (size_t j = 0; j < cb; ++j) {
    const double* bj = b + j * n;
    for (size_t i = 0; i < ca; ++i) AT(c, ca, i, j) = tall_dot(a + i * n, bj, n);
  }
}

/* dense.cpp:44-58 ; c must be zero-initialised by the caller semantics: here we zero */
void orc_times(const double* a, size_t n, size_t ca, const double* b, size_t cb, double* c) {
  memset(c, 0, n * cb * sizeof(double));
  for (size_t j = 0; j < cb; ++j) {
    double* cj = c + j * n;
    for (size_t k = 0; k < ca; ++k) {
      const double bkj = AT(b, ca, k, j);
      if (bkj == 0.0) continue;
      const double* ak = a + k * n;
      for (size_t r = 0; r < n; ++r) cj[r] += ak[r] * bkj;
    }
  }
}

/* dense.cpp:60-73 */
void orc_subtract_product(double* b, size_t n, size_t cb, const double* q, size_t cq,
                          const double* c) {
  for (size_t j = 0; j < cb; ++j) {
    double* bj = b + j * n;
    for (size_t k = 0; k < cq; ++k) {
      const double ckj = AT(c, cq, k, j);
      if (ckj == 0.0) continue;
      const double* qk = q + k * n;
      for (size_t r = 0; r < n; ++r) bj[r] -= qk[r] * ckj;
    }
  }
}

/* dense.cpp:75-102 (up-looking order; pivot floor = tol * max diag) */
size_t orc_cholesky(const double* g, size_t k, double rel_pivot_tol, double* r,
                    double* pivot_out) {
  memset(r, 0, k * k * sizeof(double));
  double max_diag = 0.0;
  for (size_t i = 0; i < k; ++i) {
    const double d = AT(g, k, i, i);
    max_diag = max_diag < d ? d : max_diag; /* std::max(max_diag, d) */
  }
  const double pivot_floor = rel_pivot_tol * max_diag;
  for (size_t j = 0; j < k; ++j) {
    for (size_t i = 0; i < j; ++i) {
      double s = AT(g, k, i, j);
      for (size_t t = 0; t < i; ++t) s -= AT(r, k, t, i) * AT(r, k, t, j);
      AT(r, k, i, j) = s / AT(r, k, i, i);
    }
    double pivot = AT(g, k, j, j);
    for (size_t t = 0; t < j; ++t) pivot -= AT(r, k, t, j) * AT(r, k, t, j);
    if (pivot <= pivot_floor) {
      if (pivot_out) *pivot_out = pivot;
      return j + 1;
    }
    AT(r, k, j, j) = sqrt(pivot);
  }
  if (pivot_out) *pivot_out = 0.0;
  return 0;
}
#define ORC_DEFAULT_PIVOT_TOL 2.220446049250313e-16

/* dense.cpp:104-164 thin Householder QR, sign-normalised R */
void orc_householder_qr(const double* v, size_t n, size_t k, double* qout, double* rout) {
  double* a = ddup(v, n * k);
  double* w = dalloc(n * k);
  double* tau = dalloc(k);
  for (size_t j = 0; j < k; ++j) {
    double norm2 = 0.0;
    for (size_t i = j; i < n; ++i) norm2 += AT(a, n, i, j) * AT(a, n, i, j);
    const double norm = sqrt(norm2);
    if (norm == 0.0) {
      tau[j] = 0.0;
      continue;
    }
    const double alpha = AT(a, n, j, j) >= 0.0 ? -norm : norm;
    const double v0 = AT(a, n, j, j) - alpha;
    AT(w, n, j, j) = 1.0;
    for (size_t i = j + 1; i < n; ++i) AT(w, n, i, j) = AT(a, n, i, j) / v0;
    tau[j] = -v0 / alpha;
    AT(a, n, j, j) = alpha;
    for (size_t i = j + 1; i < n; ++i) AT(a, n, i, j) = 0.0;
    for (size_t c = j + 1; c < k; ++c) {
      double s = AT(a, n, j, c);
      for (size_t i = j + 1; i < n; ++i) s += AT(w, n, i, j) * AT(a, n, i, c);
      s *= tau[j];
      AT(a, n, j, c) -= s;
      for (size_t i = j + 1; i < n; ++i) AT(a, n, i, c) -= s * AT(w, n, i, j);
    }
  }
  double* q = dalloc(n * k);
  for (size_t j = 0; j < k; ++j) AT(q, n, j, j) = 1.0;
  for (size_t jj = k; jj-- > 0;) {
    if (tau[jj] == 0.0) continue;
    for (size_t c = jj; c < k; ++c) {
      double s = AT(q, n, jj, c);
      for (size_t i = jj + 1; i < n; ++i) s += AT(w, n, i, jj) * AT(q, n, i, c);
      s *= tau[jj];
      AT(q, n, jj, c) -= s;
      for (size_t i = jj + 1; i < n; ++i) AT(q, n, i, c) -= s * AT(w, n, i, jj);
    }
  }
  memset(rout, 0, k * k * sizeof(double));
  for (size_t i = 0; i < k; ++i) {
    const double flip = AT(a, n, i, i) < 0.0 ? -1.0 : 1.0;
    for (size_t j = i; j < k; ++j) AT(rout, k, i, j) = flip * AT(a, n, i, j);
    if (flip < 0.0)
      for (size_t r = 0; r < n; ++r) AT(q, n, r, i) = -AT(q, n, r, i);
  }
  memcpy(qout, q, n * k * sizeof(double));
  free(q);
  free(a);
  free(w);
  free(tau);
}

/* dense.cpp:166-186 forward column substitution X = V R^{-1} */
int orc_apply_inv_upper(const double* v, size_t n, size_t k, const double* r, double* x) {
  for (size_t j = 0; j < k; ++j)
    if (AT(r, k, j, j) == 0.0) return err_singular(j);
  if (x != v) memcpy(x, v, n * k * sizeof(double));
  for (size_t j = 0; j < k; ++j) {
    double* xj = x + j * n;
    for (size_t i = 0; i < j; ++i) {
      const double rij = AT(r, k, i, j);
      if (rij == 0.0) continue;
      const double* xi = x + i * n;
      for (size_t t = 0; t < n; ++t) xj[t] -= rij * xi[t];
    }
    const double d = AT(r, k, j, j);
    for (size_t t = 0; t < n; ++t) xj[t] /= d;
  }
  return ORC_OK;
}

/* dense.cpp:188-198 */
void orc_multiply_upper(const double* t, const double* r, size_t k, double* out) {
  double* o = dalloc(k * k);
  for (size_t i = 0; i < k; ++i)
    for (size_t j = i; j < k; ++j) {
      double s = 0.0;
      for (size_t l = i; l <= j; ++l) s += AT(t, k, i, l) * AT(r, k, l, j);
      AT(o, k, i, j) = s;
    }
  memcpy(out, o, k * k * sizeof(double));
  free(o);
}

static double frobenius(const double* m, size_t rows, size_t cols) {
  double s = 0.0;
  for (size_t j = 0; j < cols; ++j)
    for (size_t i = 0; i < rows; ++i) s += AT(m, rows, i, j) * AT(m, rows, i, j);
  return sqrt(s);
}
static double vec_norm(const double* v, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += v[i] * v[i];
  return sqrt(s);
}

/* ------------------------------------------------------------------------ */
/* sketch — proj/src/sketch.cpp                                             */
/* ------------------------------------------------------------------------ */
struct orc_sketch {
  int kind;
  size_t n, mhat, mhat_count;
  double* dense; /* gaussian n x mhat ; count_gauss mhat_count x mhat */
  size_t dense_rows, dense_cols;
  uint32_t* bucket; /* count stage, one entry per row */
  double* sign;
};

/* sketch.cpp:30-35 */
static double* gaussian_matrix(size_t rows, size_t cols, double scale, orc_rng* rng) {
  double* m = dalloc(rows * cols);
  for (size_t j = 0; j < cols; ++j)
    for (size_t i = 0; i < rows; ++i) AT(m, rows, i, j) = scale * orc_rng_normal(rng);
  return m;
}
/* sketch.cpp:37-45 (one +-1 per row; CSR row order == row order) */
static void count_matrix(size_t n, size_t width, orc_rng* rng, uint32_t* bucket, double* sign) {
  for (size_t i = 0; i < n; ++i) {
    const uint64_t c = orc_rng_uniform_index(rng, width);
    bucket[i] = (uint32_t)c;
    sign[i] = orc_rng_sign(rng);
  }
}
/* sketch.cpp:48-62 */
static void count_apply_transposed(const uint32_t* bucket, const double* sign, size_t width,
                                   const double* v, size_t n, size_t k, double* out) {
  memset(out, 0, width * k * sizeof(double));
  for (size_t i = 0; i < n; ++i) {
    const size_t r = bucket[i];
    const double s = sign[i];
    for (size_t c = 0; c < k; ++c) AT(out, width, r, c) += s * AT(v, n, i, c);
  }
}

/* sketch.cpp:66-99 */
orc_sketch* orc_sketch_build(int kind, size_t n, size_t shat, uint64_t seed) {
  clear_status();
  const size_t cols = shat + 1;
  orc_sketch* op = (orc_sketch*)calloc(1, sizeof *op);
  op->kind = kind;
  op->n = n;
  orc_rng* rng = orc_rng_new(orc_derive_seed(seed, 0));
  switch (kind) {
    case ORC_SK_GAUSSIAN:
      op->mhat = 2 * cols;
      if (n <= op->mhat) goto too_small;
      op->dense = gaussian_matrix(n, op->mhat, 1.0 / sqrt((double)op->mhat), rng);
      op->dense_rows = n;
      op->dense_cols = op->mhat;
      break;
    case ORC_SK_COUNT:
      op->mhat = 2 * cols * cols;
      if (n <= op->mhat) goto too_small;
      op->bucket = (uint32_t*)malloc(n * sizeof(uint32_t));
      op->sign = dalloc(n);
      count_matrix(n, op->mhat, rng, op->bucket, op->sign);
      break;
    case ORC_SK_COUNT_GAUSS: {
      op->mhat_count = 2 * cols * cols;
      op->mhat = 2 * cols;
      if (n <= op->mhat_count) {
        op->mhat = op->mhat_count; /* AmbientTooSmall(n, mhat_count) */
        goto too_small;
      }
      op->bucket = (uint32_t*)malloc(n * sizeof(uint32_t));
      op->sign = dalloc(n);
      count_matrix(n, op->mhat_count, rng, op->bucket, op->sign);
      orc_rng* rg = orc_rng_new(orc_derive_seed(seed, 1));
      op->dense = gaussian_matrix(op->mhat_count, op->mhat, 1.0 / sqrt((double)op->mhat), rg);
      op->dense_rows = op->mhat_count;
      op->dense_cols = op->mhat;
      orc_rng_free(rg);
      break;
    }
    default:
      orc_rng_free(rng);
      free(op);
      set_status(ORC_INVALID, 0, 0.0, "unknown sketch kind");
      return NULL;
  }
  orc_rng_free(rng);
  return op;
too_small:
  /* errors.hpp:45-49 AmbientTooSmall */
  set_status(ORC_AMBIENT_TOO_SMALL, 0, 0.0,
             "ambient dimension n=%zu must exceed sketch size mhat=%zu", n, op->mhat);
  orc_rng_free(rng);
  free(op);
  return NULL;
}

/* sketch.cpp:101-108 */
orc_sketch* orc_sketch_from_dense(const double* theta, size_t n, size_t mhat) {
  orc_sketch* op = (orc_sketch*)calloc(1, sizeof *op);
  op->kind = ORC_SK_GAUSSIAN;
  op->n = n;
  op->mhat = mhat;
  op->dense = ddup(theta, n * mhat);
  op->dense_rows = n;
  op->dense_cols = mhat;
  return op;
}
void orc_sketch_free(orc_sketch* s) {
  if (!s) return;
  free(s->dense);
  free(s->bucket);
  free(s->sign);
  free(s);
}
size_t orc_sketch_size(const orc_sketch* s) { return s->mhat; }
size_t orc_sketch_count_width(const orc_sketch* s) {
  return s->kind == ORC_SK_COUNT ? s->mhat : s->mhat_count;
}
int orc_sketch_kind(const orc_sketch* s) { return s->kind; }
const double* orc_sketch_dense(const orc_sketch* s, size_t* rows, size_t* cols) {
  if (rows) *rows = s->dense_rows;
  if (cols) *cols = s->dense_cols;
  return s->dense;
}
const uint32_t* orc_sketch_buckets(const orc_sketch* s) { return s->bucket; }
const double* orc_sketch_signs(const orc_sketch* s) { return s->sign; }

/* sketch.cpp:110-126 (ledger recorded by the caller) */
void orc_sketch_apply(const orc_sketch* s, const double* v, size_t n, size_t k, double* out) {
  switch (s->kind) {
    case ORC_SK_GAUSSIAN:
      orc_transpose_times(s->dense, n, s->mhat, v, k, out);
      break;
    case ORC_SK_COUNT:
      count_apply_transposed(s->bucket, s->sign, s->mhat, v, n, k, out);
      break;
    case ORC_SK_COUNT_GAUSS: {
      double* tmp = dalloc(s->mhat_count * k);
      count_apply_transposed(s->bucket, s->sign, s->mhat_count, v, n, k, tmp);
      orc_transpose_times(s->dense, s->mhat_count, s->mhat, tmp, k, out);
      free(tmp);
      break;
    }
  }
}
static void sketch_apply_led(const orc_sketch* s, const double* v, size_t n, size_t k,
                             double* out, orc_ledger led) {
  orc_sketch_apply(s, v, n, k, out);
  led[2]++;
}

/* ------------------------------------------------------------------------ */
/* intra-orth — proj/src/intra_orth.cpp                                     */
/* ------------------------------------------------------------------------ */
/* intra_orth.cpp:11-19 ; q may alias nothing; r k*k */
int orc_cholqr(const double* v, size_t n, size_t k, double* q, double* r, orc_ledger led) {
  clear_status();
  double* g = dalloc(k * k);
  gram_led(v, n, k, g, led);
  double piv;
  const size_t f = orc_cholesky(g, k, ORC_DEFAULT_PIVOT_TOL, r, &piv);
  free(g);
  if (f) {
    err_cholesky(f, "cholqr");
    g_status.pivot = piv;
    return ORC_CHOLESKY_BREAKDOWN;
  }
  return orc_apply_inv_upper(v, n, k, r, q);
}

/* intra_orth.cpp:21-26 */
int orc_cholqr2(const double* v, size_t n, size_t k, double* q, double* r, orc_ledger led) {
  double* q1 = dalloc(n * k);
  double* r1 = dalloc(k * k);
  int st = orc_cholqr(v, n, k, q1, r1, led);
  if (st == ORC_OK) {
    double* r2 = dalloc(k * k);
    st = orc_cholqr(q1, n, k, q, r2, led);
    if (st == ORC_OK) orc_multiply_upper(r2, r1, k, r);
    free(r2);
  }
  free(q1);
  free(r1);
  return st;
}

/* intra_orth.cpp:28-39 */
int orc_rand_cholqr(const double* v, size_t n, size_t k, const orc_sketch* th, double* q,
                    double* r, orc_ledger led) {
  clear_status();
  const size_t mh = th->mhat;
  double* sk = dalloc(mh * k);
  sketch_apply_led(th, v, n, k, sk, led);
  double* sq = dalloc(mh * k);
  double* rs = dalloc(k * k);
  orc_householder_qr(sk, mh, k, sq, rs);
  double* pre = dalloc(n * k);
  int st = orc_apply_inv_upper(v, n, k, rs, pre);
  if (st == ORC_OK) {
    double* rc = dalloc(k * k);
    st = orc_cholqr(pre, n, k, q, rc, led);
    if (st == ORC_OK) orc_multiply_upper(rc, rs, k, r);
    free(rc);
  }
  free(sk);
  free(sq);
  free(rs);
  free(pre);
  return st;
}

/* intra_orth.cpp:43-139 recursive CholQR */
typedef struct {
  size_t n, k;
  double* q;      /* n x k capacity */
  size_t nq;      /* kept columns so far */
  double* coeffs; /* k x k (acc.coeffs) */
  size_t* kept;
  size_t nkept;
  size_t* disc;
  double* disc_norm;
  size_t ndisc;
  size_t depth;
} rec_acc;

static int rec_impl(const double* v, size_t n, size_t w, const size_t* col_ids, orc_ledger led,
                    rec_acc* acc) {
  if (w == 0) return ORC_OK;
  const size_t K = acc->k;
  double* g = dalloc(w * w);
  gram_led(v, n, w, g, led);
  double* r = dalloc(w * w);
  double piv;
  const size_t f = orc_cholesky(g, w, ORC_DEFAULT_PIVOT_TOL, r, &piv);
  int st = ORC_OK;
  if (f == 0) {
    double* q = dalloc(n * w);
    st = orc_apply_inv_upper(v, n, w, r, q);
    if (st == ORC_OK) {
      const size_t base = acc->nkept;
      for (size_t j = 0; j < w; ++j) {
        acc->kept[acc->nkept++] = col_ids[j];
        for (size_t i = 0; i <= j; ++i) AT(acc->coeffs, K, base + i, col_ids[j]) = AT(r, w, i, j);
      }
      memcpy(acc->q + acc->nq * n, q, n * w * sizeof(double));
      acc->nq += w;
    }
    free(q);
    free(g);
    free(r);
    return st;
  }
  if (f == 1) {
    for (size_t j = 0; j < w; ++j) {
      acc->disc[acc->ndisc] = col_ids[j];
      const double d = AT(g, w, j, j);
      acc->disc_norm[acc->ndisc] = sqrt(d > 0.0 ? d : 0.0); /* sqrt(max(g,0)) */
      acc->ndisc++;
    }
    acc->depth++;
    free(g);
    free(r);
    return ORC_OK;
  }
  const size_t good = f - 1;
  double* r11 = dalloc(good * good);
  for (size_t i = 0; i < good; ++i)
    for (size_t j = i; j < good; ++j) AT(r11, good, i, j) = AT(r, w, i, j);
  double* q_good = dalloc(n * good);
  st = orc_apply_inv_upper(v, n, good, r11, q_good); /* v_good = first `good` columns */
  if (st != ORC_OK) {
    free(r11);
    free(q_good);
    free(g);
    free(r);
    return st;
  }
  const size_t base = acc->nkept;
  for (size_t j = 0; j < good; ++j) {
    acc->kept[acc->nkept++] = col_ids[j];
    for (size_t i = 0; i <= j; ++i) AT(acc->coeffs, K, base + i, col_ids[j]) = AT(r, w, i, j);
  }
  memcpy(acc->q + acc->nq * n, q_good, n * good * sizeof(double));
  acc->nq += good;

  const size_t wr = w - good;
  double* rest = ddup(v + good * n, n * wr);
  double* r12 = dalloc(good * wr);
  for (size_t j = 0; j < wr; ++j)
    for (size_t i = 0; i < good; ++i) {
      const double c = AT(r, w, i, good + j);
      AT(r12, good, i, j) = c;
      AT(acc->coeffs, K, base + i, col_ids[good + j]) = c;
    }
  orc_subtract_product(rest, n, wr, q_good, good, r12);
  acc->depth++;
  st = rec_impl(rest, n, wr, col_ids + good, led, acc);
  free(rest);
  free(r12);
  free(r11);
  free(q_good);
  free(g);
  free(r);
  return st;
}

int orc_recursive_cholqr(const double* v, size_t n, size_t k, double* q, double* coeffs,
                         size_t* kept, size_t* nkept, size_t* disc, double* disc_norm,
                         size_t* ndisc, size_t* depth, orc_ledger led) {
  clear_status();
  rec_acc acc;
  memset(&acc, 0, sizeof acc);
  acc.n = n;
  acc.k = k;
  acc.q = dalloc(n * k);
  acc.coeffs = dalloc(k * k);
  acc.kept = (size_t*)calloc(k + 1, sizeof(size_t));
  acc.disc = (size_t*)calloc(k + 1, sizeof(size_t));
  acc.disc_norm = dalloc(k + 1);
  size_t* ids = (size_t*)calloc(k + 1, sizeof(size_t));
  for (size_t j = 0; j < k; ++j) ids[j] = j;
  int st = rec_impl(v, n, k, ids, led, &acc);
  if (st == ORC_OK && acc.nkept == 0)
    st = set_status(ORC_ALL_COLUMNS_DISCARDED, 0, 0.0, "recursive CholQR discarded all columns");
  if (q) memcpy(q, acc.q, n * acc.nq * sizeof(double));
  if (coeffs) memcpy(coeffs, acc.coeffs, k * k * sizeof(double));
  if (kept) memcpy(kept, acc.kept, acc.nkept * sizeof(size_t));
  if (nkept) *nkept = acc.nkept;
  if (disc) memcpy(disc, acc.disc, acc.ndisc * sizeof(size_t));
  if (disc_norm) memcpy(disc_norm, acc.disc_norm, acc.ndisc * sizeof(double));
  if (ndisc) *ndisc = acc.ndisc;
  if (depth) *depth = acc.depth;
  free(acc.q);
  free(acc.coeffs);
  free(acc.kept);
  free(acc.disc);
  free(acc.disc_norm);
  free(ids);
  return st;
}

/* ------------------------------------------------------------------------ */
/* metrics — proj/src/metrics.cpp:19-41 semantics without Eigen             */
/* ------------------------------------------------------------------------ */
#include "metrics_impl.h"

/* metrics.cpp:19-27 */
double orc_orthogonality_error(const double* q, size_t n, size_t k) {
  if (n == 0 || k == 0) return 0.0;
  double* d = dalloc(k * k);
  orc_transpose_times(q, n, k, q, k, d);
  for (size_t j = 0; j < k; ++j)
    for (size_t i = 0; i < k; ++i) AT(d, k, i, j) = (i == j ? 1.0 : 0.0) - AT(d, k, i, j);
  double* ev = dalloc(k);
  mi_sym_eigenvalues(d, k, ev);
  double m = 0.0;
  for (size_t i = 0; i < k; ++i) m = fabs(ev[i]) > m ? fabs(ev[i]) : m;
  free(d);
  free(ev);
  return m;
}

/* metrics.cpp:29-33 */
void orc_singular_values(const double* m, size_t rows, size_t cols, double* sv) {
  mi_singular_values(m, rows, cols, sv);
}

/* metrics.cpp:35-41 */
double orc_condition_number(const double* v, size_t n, size_t k) {
  const size_t m = n < k ? n : k;
  if (m == 0) {
    set_status(ORC_ZERO_MATRIX, 0, 0.0, "matrix is identically zero");
    return NAN;
  }
  double* sv = dalloc(m);
  orc_singular_values(v, n, k, sv);
  if (sv[0] == 0.0) {
    free(sv);
    set_status(ORC_ZERO_MATRIX, 0, 0.0, "matrix is identically zero");
    return NAN;
  }
  const double smin = sv[m - 1];
  const double out = smin == 0.0 ? INFINITY : sv[0] / smin;
  free(sv);
  return out;
}

/* ------------------------------------------------------------------------ */
/* BasisStore — proj/src/block_orth.cpp:10-153                              */
/* ------------------------------------------------------------------------ */
struct orc_basis {
  size_t n, cap, cols;
  double* q; /* n x cap */
  double* r; /* cap x cap */
  double* c; /* cap x cap */
  unsigned char* seeded;
  size_t* bounds;
  size_t nbounds;
  size_t bp_lo;
  double* sk; /* sk_rows x sk_cols */
  size_t sk_rows, sk_cols;
  orc_ledger led;
};

orc_basis* orc_basis_new(size_t n, size_t cap) {
  orc_basis* b = (orc_basis*)calloc(1, sizeof *b);
  b->n = n;
  b->cap = cap;
  b->q = dalloc(n * cap);
  b->r = dalloc(cap * cap);
  b->c = dalloc(cap * cap);
  b->seeded = (unsigned char*)calloc(cap + 1, 1);
  b->bounds = (size_t*)calloc(cap + 1, sizeof(size_t));
  return b;
}
void orc_basis_free(orc_basis* b) {
  if (!b) return;
  free(b->q);
  free(b->r);
  free(b->c);
  free(b->seeded);
  free(b->bounds);
  free(b->sk);
  free(b);
}
size_t orc_basis_cols(const orc_basis* b) { return b->cols; }
const double* orc_basis_q(const orc_basis* b) { return b->q; }
const double* orc_basis_r(const orc_basis* b) { return b->r; }
const double* orc_basis_c(const orc_basis* b) { return b->c; }
void orc_basis_ledger(const orc_basis* b, uint64_t out[4]) { memcpy(out, b->led, sizeof b->led); }
size_t orc_basis_num_boundaries(const orc_basis* b) { return b->nbounds; }
void orc_basis_boundaries(const orc_basis* b, size_t* out) {
  memcpy(out, b->bounds, b->nbounds * sizeof(size_t));
}

/* block_orth.cpp:40-45 */
void orc_basis_mark_seed(orc_basis* b, size_t col) {
  for (size_t i = 0; i < b->cap; ++i) AT(b->c, b->cap, i, col) = 0.0;
  AT(b->c, b->cap, col, col) = 1.0;
  b->seeded[col] = 1;
}
int orc_basis_is_seed(const orc_basis* b, size_t col) { return col < b->cap && b->seeded[col]; }
/* block_orth.cpp:47-52 */
void orc_basis_input_coeff_col(const orc_basis* b, size_t k, size_t len, double* out) {
  const double* src = orc_basis_is_seed(b, k) ? b->c : b->r;
  for (size_t i = 0; i < len; ++i) out[i] = AT(src, b->cap, i, k);
}
/* block_orth.cpp:54-57 */
void orc_basis_begin_big_panel(orc_basis* b, size_t sketch_rows, int overlap) {
  b->bp_lo = b->cols - ((overlap && b->cols > 0) ? 1 : 0);
  free(b->sk);
  b->sk = NULL;
  b->sk_rows = sketch_rows;
  b->sk_cols = 0;
}
size_t orc_basis_big_panel_lo(const orc_basis* b) { return b->bp_lo; }
size_t orc_basis_sketched(const orc_basis* b, const double** data, size_t* rows) {
  if (data) *data = b->sk;
  if (rows) *rows = b->sk_rows;
  return b->sk_cols;
}

/* block_orth.cpp:59-73 */
static void fold_overlap_column(orc_basis* b, const double* proj, size_t proj_rows,
                                const double* diag, size_t k) {
  const size_t cap = b->cap;
  const size_t k0 = b->cols - 1;
  const double scale = AT(diag, k, 0, 0);
  const double r_diag = AT(b->r, cap, k0, k0);
  for (size_t i = 0; i < k0; ++i) AT(b->r, cap, i, k0) += r_diag * AT(proj, proj_rows, i, 0);
  AT(b->r, cap, k0, k0) = r_diag * scale;
  if (orc_basis_is_seed(b, k0)) {
    const double c_diag = AT(b->c, cap, k0, k0);
    for (size_t i = 0; i < k0; ++i) AT(b->c, cap, i, k0) += c_diag * AT(proj, proj_rows, i, 0);
    AT(b->c, cap, k0, k0) = c_diag * scale;
  }
}

/* block_orth.cpp:75-98 ; proj is base x k (ld = base) */
void orc_basis_push_panel(orc_basis* b, const double* qblock, size_t k, const double* proj,
                          const double* diag, int overlap) {
  const size_t cap = b->cap, n = b->n;
  const size_t base = overlap ? b->cols - 1 : b->cols;
  if (overlap) fold_overlap_column(b, proj, base, diag, k);
  for (size_t j = 0; j < k; ++j) {
    const size_t g = base + j;
    if (!(overlap && j == 0)) {
      for (size_t i = 0; i < base; ++i) AT(b->r, cap, i, g) = AT(proj, base, i, j);
      for (size_t i = 0; i <= j; ++i) AT(b->r, cap, base + i, g) = AT(diag, k, i, j);
    }
    memcpy(b->q + g * n, qblock + j * n, n * sizeof(double));
  }
  b->bounds[b->nbounds++] = base;
  b->cols = base + k;
}

/* block_orth.cpp:100-110 */
static void push_sketched(orc_basis* b, const double* cols, size_t kc, int overlap) {
  const size_t have = b->sk_cols;
  const size_t base = (overlap && have > 0) ? have - 1 : have;
  const size_t rows = b->sk_rows;
  double* grown = dalloc(rows * (base + kc));
  if (base) memcpy(grown, b->sk, rows * base * sizeof(double));
  memcpy(grown + rows * base, cols, rows * kc * sizeof(double));
  free(b->sk);
  b->sk = grown;
  b->sk_cols = base + kc;
}

/* block_orth.cpp:112-132 */
static void refactor_update(double* m, size_t cap, size_t lo, size_t w, size_t col,
                            const double* t, double* seg) {
  for (size_t i = 0; i < w; ++i) seg[i] = AT(m, cap, lo + i, col);
  for (size_t i = 0; i < w; ++i) {
    double s = 0.0;
    for (size_t l = i; l < w; ++l) s += AT(t, w, i, l) * seg[l];
    AT(m, cap, lo + i, col) = s;
  }
}
static void refactor_block(orc_basis* b, size_t lo, const double* qnew, const double* t) {
  const size_t w = b->cols - lo, n = b->n;
  memcpy(b->q + lo * n, qnew, n * w * sizeof(double));
  double* seg = dalloc(w);
  for (size_t col = lo; col < b->cols; ++col) {
    refactor_update(b->r, b->cap, lo, w, col, t, seg);
    if (orc_basis_is_seed(b, col)) refactor_update(b->c, b->cap, lo, w, col, t, seg);
  }
  free(seg);
}
/* block_orth.cpp:134-153 ; tproj lo x w */
static void reorth_spray(double* m, size_t cap, size_t lo, size_t w, size_t col,
                         const double* tproj) {
  for (size_t i = 0; i < lo; ++i) {
    double s = 0.0;
    for (size_t l = 0; l < w; ++l) s += AT(tproj, lo, i, l) * AT(m, cap, lo + l, col);
    AT(m, cap, i, col) += s;
  }
}
static void reorthogonalize_block(orc_basis* b, size_t lo, const double* qnew,
                                  const double* tproj, const double* t) {
  const size_t w = b->cols - lo;
  for (size_t col = lo; col < b->cols; ++col) {
    reorth_spray(b->r, b->cap, lo, w, col, tproj);
    if (orc_basis_is_seed(b, col)) reorth_spray(b->c, b->cap, lo, w, col, tproj);
  }
  refactor_block(b, lo, qnew, t);
}

/* block_orth.cpp:157-171 */
void orc_bcgs_project_range(orc_basis* b, const double* v, size_t k, size_t lo, size_t hi,
                            double* vhat, double* coeffs) {
  const size_t n = b->n, p = hi - lo;
  memcpy(vhat, v, n * k * sizeof(double));
  if (p == 0) return;
  const double* qrange = b->q + lo * n; /* basis_block_copy: same values */
  orc_transpose_times(qrange, n, p, v, k, coeffs);
  b->led[0]++;
  orc_subtract_product(vhat, n, k, qrange, p, coeffs);
}

static int run_intra(const double* v, size_t n, size_t k, int intra, const orc_sketch* th,
                     double* q, double* r, orc_ledger led) {
  if (intra == ORC_INTRA_CHOLQR2) return orc_cholqr2(v, n, k, q, r, led);
  if (th == NULL)
    return set_status(ORC_INVALID, 0, 0.0,
                      "rand_cholqr intra-orthogonalization needs a sketch operator");
  return orc_rand_cholqr(v, n, k, th, q, r, led);
}

/* block_orth.cpp:191-203 proj + t * rdiag */
static void update_projection(const double* proj, const double* t, size_t p, size_t k,
                              const double* rdiag, double* out) {
  double* tmp = dalloc(p * k);
  orc_times(t, p, k, rdiag, k, tmp);
  for (size_t j = 0; j < k; ++j)
    for (size_t i = 0; i < p; ++i) AT(out, p, i, j) = AT(proj, p, i, j) + AT(tmp, p, i, j);
  free(tmp);
}

/* block_orth.cpp:207-226 */
int orc_bcgs2(orc_basis* b, const double* v, size_t k, int intra, const orc_sketch* th,
              int overlap) {
  clear_status();
  const size_t n = b->n;
  const int eff_overlap = overlap && b->cols > 0;
  const size_t hi = b->cols - (eff_overlap ? 1 : 0);
  int st;
  if (hi == 0) {
    double* q = dalloc(n * k);
    double* r = dalloc(k * k);
    st = run_intra(v, n, k, intra, th, q, r, b->led);
    if (st == ORC_OK) orc_basis_push_panel(b, q, k, NULL, r, eff_overlap);
    free(q);
    free(r);
    return st;
  }
  double* vhat = dalloc(n * k);
  double* c1 = dalloc(hi * k);
  double* qi = dalloc(n * k);
  double* ri = dalloc(k * k);
  double* zhat = dalloc(n * k);
  double* c2 = dalloc(hi * k);
  double* qo = dalloc(n * k);
  double* ro = dalloc(k * k);
  orc_bcgs_project_range(b, v, k, 0, hi, vhat, c1);
  st = run_intra(vhat, n, k, intra, th, qi, ri, b->led);
  if (st == ORC_OK) {
    orc_bcgs_project_range(b, qi, k, 0, hi, zhat, c2);
    st = orc_cholqr(zhat, n, k, qo, ro, b->led);
    if (st == ORC_OK) {
      double* coeffs = dalloc(hi * k);
      double* rjj = dalloc(k * k);
      update_projection(c1, c2, hi, k, ri, coeffs);
      orc_multiply_upper(ro, ri, k, rjj);
      orc_basis_push_panel(b, qo, k, coeffs, rjj, eff_overlap);
      free(coeffs);
      free(rjj);
    }
  }
  free(vhat);
  free(c1);
  free(qi);
  free(ri);
  free(zhat);
  free(c2);
  free(qo);
  free(ro);
  return st;
}

/* block_orth.cpp:230-269 */
static int bcgs_pip_impl(orc_basis* b, const double* vhat, size_t k, const double* rbig,
                         int overlap) {
  const size_t n = b->n, bp = b->bp_lo;
  const int eff_overlap = overlap && b->cols > 0;
  const size_t hi = b->cols - (eff_overlap ? 1 : 0);
  const size_t p = hi - bp;
  const double* qrange = b->q + bp * n;
  double* proj = dalloc(p * k);
  if (p > 0) orc_transpose_times(qrange, n, p, vhat, k, proj);
  double* g = dalloc(k * k);
  orc_transpose_times(vhat, n, k, vhat, k, g);
  b->led[1]++;
  for (size_t j = 0; j < k; ++j)
    for (size_t i = 0; i < k; ++i) {
      double s = 0.0;
      for (size_t l = 0; l < p; ++l) s += AT(proj, p, l, i) * AT(proj, p, l, j);
      AT(g, k, i, j) -= s;
    }
  double* r = dalloc(k * k);
  double piv;
  const size_t f = orc_cholesky(g, k, ORC_DEFAULT_PIVOT_TOL, r, &piv);
  int st = ORC_OK;
  if (f) {
    st = err_cholesky(f, "bcgs_pip");
    g_status.pivot = piv;
  } else {
    double* resid = ddup(vhat, n * k);
    if (p > 0) orc_subtract_product(resid, n, k, qrange, p, proj);
    double* qj = dalloc(n * k);
    st = orc_apply_inv_upper(resid, n, k, r, qj);
    if (st == ORC_OK) {
      double* full = dalloc(hi * k);
      for (size_t j = 0; j < k; ++j) {
        for (size_t i = 0; i < bp; ++i) AT(full, hi, i, j) = rbig ? AT(rbig, bp, i, j) : 0.0;
        for (size_t i = 0; i < p; ++i) AT(full, hi, bp + i, j) = AT(proj, p, i, j);
      }
      orc_basis_push_panel(b, qj, k, full, r, eff_overlap);
      free(full);
    }
    free(resid);
    free(qj);
  }
  free(proj);
  free(g);
  free(r);
  return st;
}

/* block_orth.cpp:271-325 */
static int rand_bcgs_impl(orc_basis* b, const double* vhat, size_t k, const double* rbig,
                          const orc_sketch* th, int overlap) {
  const size_t n = b->n, bp = b->bp_lo;
  const int eff_overlap = overlap && b->cols > 0;
  const size_t hi = b->cols - (eff_overlap ? 1 : 0);
  const size_t mh = th->mhat;
  double* sk = dalloc(mh * k);
  sketch_apply_led(th, vhat, n, k, sk, b->led);
  const size_t sk_have = b->sk_cols;
  const size_t sk_p = (eff_overlap && sk_have > 0) ? sk_have - 1 : sk_have;
  const double* qsk_prior = b->sk; /* first sk_p columns, ld = mh */
  double* proj_sk = dalloc(sk_p * k);
  double* qsk = dalloc(mh * k);
  double* rdiag = dalloc(k * k);
  if (sk_p == 0) {
    orc_householder_qr(sk, mh, k, qsk, rdiag);
  } else {
    double* proj1 = dalloc(sk_p * k);
    orc_transpose_times(qsk_prior, mh, sk_p, sk, k, proj1);
    double* skhat = ddup(sk, mh * k);
    orc_subtract_product(skhat, mh, k, qsk_prior, sk_p, proj1);
    double* iq = dalloc(mh * k);
    double* ir = dalloc(k * k);
    orc_householder_qr(skhat, mh, k, iq, ir);
    double* t1 = dalloc(sk_p * k);
    orc_transpose_times(qsk_prior, mh, sk_p, iq, k, t1);
    double* q2 = ddup(iq, mh * k);
    orc_subtract_product(q2, mh, k, qsk_prior, sk_p, t1);
    double* orr = dalloc(k * k);
    orc_householder_qr(q2, mh, k, qsk, orr);
    update_projection(proj1, t1, sk_p, k, ir, proj_sk);
    orc_multiply_upper(orr, ir, k, rdiag);
    free(proj1);
    free(skhat);
    free(iq);
    free(ir);
    free(t1);
    free(q2);
    free(orr);
  }
  double* resid = ddup(vhat, n * k);
  if (sk_p > 0) orc_subtract_product(resid, n, k, b->q + bp * n, sk_p, proj_sk);
  double* qj = dalloc(n * k);
  int st = orc_apply_inv_upper(resid, n, k, rdiag, qj);
  if (st == ORC_OK) {
    double* full = dalloc(hi * k);
    for (size_t j = 0; j < k; ++j) {
      for (size_t i = 0; i < bp; ++i) AT(full, hi, i, j) = rbig ? AT(rbig, bp, i, j) : 0.0;
      for (size_t i = 0; i < sk_p; ++i) AT(full, hi, bp + i, j) = AT(proj_sk, sk_p, i, j);
    }
    orc_basis_push_panel(b, qj, k, full, rdiag, eff_overlap);
    push_sketched(b, qsk, k, eff_overlap);
    free(full);
  }
  free(sk);
  free(proj_sk);
  free(qsk);
  free(rdiag);
  free(resid);
  free(qj);
  return st;
}

/* block_orth.cpp:329-336 */
int orc_bcgs_pip(orc_basis* b, const double* v, size_t k, int overlap) {
  clear_status();
  return bcgs_pip_impl(b, v, k, NULL, overlap);
}
int orc_rand_bcgs_preproc(orc_basis* b, const double* v, size_t k, const orc_sketch* th,
                          int overlap) {
  clear_status();
  return rand_bcgs_impl(b, v, k, NULL, th, overlap);
}

/* block_orth.cpp:338-356 */
int orc_two_stage_panel(orc_basis* b, const double* v, size_t k, int preproc,
                        const orc_sketch* th, int overlap) {
  clear_status();
  if (preproc == ORC_PRE_RAND_BCGS && th == NULL)
    return set_status(ORC_INVALID, 0, 0.0, "rand_bcgs preprocessing needs a sketch operator");
  const size_t n = b->n, bp = b->bp_lo;
  const int eff_overlap = overlap && b->cols > 0;
  double* vhat = ddup(v, n * k);
  double* rbig = dalloc(bp * k);
  if (bp > 0) orc_bcgs_project_range(b, v, k, 0, bp, vhat, rbig);
  int st = preproc == ORC_PRE_PIP ? bcgs_pip_impl(b, vhat, k, rbig, eff_overlap)
                                  : rand_bcgs_impl(b, vhat, k, rbig, th, eff_overlap);
  free(vhat);
  free(rbig);
  return st;
}

/* block_orth.cpp:358-380 */
int orc_two_stage_finish(orc_basis* b, int preproc, int reorthogonalize, int record,
                         double* stats) {
  clear_status();
  const size_t n = b->n, bp = b->bp_lo, w = b->cols - bp;
  if (record && stats) {
    stats[0] = orc_condition_number(b->q + bp * n, n, w);
    if (isnan(stats[0])) return g_status.code;
    stats[1] = preproc == ORC_PRE_RAND_BCGS ? orc_orthogonality_error(b->sk, b->sk_rows, b->sk_cols)
                                            : 0.0;
  }
  double* bq = dalloc(n * w);
  double* br = dalloc(w * w);
  int st = orc_cholqr(b->q + bp * n, n, w, bq, br, b->led);
  if (st != ORC_OK) {
    free(bq);
    free(br);
    return st;
  }
  refactor_block(b, bp, bq, br);
  if (bp > 0 && reorthogonalize) {
    double* vhat = dalloc(n * w);
    double* coeffs = dalloc(bp * w);
    orc_bcgs_project_range(b, bq, w, 0, bp, vhat, coeffs);
    double* fq = dalloc(n * w);
    double* fr = dalloc(w * w);
    st = orc_cholqr(vhat, n, w, fq, fr, b->led);
    if (st == ORC_OK) reorthogonalize_block(b, bp, fq, coeffs, fr);
    free(vhat);
    free(coeffs);
    free(fq);
    free(fr);
  }
  free(bq);
  free(br);
  return st;
}

/* ------------------------------------------------------------------------ */
/* sparse + problems — proj/src/sparse.cpp, proj/src/problems.cpp           */
/* ------------------------------------------------------------------------ */
typedef struct {
  size_t r, c, seq;
  double v;
} trip;
static int trip_cmp(const void* a, const void* b) {
  const trip *x = (const trip*)a, *y = (const trip*)b;
  if (x->r != y->r) return x->r < y->r ? -1 : 1;
  if (x->c != y->c) return x->c < y->c ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq); /* stable for duplicates */
}
/* sparse.cpp:13-42 */
orc_csr* orc_csr_from_triplets(size_t nrows, size_t ncols, size_t nt, const size_t* rows,
                               const size_t* cols, const double* vals) {
  trip* t = (trip*)malloc((nt ? nt : 1) * sizeof(trip));
  for (size_t i = 0; i < nt; ++i) t[i] = (trip){rows[i], cols[i], i, vals[i]};
  qsort(t, nt, sizeof(trip), trip_cmp);
  orc_csr* m = (orc_csr*)calloc(1, sizeof *m);
  m->nrows = nrows;
  m->ncols = ncols;
  m->row_ptr = (size_t*)calloc(nrows + 1, sizeof(size_t));
  m->col_idx = (size_t*)malloc((nt ? nt : 1) * sizeof(size_t));
  m->values = dalloc(nt);
  size_t nnz = 0;
  for (size_t i = 0; i < nt;) {
    const size_t r = t[i].r, c = t[i].c;
    double v = 0.0;
    while (i < nt && t[i].r == r && t[i].c == c) {
      v += t[i].v;
      ++i;
    }
    m->col_idx[nnz] = c;
    m->values[nnz] = v;
    ++nnz;
    m->row_ptr[r + 1] = nnz;
  }
  for (size_t r = 0; r < nrows; ++r)
    if (m->row_ptr[r + 1] < m->row_ptr[r]) m->row_ptr[r + 1] = m->row_ptr[r];
  m->nnz = nnz;
  free(t);
  return m;
}
void orc_csr_free(orc_csr* a) {
  if (!a) return;
  free(a->row_ptr);
  free(a->col_idx);
  free(a->values);
  free(a);
}

/* problems.cpp:65-113 — rows emitted directly in ascending column order
 * (identical CSR to from_triplets of the reference triplet list) */
static orc_csr* laplace_grid(size_t k, int dims) {
  const size_t n = dims == 2 ? k * k : k * k * k;
  const double diag = dims == 2 ? 4.0 : 6.0;
  orc_csr* m = (orc_csr*)calloc(1, sizeof *m);
  m->nrows = m->ncols = n;
  const size_t cap = n * (size_t)(2 * dims + 1);
  m->row_ptr = (size_t*)calloc(n + 1, sizeof(size_t));
  m->col_idx = (size_t*)malloc(cap * sizeof(size_t));
  m->values = dalloc(cap);
  size_t nnz = 0;
#define PUSH(c, v)            \
  do {                        \
    m->col_idx[nnz] = (c);    \
    m->values[nnz] = (v);     \
    ++nnz;                    \
  } while (0)
  if (dims == 2) {
    for (size_t i = 0; i < k; ++i)
      for (size_t j = 0; j < k; ++j) {
        const size_t me = i * k + j;
        if (i > 0) PUSH(me - k, -1.0);
        if (j > 0) PUSH(me - 1, -1.0);
        PUSH(me, diag);
        if (j + 1 < k) PUSH(me + 1, -1.0);
        if (i + 1 < k) PUSH(me + k, -1.0);
        m->row_ptr[me + 1] = nnz;
      }
  } else {
    for (size_t i = 0; i < k; ++i)
      for (size_t j = 0; j < k; ++j)
        for (size_t l = 0; l < k; ++l) {
          const size_t me = (i * k + j) * k + l;
          if (i > 0) PUSH(me - k * k, -1.0);
          if (j > 0) PUSH(me - k, -1.0);
          if (l > 0) PUSH(me - 1, -1.0);
          PUSH(me, diag);
          if (l + 1 < k) PUSH(me + 1, -1.0);
          if (j + 1 < k) PUSH(me + k, -1.0);
          if (i + 1 < k) PUSH(me + k * k, -1.0);
          m->row_ptr[me + 1] = nnz;
        }
  }
#undef PUSH
  m->nnz = nnz;
  return m;
}
orc_csr* orc_laplace_2d(size_t k) { return laplace_grid(k, 2); }
orc_csr* orc_laplace_3d(size_t k) { return laplace_grid(k, 3); }

/* sparse.cpp:51-63 */
void orc_spmv(const orc_csr* a, const double* x, double* y) {
  for (size_t r = 0; r < a->nrows; ++r) {
    double s = 0.0;
    for (size_t k = a->row_ptr[r]; k < a->row_ptr[r + 1]; ++k) s += a->values[k] * x[a->col_idx[k]];
    y[r] = s;
  }
}
/* gmres.cpp:48-58 */
void orc_mpk(const orc_csr* a, const double* v0, size_t s, double* v) {
  const size_t n = a->nrows;
  memcpy(v, v0, n * sizeof(double));
  for (size_t k = 0; k < s; ++k) orc_spmv(a, v + k * n, v + (k + 1) * n);
}

/* problems.cpp:11-17 */
static void random_orthonormal(size_t rows, size_t cols, orc_rng* rng, double* q) {
  double* g = dalloc(rows * cols);
  for (size_t j = 0; j < cols; ++j)
    for (size_t i = 0; i < rows; ++i) AT(g, rows, i, j) = orc_rng_normal(rng);
  double* r = dalloc(cols * cols);
  orc_householder_qr(g, rows, cols, q, r);
  free(g);
  free(r);
}
/* problems.cpp:21-61 */
void orc_gen_glued(size_t n, size_t np, size_t w, double kp, double kg, uint64_t seed,
                   double* v) {
  const size_t total = np * w;
  orc_rng* rng = orc_rng_new(orc_derive_seed(seed, 0));
  double* u = dalloc(n * total);
  random_orthonormal(n, total, rng, u);
  orc_rng_free(rng);
  double* sigma = dalloc(total);
  double span = kg / kp;
  if (span < 1.0) span = 1.0; /* std::max(kg/kp, 1.0) */
  for (size_t p = 0; p < np; ++p) {
    const double scale = np == 1 ? 1.0 : pow(span, -(double)p / (double)(np - 1));
    for (size_t c = 0; c < w; ++c) {
      const double inner = w == 1 ? 1.0 : pow(kp, -(double)c / (double)(w - 1));
      sigma[p * w + c] = scale * inner;
    }
  }
  memset(v, 0, n * total * sizeof(double));
  double* wj = dalloc(w * w);
  for (size_t p = 0; p < np; ++p) {
    orc_rng* prng = orc_rng_new(orc_derive_seed(seed, 1 + p));
    random_orthonormal(w, w, prng, wj);
    orc_rng_free(prng);
    for (size_t c = 0; c < w; ++c)
      for (size_t l = 0; l < w; ++l) {
        const double coef = sigma[p * w + l] * AT(wj, w, c, l);
        if (coef == 0.0) continue;
        const size_t ucol = p * w + l;
        double* dst = v + (p * w + c) * n;
        const double* src = u + ucol * n;
        for (size_t i = 0; i < n; ++i) dst[i] += coef * src[i];
      }
  }
  free(wj);
  free(sigma);
  free(u);
}

/* ------------------------------------------------------------------------ */
/* s-step GMRES — proj/src/gmres.cpp                                        */
/* ------------------------------------------------------------------------ */
/* gmres.cpp:69-87 X U = B */
int orc_solve_upper_right(const double* b, size_t p, size_t q, const double* u, double* x) {
  for (size_t j = 0; j < q; ++j)
    if (AT(u, q, j, j) == 0.0) return err_singular(j);
  if (x != b) memcpy(x, b, p * q * sizeof(double));
  for (size_t j = 0; j < q; ++j) {
    for (size_t i = 0; i < j; ++i) {
      const double uij = AT(u, q, i, j);
      if (uij == 0.0) continue;
      for (size_t r = 0; r < p; ++r) AT(x, p, r, j) -= AT(x, p, r, i) * uij;
    }
    for (size_t r = 0; r < p; ++r) AT(x, p, r, j) /= AT(u, q, j, j);
  }
  return ORC_OK;
}

/* gmres.cpp:106-151 Givens least squares; returns the residual, y (q) */
double orc_solve_lsq(const double* h, size_t p, size_t q, double gamma, double* y) {
  double* work = ddup(h, p * q);
  double* rhs = dalloc(p);
  rhs[0] = gamma;
  for (size_t k = 0; k < q && k + 1 < p; ++k) {
    const double a = AT(work, p, k, k);
    const double bb = AT(work, p, k + 1, k);
    if (bb == 0.0) continue;
    const double r = hypot(a, bb);
    const double c = a / r;
    const double s = bb / r;
    for (size_t j = k; j < q; ++j) {
      const double t0 = AT(work, p, k, j);
      const double t1 = AT(work, p, k + 1, j);
      AT(work, p, k, j) = c * t0 + s * t1;
      AT(work, p, k + 1, j) = -s * t0 + c * t1;
    }
    const double g0 = rhs[k], g1 = rhs[k + 1];
    rhs[k] = c * g0 + s * g1;
    rhs[k + 1] = -s * g0 + c * g1;
  }
  for (size_t j = 0; j < q; ++j) y[j] = 0.0;
  for (size_t kk = q; kk-- > 0;) {
    if (AT(work, p, kk, kk) == 0.0) {
      y[kk] = 0.0;
      continue;
    }
    double s = rhs[kk];
    for (size_t j = kk + 1; j < q; ++j) s -= AT(work, p, kk, j) * y[j];
    y[kk] = s / AT(work, p, kk, kk);
  }
  double* resid = dalloc(p);
  resid[0] = gamma;
  for (size_t j = 0; j < q; ++j)
    for (size_t i = 0; i < p; ++i) resid[i] -= AT(h, p, i, j) * y[j];
  const double out = vec_norm(resid, p);
  free(resid);
  free(work);
  free(rhs);
  return out;
}

#define HAPPY_TOL 1e-8 /* gmres.cpp:161 */

typedef struct {
  int happy, aborted;
  char detail[512];
  double* happy_col;
} cycle_state;

/* gmres.cpp:173-191 ; returns status, h (p_rows x q) written to hout */
static int assemble_hessenberg(const orc_basis* b, size_t q, const double* happy_col,
                               double* hout) {
  const size_t p = b->cols, cap = b->cap;
  double* rshift = dalloc(p * q);
  double* ceff = dalloc(q * q);
  double* c = dalloc(q);
  for (size_t k = 0; k < q; ++k) {
    if (happy_col && k + 1 == q) {
      for (size_t i = 0; i < p; ++i) AT(rshift, p, i, k) = happy_col[i];
    } else {
      for (size_t i = 0; i < p && i <= k + 1; ++i) AT(rshift, p, i, k) = AT(b->r, cap, i, k + 1);
    }
    orc_basis_input_coeff_col(b, k, q, c);
    for (size_t i = 0; i < q; ++i) AT(ceff, q, i, k) = c[i];
  }
  int st = orc_solve_upper_right(rshift, p, q, ceff, hout);
  free(rshift);
  free(ceff);
  free(c);
  return st;
}

/* gmres.cpp:195-248 */
static void recover_panel(orc_basis* b, const double* v, size_t w, int overlap,
                          const char* scheme_detail, cycle_state* cs) {
  const size_t n = b->n;
  const int eff_overlap = overlap && b->cols > 0;
  const size_t hi = b->cols - (eff_overlap ? 1 : 0);
  double* vhat = dalloc(n * w);
  double* pc = dalloc(hi * w);
  orc_bcgs_project_range(b, v, w, 0, hi, vhat, pc);
  double* rq = dalloc(n * w);
  double* rc = dalloc(w * w);
  size_t kept[64], nkept = 0, disc[64], ndisc = 0, depth = 0;
  double dnorm[64];
  int st = orc_recursive_cholqr(vhat, n, w, rq, rc, kept, &nkept, disc, dnorm, &ndisc, &depth,
                                b->led);
  if (st != ORC_OK) {
    cs->aborted = 1;
    snprintf(cs->detail, sizeof cs->detail, "%s; recovery failed: %s", scheme_detail,
             g_status.msg);
    goto out;
  }
  {
    const size_t d = ndisc == 0 ? w : disc[0];
    if (d == 0) {
      cs->aborted = 1;
      snprintf(cs->detail, sizeof cs->detail, "%s; recovery kept nothing", scheme_detail);
      goto out;
    }
    double* proj = dalloc(hi * d);
    for (size_t j = 0; j < d; ++j)
      for (size_t i = 0; i < hi; ++i) AT(proj, hi, i, j) = AT(pc, hi, i, j);
    double* diag = dalloc(d * d);
    for (size_t i = 0; i < d; ++i)
      for (size_t j = i; j < d; ++j) AT(diag, d, i, j) = AT(rc, w, i, j);
    orc_basis_push_panel(b, rq, d, proj, diag, eff_overlap);
    free(proj);
    free(diag);
    if (d == w) goto out;
    for (size_t t = 0; t < ndisc; ++t) {
      const size_t c = disc[t];
      if (dnorm[t] > HAPPY_TOL * vec_norm(v + c * n, n)) {
        cs->aborted = 1;
        /* std::to_string(double) == "%f" */
        snprintf(cs->detail, sizeof cs->detail, "%s; column %zu unexplained remainder %f",
                 scheme_detail, c, dnorm[t]);
        goto out;
      }
    }
    const size_t p = b->cols;
    free(cs->happy_col);
    cs->happy_col = dalloc(p);
    for (size_t i = 0; i < hi; ++i) cs->happy_col[i] = AT(pc, hi, i, d);
    for (size_t i = 0; i < d; ++i) cs->happy_col[hi + i] = AT(rc, w, i, d);
    cs->happy = 1;
  }
out:
  free(vhat);
  free(pc);
  free(rq);
  free(rc);
}

/* gmres.cpp:255-266 */
static void cycle_diagnostics(const orc_csr* a, const double* q, size_t n, size_t p,
                              const double* h, size_t hq, double a_fro, double* orth,
                              double* arn) {
  *orth = orc_orthogonality_error(q, n, p);
  double* aq = dalloc(n * hq);
  for (size_t c = 0; c < hq; ++c) orc_spmv(a, q + c * n, aq + c * n); /* spmm == per-column spmv */
  double* qh = dalloc(n * hq);
  orc_times(q, n, p, h, hq, qh);
  for (size_t j = 0; j < hq; ++j)
    for (size_t i = 0; i < n; ++i) AT(aq, n, i, j) -= AT(qh, n, i, j);
  *arn = frobenius(aq, n, hq) / a_fro;
  free(aq);
  free(qh);
}

/* gmres.cpp:34-46 */
static int validate_config(const orc_solver_config* cfg) {
  if (!(cfg->rel_tol > 0.0 && cfg->rel_tol < 1.0))
    return set_status(ORC_INVALID, 0, 0.0, "rel_tol must lie in (0, 1)");
  if (cfg->max_restarts == 0) return set_status(ORC_INVALID, 0, 0.0, "max_restarts must be positive");
  if (cfg->scheme == ORC_STANDARD_CGS2) {
    if (cfg->m < 1) return set_status(ORC_INVALID, 0, 0.0, "restart length must be positive");
    return ORC_OK;
  }
  if (cfg->s < 1 || cfg->s > cfg->shat || cfg->shat > cfg->m)
    return set_status(ORC_INVALID, 0, 0.0, "need 1 <= s <= shat <= m");
  if (cfg->shat % cfg->s != 0) return set_status(ORC_INVALID, 0, 0.0, "s must divide shat");
  if (cfg->m % cfg->shat != 0) return set_status(ORC_INVALID, 0, 0.0, "shat must divide m");
  return ORC_OK;
}

static void push_hist(orc_solve_report* rep, double relres, double lsq, double orth, double arn) {
  if (rep->nhist < 256) {
    rep->relres[rep->nhist] = relres;
    rep->lsq[rep->nhist] = lsq;
    rep->orth[rep->nhist] = orth;
    rep->arnoldi[rep->nhist] = arn;
    rep->nhist++;
  }
}

/* gmres.cpp:270-512 */
int orc_sstep_gmres(const orc_csr* a, const double* b, const double* x0,
                    const orc_solver_config* cfg, double* x, orc_solve_report* rep) {
  clear_status();
  memset(rep, 0, sizeof *rep);
  int st = validate_config(cfg);
  if (st) return st;
  if (a->nrows != a->ncols) return set_status(ORC_INVALID, 0, 0.0, "coefficient matrix must be square");
  if (cfg->n != 0 && cfg->n != a->nrows)
    return set_status(ORC_INVALID, 0, 0.0, "config n does not match the matrix dimension");
  const size_t n = a->nrows;
  memcpy(x, x0, n * sizeof(double));
  orc_ledger extra = {0, 0, 0, 0};

  double a_fro = 0.0;
  for (size_t i = 0; i < a->nnz; ++i) a_fro += a->values[i] * a->values[i];
  a_fro = sqrt(a_fro);
  if (a_fro == 0.0) a_fro = 1.0;

  double* r = dalloc(n);
  double* ax = dalloc(n);
#define TRUE_RESIDUAL()                                   \
  (orc_spmv(a, x, ax), ({                                 \
     for (size_t i_ = 0; i_ < n; ++i_) r[i_] = b[i_] - ax[i_]; \
     extra[3]++;                                          \
     vec_norm(r, n);                                      \
   }))
  double gamma = TRUE_RESIDUAL();
  const double gamma0 = gamma;
  rep->initial_residual = gamma0;
  if (gamma0 == 0.0) {
    rep->converged = 1;
    rep->final_relres = 0.0;
    free(r);
    free(ax);
    return ORC_OK;
  }
#define ACC_LEDGER(l)                                           \
  do {                                                          \
    for (int q_ = 0; q_ < 4; ++q_) rep->reduce[q_] += (l)[q_];  \
    rep->reduce_total += (l)[0] + (l)[1] + (l)[2] + (l)[3];     \
  } while (0)

  const int twostage = cfg->scheme == ORC_TWOSTAGE_PIP || cfg->scheme == ORC_TWOSTAGE_RANDBCGS;
  const int preproc = cfg->scheme == ORC_TWOSTAGE_PIP ? ORC_PRE_PIP : ORC_PRE_RAND_BCGS;
  int done = 0;
  st = ORC_OK;
  for (size_t cycle = 0; cycle < cfg->max_restarts && !done; ++cycle) {
    rep->restarts++;
    const double cycle_gamma = gamma;

    if (cfg->scheme == ORC_STANDARD_CGS2) { /* gmres.cpp:327-386 */
      const size_t m = cfg->m;
      orc_ledger led = {0, 0, 0, 0};
      double* q = dalloc(n * (m + 1));
      double* h = dalloc((m + 1) * m);
      for (size_t i = 0; i < n; ++i) q[i] = r[i] / gamma;
      size_t q_in = m;
      int happy = 0;
      double* wv = dalloc(n);
      for (size_t k = 0; k < m; ++k) {
        orc_spmv(a, q + k * n, wv);
        for (int pass = 0; pass < 2; ++pass) {
          led[0]++;
          for (size_t i = 0; i <= k; ++i) {
            double dot = 0.0;
            for (size_t t = 0; t < n; ++t) dot += q[t + i * n] * wv[t];
            AT(h, m + 1, i, k) += dot;
            for (size_t t = 0; t < n; ++t) wv[t] -= dot * q[t + i * n];
          }
        }
        const double hnorm = vec_norm(wv, n);
        led[3]++;
        double hcol = 0.0;
        for (size_t i = 0; i <= k; ++i) hcol += AT(h, m + 1, i, k) * AT(h, m + 1, i, k);
        if (hnorm <= 1e-12 * sqrt(hcol + hnorm * hnorm)) {
          q_in = k + 1;
          happy = 1;
          break;
        }
        AT(h, m + 1, k + 1, k) = hnorm;
        for (size_t i = 0; i < n; ++i) q[i + (k + 1) * n] = wv[i] / hnorm;
      }
      const size_t p = happy ? q_in : q_in + 1;
      double* heff = dalloc(p * q_in);
      for (size_t j = 0; j < q_in; ++j)
        for (size_t i = 0; i < p; ++i) AT(heff, p, i, j) = AT(h, m + 1, i, j);
      double* y = dalloc(q_in);
      const double lsq = orc_solve_lsq(heff, p, q_in, gamma, y);
      for (size_t j = 0; j < q_in; ++j)
        for (size_t i = 0; i < n; ++i) x[i] += q[i + j * n] * y[j];
      gamma = TRUE_RESIDUAL();
      rep->iterations += q_in;
      rep->happy_breakdown = rep->happy_breakdown || happy;
      ACC_LEDGER(led);
      double orth = 0, arn = 0;
      if (cfg->diagnostics) cycle_diagnostics(a, q, n, p, heff, q_in, a_fro, &orth, &arn);
      push_hist(rep, gamma / gamma0, lsq, orth, arn);
      if (gamma / gamma0 <= cfg->rel_tol) {
        rep->converged = 1;
        done = 1;
      } else if (happy) {
        snprintf(rep->breakdown_detail, sizeof rep->breakdown_detail,
                 "stagnated on an invariant subspace");
        done = 1;
      }
      free(q);
      free(h);
      free(wv);
      free(heff);
      free(y);
      continue;
    }

    orc_basis* store = orc_basis_new(n, cfg->m + 1);
    orc_sketch* theta = NULL;
    if (cfg->scheme == ORC_BCGS2_RANDCHOLQR)
      theta = orc_sketch_build(cfg->sketch, n, cfg->s, orc_derive_seed(cfg->seed, cycle + 1));
    else if (cfg->scheme == ORC_TWOSTAGE_RANDBCGS)
      theta = orc_sketch_build(cfg->sketch, n, cfg->shat, orc_derive_seed(cfg->seed, cycle + 1));
    if ((cfg->scheme == ORC_BCGS2_RANDCHOLQR || cfg->scheme == ORC_TWOSTAGE_RANDBCGS) && !theta) {
      orc_basis_free(store);
      st = g_status.code;
      break; /* AmbientTooSmall escapes sstep_gmres_solve */
    }
    double* q1 = dalloc(n);
    for (size_t i = 0; i < n; ++i) q1[i] = r[i] / gamma;

    cycle_state cs;
    memset(&cs, 0, sizeof cs);
    const size_t panels = cfg->m / cfg->s;
    const size_t ppb = twostage ? cfg->shat / cfg->s : panels;
    const size_t k = cfg->s + 1;
    double* v = dalloc(n * k);
    double* seed_vec = dalloc(n);
    for (size_t j = 0; j < panels && !cs.happy && !cs.aborted; ++j) {
      if (j == 0) {
        memcpy(seed_vec, q1, n * sizeof(double));
      } else {
        const size_t k0 = store->cols - 1;
        orc_basis_mark_seed(store, k0);
        memcpy(seed_vec, store->q + k0 * n, n * sizeof(double));
      }
      orc_mpk(a, seed_vec, cfg->s, v);
      const int overlap = j > 0;
      if (twostage && j % ppb == 0)
        orc_basis_begin_big_panel(store, theta ? theta->mhat : 0, overlap);
      int pst;
      if (twostage)
        pst = orc_two_stage_panel(store, v, k, preproc, theta, overlap);
      else
        pst = orc_bcgs2(store, v, k,
                        cfg->scheme == ORC_BCGS2_CHOLQR2 ? ORC_INTRA_CHOLQR2 : ORC_INTRA_RAND_CHOLQR,
                        theta, overlap);
      if (pst != ORC_OK) {
        char what[512];
        snprintf(what, sizeof what, "%s", g_status.msg);
        if (!twostage || store->cols == 0) {
          recover_panel(store, v, k, overlap, what, &cs);
        } else {
          cs.aborted = 1;
          snprintf(cs.detail, sizeof cs.detail, "%s", what);
        }
      }
      if (twostage && !cs.happy && !cs.aborted && (j + 1) % ppb == 0) {
        if (orc_two_stage_finish(store, preproc, cfg->reorthogonalize, 0, NULL) != ORC_OK) {
          cs.aborted = 1;
          snprintf(cs.detail, sizeof cs.detail, "second stage: %s", g_status.msg);
        }
      }
    }
    if (twostage && cs.aborted && store->cols > store->bp_lo && store->cols > 0) {
      if (orc_two_stage_finish(store, preproc, cfg->reorthogonalize, 0, NULL) != ORC_OK) {
        size_t L = strlen(cs.detail);
        snprintf(cs.detail + L, sizeof cs.detail - L,
                 "; basis after the last completed big panel unusable");
        orc_basis_free(store);
        store = orc_basis_new(n, 1);
      }
    }
    ACC_LEDGER(store->led);

    const size_t p = store->cols;
    const size_t q_in = cs.happy ? p : (p > 0 ? p - 1 : 0);
    if (q_in == 0) {
      rep->breakdown = cs.aborted;
      snprintf(rep->breakdown_detail, sizeof rep->breakdown_detail, "%s", cs.detail);
      rep->final_relres = gamma / gamma0;
      done = 1;
    } else {
      const size_t hp = cs.happy ? p : p; /* rows of H = store.cols() */
      double* h = dalloc(hp * q_in);
      st = assemble_hessenberg(store, q_in, cs.happy ? cs.happy_col : NULL, h);
      if (st != ORC_OK) { /* SingularTriangular escapes the solver */
        free(h);
        free(q1);
        free(v);
        free(seed_vec);
        free(cs.happy_col);
        orc_sketch_free(theta);
        orc_basis_free(store);
        break;
      }
      double* y = dalloc(q_in);
      const double lsq = orc_solve_lsq(h, hp, q_in, gamma, y);
      for (size_t j = 0; j < q_in; ++j) {
        const double* col = store->q + j * n;
        for (size_t i = 0; i < n; ++i) x[i] += col[i] * y[j];
      }
      gamma = TRUE_RESIDUAL();
      rep->iterations += q_in;
      rep->happy_breakdown = rep->happy_breakdown || cs.happy;
      double orth = 0, arn = 0;
      if (cfg->diagnostics) cycle_diagnostics(a, store->q, n, p, h, q_in, a_fro, &orth, &arn);
      push_hist(rep, gamma / gamma0, lsq, orth, arn);
      if (gamma / gamma0 <= cfg->rel_tol) {
        rep->converged = 1;
        done = 1;
      } else if (cs.aborted) {
        rep->breakdown = 1;
        snprintf(rep->breakdown_detail, sizeof rep->breakdown_detail, "%s", cs.detail);
        done = 1;
      } else if (cs.happy && gamma >= cycle_gamma * (1.0 - 1e-12)) {
        snprintf(rep->breakdown_detail, sizeof rep->breakdown_detail,
                 "stagnated on an invariant subspace");
        done = 1;
      }
      free(h);
      free(y);
    }
    free(q1);
    free(v);
    free(seed_vec);
    free(cs.happy_col);
    orc_sketch_free(theta);
    orc_basis_free(store);
  }
  ACC_LEDGER(extra);
  rep->final_relres = gamma / gamma0;
  free(r);
  free(ax);
  if (st == ORC_OK) clear_status();
  return st;
#undef TRUE_RESIDUAL
#undef ACC_LEDGER
}
