// mt64_jump.cpp — MT19937-64 jump-ahead polynomials (host side).
//
// The reference draws every sketch entry from one sequential std::mt19937_64
// stream (proj/include/blkorth/rng.hpp:22-64, proj/src/sketch.cpp:30-45).  To
// generate that exact stream in parallel on the GPU, each chunk of the stream
// starts from a jumped state.  MT19937-64 is F2-linear: every bit position of
// the generated (untempered) word sequence g[i] satisfies the same linear
// recurrence whose characteristic polynomial phi has degree 19937.  Hence, for
// p(x) = x^J mod phi(x),
//     g[J + t] = XOR_{k : p_k = 1} g[k + t]      for every t >= 0,
// so the 312-word window starting at J is an XOR of windows of the first
// 20248 generated words.  phi was recovered with Berlekamp-Massey and is
// compiled in (mt64_phi_table.h, scripts/gen_mt64_phi.sh); the
// seed-independent polynomials x^J mod phi are computed with carry-less
// multiplication + Barrett reduction and cached for the process lifetime.
//
// Conventions: g[0] is the first word produced by the first twist after
// seeding (so output draw d == temper(g[d])).

#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "mt64_jump.h"
#ifndef BO_MT64_NO_PHI_TABLE
#include "mt64_phi_table.h"
#endif

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace bo {
namespace mt64 {

namespace {

constexpr int kDeg = 19937;            // degree of phi
constexpr int kWords = (kDeg + 63) / 64;  // 312 words hold a reduced polynomial

using Poly = std::vector<uint64_t>;

inline int get_bit(const Poly& p, long i) { return (p[i >> 6] >> (i & 63)) & 1; }
inline void flip_bit(Poly& p, long i) { p[i >> 6] ^= 1ULL << (i & 63); }

// ---- carry-less multiply ----------------------------------------------------
#if defined(__x86_64__)
__attribute__((target("pclmul,sse2"))) static void clmul_words(const uint64_t* a, size_t na,
                                                                const uint64_t* b, size_t nb,
                                                                uint64_t* out /* na+nb */) {
  std::memset(out, 0, (na + nb) * sizeof(uint64_t));
  for (size_t i = 0; i < na; ++i) {
    if (a[i] == 0) continue;
    const __m128i av = _mm_set_epi64x(0, (long long)a[i]);
    for (size_t j = 0; j < nb; ++j) {
      const __m128i bv = _mm_set_epi64x(0, (long long)b[j]);
      const __m128i pr = _mm_clmulepi64_si128(av, bv, 0x00);
      out[i + j] ^= (uint64_t)_mm_cvtsi128_si64(pr);
      out[i + j + 1] ^= (uint64_t)_mm_cvtsi128_si64(_mm_unpackhi_epi64(pr, pr));
    }
  }
}
static bool have_pclmul() { return __builtin_cpu_supports("pclmul"); }
#else
static void clmul_words(const uint64_t*, size_t, const uint64_t*, size_t, uint64_t*) {}
static bool have_pclmul() { return false; }
#endif

static inline void clmul64_soft(uint64_t a, uint64_t b, uint64_t& lo, uint64_t& hi) {
  lo = hi = 0;
  for (int i = 0; i < 64; ++i)
    if ((b >> i) & 1) {
      lo ^= a << i;
      if (i) hi ^= a >> (64 - i);
    }
}
static void clmul_words_soft(const uint64_t* a, size_t na, const uint64_t* b, size_t nb,
                             uint64_t* out) {
  std::memset(out, 0, (na + nb) * sizeof(uint64_t));
  for (size_t i = 0; i < na; ++i) {
    if (a[i] == 0) continue;
    for (size_t j = 0; j < nb; ++j) {
      uint64_t lo, hi;
      clmul64_soft(a[i], b[j], lo, hi);
      out[i + j] ^= lo;
      out[i + j + 1] ^= hi;
    }
  }
}
static void clmul(const Poly& a, const Poly& b, Poly& out) {
  out.assign(a.size() + b.size(), 0);
  if (have_pclmul())
    clmul_words(a.data(), a.size(), b.data(), b.size(), out.data());
  else
    clmul_words_soft(a.data(), a.size(), b.data(), b.size(), out.data());
}

// bits [lo, lo+count) of p as a new polynomial
static Poly extract(const Poly& p, long lo, long count) {
  Poly out((count + 63) / 64, 0);
  for (long w = 0; w < (long)out.size(); ++w) {
    const long bit = lo + w * 64;
    const long wi = bit >> 6, sh = bit & 63;
    uint64_t v = 0;
    if (wi < (long)p.size()) v = p[wi] >> sh;
    if (sh && wi + 1 < (long)p.size()) v |= p[wi + 1] << (64 - sh);
    out[w] = v;
  }
  const long extra = (long)out.size() * 64 - count;
  if (extra > 0) out.back() &= (~0ULL) >> extra;
  return out;
}

struct Field {
  Poly phi;  // degree kDeg, kWords+1 words
  Poly mu;   // floor(x^(2d) / phi), degree d
  std::map<uint64_t, Poly> cache;
  std::mutex mu_lock;
  bool ready = false;
};
Field& field() {
  static Field f;
  return f;
}

// ---- std::mt19937_64 reference generator (host) ---------------------------
struct Mt {
  uint64_t s[312];
  int idx;
  explicit Mt(uint64_t seed) {
    s[0] = seed;
    for (int i = 1; i < 312; ++i) s[i] = 6364136223846793005ULL * (s[i - 1] ^ (s[i - 1] >> 62)) + i;
    idx = 312;
  }
  void twist() {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (s[i] & 0xFFFFFFFF80000000ULL) | (s[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
      s[i] = s[(i + 156) % 312] ^ xa;
    }
    idx = 0;
  }
  uint64_t raw() {  // untempered g[i]
    if (idx >= 312) twist();
    return s[idx++];
  }
};

// Berlekamp-Massey over GF(2) on bit sequence s[0..N): returns connection
// polynomial C (C[0]=1) of length L+1 with s[i] = sum_{j=1..L} C[j] s[i-j].
static Poly berlekamp_massey(const std::vector<uint8_t>& s, int& L_out) {
  const long N = (long)s.size();
  const long W = (N + 64) / 64 + 1;
  Poly C(W, 0), B(W, 0), T;
  C[0] = B[0] = 1;
  long L = 0, m = 1;
  for (long n = 0; n < N; ++n) {
    int d = s[n];
    for (long i = 1; i <= L; ++i) d ^= get_bit(C, i) & s[n - i];
    if (d == 0) {
      ++m;
      continue;
    }
    T = C;
    // C ^= B << m
    const long ws = m >> 6, bs = m & 63;
    for (long i = W - 1; i >= ws; --i) {
      uint64_t v = B[i - ws] << bs;
      if (bs && i - ws - 1 >= 0) v |= B[i - ws - 1] >> (64 - bs);
      C[i] ^= v;
    }
    if (2 * L <= n) {
      L = n + 1 - L;
      B = T;
      m = 1;
    } else {
      ++m;
    }
  }
  L_out = (int)L;
  return C;
}

// r = a mod phi for deg(a) < 2d (Barrett with precomputed mu)
static Poly reduce(const Field& f, const Poly& a) {
  // q = floor( floor(a / x^d) * mu / x^d )
  const Poly ahi = extract(a, kDeg, kDeg + 1);
  Poly t;
  clmul(ahi, f.mu, t);
  const Poly q = extract(t, kDeg, kDeg + 1);
  Poly qp;
  clmul(q, f.phi, qp);
  Poly r(kWords, 0);
  for (int i = 0; i < kWords; ++i) r[i] = (i < (int)a.size() ? a[i] : 0) ^ (i < (int)qp.size() ? qp[i] : 0);
  const int extra = kWords * 64 - kDeg;
  r[kWords - 1] &= (~0ULL) >> extra;
  return r;
}

static Poly mulmod(const Field& f, const Poly& a, const Poly& b) {
  Poly t;
  clmul(a, b, t);
  return reduce(f, t);
}

// phi(x) recovered from the generator itself: Berlekamp-Massey over the LSB of
// 2 deg + 64 untempered words (any nonzero seed).  Empty if the recovered
// degree is not 19937.
static Poly phi_by_berlekamp_massey() {
  Mt mt(5489ULL);
  const long N = 2 * kDeg + 64;
  std::vector<uint8_t> bits(N);
  for (long i = 0; i < N; ++i) bits[i] = (uint8_t)(mt.raw() & 1);
  int L = 0;
  const Poly C = berlekamp_massey(bits, L);
  if (L != kDeg) return Poly();
  // phi(x) = x^L C(1/x): coefficient of x^(L-j) is C[j]
  Poly phi(kWords + 1, 0);
  for (int j = 0; j <= L; ++j)
    if (get_bit(C, j)) flip_bit(phi, L - j);
  return phi;
}

static void init_field(Field& f) {
#ifdef BO_MT64_NO_PHI_TABLE
  f.phi = phi_by_berlekamp_massey();
#else
  // the table scripts/gen_mt64_phi.sh printed from phi_by_berlekamp_massey()
  // (0.5-0.7 s saved per process); the jump-window tests check the result
  // against the sequential generator
  f.phi.assign(kMt64Phi, kMt64Phi + sizeof(kMt64Phi) / sizeof(kMt64Phi[0]));
#endif
  f.ready = f.phi.size() == (size_t)kWords + 1 && get_bit(f.phi, kDeg) && get_bit(f.phi, 0) &&
            f.phi[kWords] == 0 && (f.phi[kDeg >> 6] >> ((kDeg & 63) + 1)) == 0;
  if (!f.ready) return;
  // mu = floor(x^(2d) / phi) by long division
  const long top = 2L * kDeg;
  Poly rem((top + 64) / 64 + 1, 0);
  flip_bit(rem, top);
  f.mu.assign(kWords + 1, 0);
  for (long i = top; i >= kDeg; --i) {
    if (!get_bit(rem, i)) continue;
    const long sh = i - kDeg;
    flip_bit(f.mu, sh);
    // rem ^= phi << sh
    const long ws = sh >> 6, bs = sh & 63;
    for (long w = 0; w < (long)f.phi.size(); ++w) {
      const uint64_t v = f.phi[w];
      if (!v) continue;
      rem[w + ws] ^= v << bs;
      if (bs && w + ws + 1 < (long)rem.size()) rem[w + ws + 1] ^= v >> (64 - bs);
    }
  }
}

// x^J mod phi by square-and-multiply (multiply by x is a shift + reduce)
static Poly xpow(const Field& f, uint64_t J) {
  Poly r(kWords, 0);
  r[0] = 1;
  if (J == 0) return r;
  int hb = 63;
  while (!((J >> hb) & 1)) --hb;
  for (int b = hb; b >= 0; --b) {
    r = mulmod(f, r, r);
    if ((J >> b) & 1) {
      // r *= x
      Poly s(kWords + 1, 0);
      for (int i = 0; i < kWords; ++i) {
        s[i] |= r[i] << 1;
        s[i + 1] |= r[i] >> 63;
      }
      r = reduce(f, s);
    }
  }
  return r;
}

}  // namespace

bool ready() {
  Field& f = field();
  std::lock_guard<std::mutex> g(f.mu_lock);
  if (!f.ready && f.phi.empty()) init_field(f);
  return f.ready;
}

// p = x^J mod phi as kWords uint64 words (bit k = coefficient of x^k).
// Consecutive requests J, J+L, J+2L ... reuse the cache by chaining.
void jump_poly(uint64_t J, uint64_t* out) {
  Field& f = field();
  std::lock_guard<std::mutex> g(f.mu_lock);
  if (!f.ready && f.phi.empty()) init_field(f);
  auto it = f.cache.find(J);
  if (it == f.cache.end()) {
    // find the closest cached J' < J with (J - J') a cached delta, else direct
    Poly r;
    auto lb = f.cache.lower_bound(J);
    bool done = false;
    if (lb != f.cache.begin()) {
      auto prev = std::prev(lb);
      const uint64_t d = J - prev->first;
      auto dit = f.cache.find(d);
      if (dit != f.cache.end()) {
        r = mulmod(f, prev->second, dit->second);
        done = true;
      }
    }
    if (!done) r = xpow(f, J);
    it = f.cache.emplace(J, std::move(r)).first;
  }
  std::memcpy(out, it->second.data(), kWords * sizeof(uint64_t));
}

void jump_polys_strided(uint64_t J0, uint64_t L, uint64_t count, uint64_t* out) {
  Field& f = field();
  {
    std::lock_guard<std::mutex> g(f.mu_lock);
    if (!f.ready && f.phi.empty()) init_field(f);
  }
  if (count == 0) return;
  // cache x^L first so that chaining works
  std::vector<uint64_t> tmp(kWords);
  if (L) jump_poly(L, tmp.data());
  for (uint64_t c = 0; c < count; ++c) jump_poly(J0 + c * L, out + c * kWords);
}

int poly_words() { return kWords; }
int prefix_words() { return kDeg + 311; }  // g[0 .. kDeg-1+311]

void prefix(uint64_t seed, uint64_t* g) {
  Mt mt(seed);
  for (int i = 0; i < prefix_words(); ++i) g[i] = mt.raw();
}

// Host-side reference jump (tests): window g[J .. J+311] for the given seed.
void jump_window_host(uint64_t seed, uint64_t J, uint64_t* w) {
  std::vector<uint64_t> g(prefix_words());
  prefix(seed, g.data());
  std::vector<uint64_t> p(kWords);
  jump_poly(J, p.data());
  std::memset(w, 0, 312 * sizeof(uint64_t));
  for (int k = 0; k < kDeg; ++k)
    if ((p[k >> 6] >> (k & 63)) & 1)
      for (int t = 0; t < 312; ++t) w[t] ^= g[k + t];
}

}  // namespace mt64
}  // namespace bo
