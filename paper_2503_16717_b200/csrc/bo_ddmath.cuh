// bo_ddmath.cuh — correctly-rounded (to ~2^-90 relative before the final
// rounding) natural log and sin/cos in double-double arithmetic, for the
// device Box-Muller of the Gaussian sketch (bo_sketch_gen.cuh).
//
// The reference draws normals with glibc's log / sin / cos
// (proj/include/blkorth/rng.hpp:37-49).  glibc 2.39 is correctly rounded for
// all but ~0.1 % of these inputs (SURVEY.md finding 1) while CUDA's libdevice
// log / sincos are off by up to 1-2 ulp much more often, which put round 1's
// device sketch up to 5 ulp from the reference.  Evaluating both functions in
// double-double and rounding once makes every device value the correctly
// rounded one, so the only differences left are glibc's own misroundings.
//
// log x   : x = 2^e f, f in [0.75, 1.5); c = i/128 nearest f (i = 96..192);
//           t = (f - c)/c via the dd reciprocal table, |t| <= 0.0053;
//           log x = e ln2 + log c + log1p(t), log1p by a degree-12 series with
//           its four leading coefficients in dd.
// sin/cos : k = rint(a 2/pi), r = a - k pi/2 with a three-part pi/2;
//           r0 = j/64 nearest r, d = r - r0 (|d| <= 1/128);
//           sin r = S0 + S0 (cos d - 1) + C0 sin d, cos r = C0 + C0 (cos d - 1) - S0 sin d,
//           with dd tables of sin / cos(j/64), then the quadrant.
// The same source compiles for the host (g++ -ffp-contract=off), which the
// CPU tests use to pin it against mpmath and glibc (tests/test_ddmath.py).
#pragma once
#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define BO_DDM_FN __device__ __forceinline__
#define BO_DDM_TABLE static __device__ const
#else
#include <cmath>
#define BO_DDM_FN static inline
#define BO_DDM_TABLE static const
#endif

#include "bo_ddmath_tables.h"

namespace bo {
namespace ddm {

// unfused IEEE operations: the error-free transforms below need exactly
// these roundings, so no contraction into FMAs is allowed
#ifdef __CUDACC__
BO_DDM_FN double A(double a, double b) { return __dadd_rn(a, b); }
BO_DDM_FN double S(double a, double b) { return __dsub_rn(a, b); }
BO_DDM_FN double M(double a, double b) { return __dmul_rn(a, b); }
BO_DDM_FN double F(double a, double b, double c) { return __fma_rn(a, b, c); }
BO_DDM_FN double RINT(double a) { return rint(a); }
BO_DDM_FN double TAB(const double* p) { return __ldg(p); }
BO_DDM_FN uint64_t BITS(double x) { return (uint64_t)__double_as_longlong(x); }
BO_DDM_FN double DBL(uint64_t u) { return __longlong_as_double((long long)u); }
#else
BO_DDM_FN double A(double a, double b) { return a + b; }
BO_DDM_FN double S(double a, double b) { return a - b; }
BO_DDM_FN double M(double a, double b) { return a * b; }
BO_DDM_FN double F(double a, double b, double c) { return std::fma(a, b, c); }
BO_DDM_FN double RINT(double a) { return std::rint(a); }
BO_DDM_FN double TAB(const double* p) { return *p; }
BO_DDM_FN uint64_t BITS(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
}
BO_DDM_FN double DBL(uint64_t u) {
  double x;
  std::memcpy(&x, &u, 8);
  return x;
}
#endif

struct DD {
  double hi, lo;
};

BO_DDM_FN DD two_sum(double a, double b) {
  const double s = A(a, b), bb = S(s, a);
  return {s, A(S(a, S(s, bb)), S(b, bb))};
}
BO_DDM_FN DD quick_two_sum(double a, double b) {  // |a| >= |b| or a == 0
  const double s = A(a, b);
  return {s, S(b, S(s, a))};
}
BO_DDM_FN DD two_prod(double a, double b) {
  const double p = M(a, b);
  return {p, F(a, b, -p)};
}
BO_DDM_FN DD neg(DD a) { return {-a.hi, -a.lo}; }
BO_DDM_FN DD add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi);
  const DD t = two_sum(a.lo, b.lo);
  s.lo = A(s.lo, t.hi);
  s = quick_two_sum(s.hi, s.lo);
  s.lo = A(s.lo, t.lo);
  return quick_two_sum(s.hi, s.lo);
}
BO_DDM_FN DD add_d(DD a, double b) {
  DD s = two_sum(a.hi, b);
  s.lo = A(s.lo, a.lo);
  return quick_two_sum(s.hi, s.lo);
}
BO_DDM_FN DD mul(DD a, DD b) {
  DD p = two_prod(a.hi, b.hi);
  p.lo = A(p.lo, F(a.hi, b.lo, M(a.lo, b.hi)));
  return quick_two_sum(p.hi, p.lo);
}
BO_DDM_FN DD mul_d(DD a, double b) {
  DD p = two_prod(a.hi, b);
  p.lo = F(a.lo, b, p.lo);
  return quick_two_sum(p.hi, p.lo);
}

// log(x) rounded to nearest, x positive, normal, finite (Box-Muller: x in [2^-53, 1])
BO_DDM_FN double log_rn(double x) {
  const uint64_t bits = BITS(x);
  int e = (int)((bits >> 52) & 0x7ff) - 1023;
  double f = DBL((bits & 0xfffffffffffffULL) | 0x3ff0000000000000ULL);  // [1, 2)
  if (f >= 1.5) {
    f = M(f, 0.5);
    e += 1;
  }
  const int i = (int)RINT(M(f, 128.0));  // 96..192
  const double d = S(f, M((double)i, 0x1p-7));  // exact
  const double* tb = kLogTab + 4 * (i - kLogLo);
  const DD rc{TAB(tb), TAB(tb + 1)}, lc{TAB(tb + 2), TAB(tb + 3)};
  const DD t = mul_d(rc, d);  // (f - c) / c
  const double th = t.hi;
  // log1p(t) = t + t^2 (-1/2 + t (1/3 + t (-1/4 + t R))), R = sum_{j>=5} (-1)^{j+1} t^{j-5} / j
  double R = F(th, -1.0 / 12.0, 1.0 / 11.0);
  R = F(th, R, -1.0 / 10.0);
  R = F(th, R, 1.0 / 9.0);
  R = F(th, R, -1.0 / 8.0);
  R = F(th, R, 1.0 / 7.0);
  R = F(th, R, -1.0 / 6.0);
  R = F(th, R, 1.0 / 5.0);
  const DD a4 = two_sum(-0.25, M(th, R));
  const DD a3 = add(DD{kThirdHi, kThirdLo}, mul(t, a4));
  const DD a2 = add_d(mul(t, a3), -0.5);
  const DD L = add(t, mul(mul(t, t), a2));
  DD el = two_prod((double)e, kLn2Hi);
  el.lo = F((double)e, kLn2Lo, el.lo);
  el = quick_two_sum(el.hi, el.lo);
  return add(add(el, lc), L).hi;
}

// sin(a), cos(a) rounded to nearest, 0 <= a < 2 pi (Box-Muller angle)
BO_DDM_FN void sincos_rn(double a, double* sn, double* cs) {
  const double kd = RINT(M(a, kTwoOverPi));  // quadrant 0..4
  const int k = (int)kd;
  DD r = add(DD{a, 0.0}, neg(two_prod(kd, kPio2_1)));
  r = add(r, neg(two_prod(kd, kPio2_2)));
  r = add_d(r, -M(kd, kPio2_3));
  const double jd = RINT(M(r.hi, 64.0));  // |j| <= 51
  const int j = (int)jd;
  const DD dl = two_sum(S(r.hi, M(jd, 0x1p-6)), r.lo);  // r - j/64 (the subtraction is exact)
  const DD z = mul(dl, dl);
  const double zh = z.hi;
  // sin d = d + d z (-1/6 + z qs);  cos d - 1 = z (-1/2 + z qc)
  const double qs = F(zh, F(zh, 1.0 / 362880.0, -1.0 / 5040.0), 1.0 / 120.0);
  const DD ps = add(DD{-kSixthHi, -kSixthLo}, two_prod(zh, qs));
  const DD sd = add(dl, mul(mul(dl, z), ps));
  const double qc = F(zh, F(zh, F(zh, -1.0 / 3628800.0, 1.0 / 40320.0), -1.0 / 720.0), 1.0 / 24.0);
  const DD cm = mul(z, two_sum(-0.5, M(zh, qc)));
  const int aj = j < 0 ? -j : j;
  const double* tb = kTrigTab + 4 * aj;
  DD s0{TAB(tb), TAB(tb + 1)};
  const DD c0{TAB(tb + 2), TAB(tb + 3)};
  if (j < 0) s0 = neg(s0);
  const DD sr = add(s0, add(mul(s0, cm), mul(c0, sd)));
  const DD cr = add(c0, add(mul(c0, cm), neg(mul(s0, sd))));
  switch (k & 3) {
    case 0: *sn = sr.hi; *cs = cr.hi; break;
    case 1: *sn = cr.hi; *cs = -sr.hi; break;
    case 2: *sn = -sr.hi; *cs = -cr.hi; break;
    default: *sn = -cr.hi; *cs = sr.hi; break;
  }
}

// ---------------------------------------------------------------------------
// Fast paths (Ziv's strategy).  The same reductions, with only the leading
// terms carried in double-double: relative error below 2^-67 before the final
// rounding (the lo parts collect every term below 2^-53 of the result).  The
// rounding of hi + lo is then certain unless hi + lo lies within 2^-65 |hi|
// of a midpoint between hi and a neighbour (probability ~2^-12); round_safe
// detects that and the caller re-evaluates with the full-precision functions
// above.  Results are identical to log_rn / sincos_rn (tests/test_ddmath.py
// compares them over 4e6 inputs); the work is ~1/3.
// ---------------------------------------------------------------------------
BO_DDM_FN bool round_safe(double hi, double lo) {
  const uint64_t hb = BITS(hi) & 0x7fffffffffffffffULL;
  if (hb == 0) return lo == 0.0;                     // an exact zero
  if ((hb & 0x000fffffffffffffULL) == 0) return false;  // hi a power of two: the ulp below it is halved
  const uint64_t eb = hb & 0x7ff0000000000000ULL;
  const double half_ulp = DBL(eb - (53ULL << 52));  // ulp(hi) / 2
  const double tol = DBL(eb - (65ULL << 52));       // 2^-65 .. 2^-64 of |hi|
  return fabs(S(fabs(lo), half_ulp)) > tol;
}

BO_DDM_FN double log_fast(double x, bool* ok) {
  const uint64_t bits = BITS(x);
  int e = (int)((bits >> 52) & 0x7ff) - 1023;
  double f = DBL((bits & 0xfffffffffffffULL) | 0x3ff0000000000000ULL);
  if (f >= 1.5) {
    f = M(f, 0.5);
    e += 1;
  }
  const int i = (int)RINT(M(f, 128.0));
  const double d = S(f, M((double)i, 0x1p-7));
  const double* tb = kLogTab + 4 * (i - kLogLo);
  const DD t = mul_d(DD{TAB(tb), TAB(tb + 1)}, d);
  const double lch = TAB(tb + 2), lcl = TAB(tb + 3);
  const double th = t.hi, tl = t.lo;
  // log1p(t) = t - t^2/2 + t^3 P(t), P = 1/3 - t/4 + ... - t^7/10 (t^3 P is < 2^-17 of t)
  double P = F(th, -1.0 / 10.0, 1.0 / 9.0);
  P = F(th, P, -1.0 / 8.0);
  P = F(th, P, 1.0 / 7.0);
  P = F(th, P, -1.0 / 6.0);
  P = F(th, P, 1.0 / 5.0);
  P = F(th, P, -0.25);
  P = F(th, P, 1.0 / 3.0);
  const DD p2 = two_prod(th, th);
  const double small = F(M(th, p2.hi), P, S(S(tl, M(0.5, p2.lo)), M(th, tl)));
  // additions ordered by magnitude (x <= 1, so e <= 0): |e ln2| >= ln 2 > |log c|
  // for e < 0 (e ln2 = 0 for e = 0), and |e ln2 + log c| >= log(128/127) >
  // |t| >= |t - t^2/2| unless it is 0 (e = 0, c = 1): quick_two_sum is exact
  const DD el = two_prod((double)e, kLn2Hi);
  const DD s1 = quick_two_sum(el.hi, lch);
  const DD s2 = quick_two_sum(th, M(-0.5, p2.hi));
  const DD s3 = quick_two_sum(s1.hi, s2.hi);
  double lo = A(s1.lo, s2.lo);
  lo = A(lo, s3.lo);
  lo = A(lo, el.lo);
  lo = F((double)e, kLn2Lo, lo);
  lo = A(lo, lcl);
  lo = A(lo, small);
  const DD r = quick_two_sum(s3.hi, lo);
  *ok = round_safe(r.hi, r.lo);
  return r.hi;
}

// sin / cos of the reduced argument r = a - k pi/2 (a double-double), fast path
BO_DDM_FN void sincos_fast_reduced(DD r, int k, double* sn, double* cs, bool* ok) {
  const double jd = RINT(M(r.hi, 64.0));
  const int j = (int)jd;
  const DD dl = two_sum(S(r.hi, M(jd, 0x1p-6)), r.lo);
  const double dh = dl.hi, dlo = dl.lo;
  const DD p = two_prod(dh, dh);
  const double z = p.hi;
  // sin d = dh + [dlo + dh z ps],        ps = -1/6 + z/120 - z^2/5040 + z^3/362880
  // cos d - 1 = -z/2 + [-p.lo/2 - dh dlo + z^2 pc],  pc = 1/24 - z/720 + z^2/40320 - z^3/3628800
  double ps = F(z, 1.0 / 362880.0, -1.0 / 5040.0);
  ps = F(z, ps, 1.0 / 120.0);
  ps = F(z, ps, -1.0 / 6.0);
  const double sdt = F(M(dh, z), ps, dlo);
  double pc = F(z, -1.0 / 3628800.0, 1.0 / 40320.0);
  pc = F(z, pc, -1.0 / 720.0);
  pc = F(z, pc, 1.0 / 24.0);
  const double cmh = M(-0.5, z);
  const double cml = F(M(z, z), pc, S(M(-0.5, p.lo), M(dh, dlo)));
  const int aj = j < 0 ? -j : j;
  const double* tb = kTrigTab + 4 * aj;
  double s0h = TAB(tb), s0l = TAB(tb + 1);
  const double c0h = TAB(tb + 2), c0l = TAB(tb + 3);
  if (j < 0) {
    s0h = -s0h;
    s0l = -s0l;
  }
  // sin r = S0 + C0 sin d + S0 (cos d - 1).  The additions are ordered by
  // magnitude, so the error-free quick_two_sum suffices: for j != 0,
  // |S0| >= sin(1/64) > |C0 d| (|d| <= 1/128) and |S0 + C0 d| >= sin(1/128) >
  // |S0 (cos d - 1)|; for j = 0, S0 = 0 (quick_two_sum(0, b) is exact).
  const DD u = two_prod(c0h, dh), v = two_prod(s0h, cmh);
  DD t1 = quick_two_sum(s0h, u.hi);
  DD t2 = quick_two_sum(t1.hi, v.hi);
  double lo = A(A(t1.lo, t2.lo), A(u.lo, v.lo));
  lo = A(lo, s0l);
  lo = F(c0h, sdt, lo);
  lo = F(c0l, dh, lo);
  lo = F(s0h, cml, lo);
  lo = F(s0l, cmh, lo);
  const DD sr = quick_two_sum(t2.hi, lo);
  // cos r = C0 - S0 sin d + C0 (cos d - 1): C0 >= cos(51/64) > 0.69 dominates
  const DD u2 = two_prod(s0h, dh), v2 = two_prod(c0h, cmh);
  t1 = quick_two_sum(c0h, -u2.hi);
  t2 = quick_two_sum(t1.hi, v2.hi);
  lo = A(A(t1.lo, t2.lo), S(v2.lo, u2.lo));
  lo = A(lo, c0l);
  lo = F(-s0h, sdt, lo);
  lo = F(-s0l, dh, lo);
  lo = F(c0h, cml, lo);
  lo = F(c0l, cmh, lo);
  const DD cr = quick_two_sum(t2.hi, lo);
  *ok = round_safe(sr.hi, sr.lo) && round_safe(cr.hi, cr.lo);
  switch (k & 3) {
    case 0: *sn = sr.hi; *cs = cr.hi; break;
    case 1: *sn = cr.hi; *cs = -sr.hi; break;
    case 2: *sn = -sr.hi; *cs = -cr.hi; break;
    default: *sn = -cr.hi; *cs = sr.hi; break;
  }
}

BO_DDM_FN void sincos_fast(double a, double* sn, double* cs, bool* ok) {
  const double kd = RINT(M(a, kTwoOverPi));
  DD r = add(DD{a, 0.0}, neg(two_prod(kd, kPio2_1)));  // accurate adds: r may be ~1e-16 (a near k pi/2)
  r = add(r, neg(two_prod(kd, kPio2_2)));
  r = add_d(r, -M(kd, kPio2_3));
  sincos_fast_reduced(r, (int)kd, sn, cs, ok);
}

// The Box-Muller angle a = fl(C u2), C = fl(2 pi), u2 = i 2^-53 in [0, 1)
// (rng.hpp:37-49), reduced without a three-part pi/2.  With kd = rint(4 u2)
// and d = u2 - kd/4 (exact: both are multiples of 2^-53 and |d| <= 1/8),
//   a = C u2 + e,  e = -(C u2 - a) = -fma(C, u2, -a)   (exact),
//   r = a - kd pi/2 = C d + e + kd (C - 2 pi)/4,
// with C d exact as two_prod(C, d) and (C - 2 pi)/4 as a double-double
// (kBmQ): two exact two_sums and three small terms, error below 2^-100 |r|
// (|r| >= 6e-17 unless a = 0, where r = 0 exactly), where the general
// reduction spends three double-double additions.  Same k as the general
// reduction up to ties, so the results are the same correctly rounded values.
constexpr double kBmC = 6.283185307179586476925286766559;
constexpr double kBmQHi = -0x1.1a62633145c07p-54, kBmQLo = 0x1.f1976b7ed8fbcp-110;  // (kBmC - 2 pi) / 4
BO_DDM_FN void sincos_bm_fast(double u2, double* sn, double* cs, bool* ok) {
  const double a = M(kBmC, u2);
  const double kd = RINT(M(u2, 4.0));
  const double d = S(u2, M(kd, 0.25));
  const double e = -F(kBmC, u2, -a);
  const DD p = two_prod(kBmC, d);
  const DD s1 = two_sum(p.hi, e);
  const DD s2 = two_sum(s1.hi, M(kd, kBmQHi));  // kd <= 4: the product is exact
  double lo = A(s1.lo, s2.lo);
  lo = A(lo, p.lo);
  lo = F(kd, kBmQLo, lo);
  sincos_fast_reduced(quick_two_sum(s2.hi, lo), (int)kd, sn, cs, ok);
}

// correctly rounded log / sincos: fast path, full precision where the fast
// result's rounding is not certain
BO_DDM_FN double log_cr(double x) {
  bool ok;
  const double y = log_fast(x, &ok);
  return ok ? y : log_rn(x);
}
BO_DDM_FN void sincos_cr(double a, double* sn, double* cs) {
  bool ok;
  sincos_fast(a, sn, cs, &ok);
  if (!ok) sincos_rn(a, sn, cs);
}
// sin / cos of the Box-Muller angle fl(kBmC u2), correctly rounded
BO_DDM_FN void sincos_bm_cr(double u2, double* sn, double* cs) {
  bool ok;
  sincos_bm_fast(u2, sn, cs, &ok);
  if (!ok) sincos_rn(M(kBmC, u2), sn, cs);
}

}  // namespace ddm
}  // namespace bo
