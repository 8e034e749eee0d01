// Host build of the device double-double log / sincos (bo_ddmath.cuh) for the
// CPU tests (tests/test_ddmath.py): the same source the sketch generator
// compiles for sm_100a, built here with g++ -ffp-contract=off.
#include <cmath>
#include <cstdint>
#include <random>

#include "../../paper_2503_16717_b200/csrc/bo_ddmath.cuh"

extern "C" {
double ddm_log(double x) { return bo::ddm::log_rn(x); }
// fast path with its certainty flag, and the combined (what the device uses)
void ddm_fast_n(const double* x, const double* a, double* lg, double* s, double* c, unsigned char* okl,
                unsigned char* oks, long n) {
  for (long i = 0; i < n; ++i) {
    bool o1, o2;
    lg[i] = bo::ddm::log_fast(x[i], &o1);
    bo::ddm::sincos_fast(a[i], s + i, c + i, &o2);
    okl[i] = o1;
    oks[i] = o2;
  }
}
void ddm_cr_n(const double* x, const double* a, double* lg, double* s, double* c, long n) {
  for (long i = 0; i < n; ++i) {
    lg[i] = bo::ddm::log_cr(x[i]);
    bo::ddm::sincos_cr(a[i], s + i, c + i);
  }
}
void ddm_sincos(double a, double* s, double* c) { bo::ddm::sincos_rn(a, s, c); }
// the Box-Muller-specific reduction (device generator): fast path with its
// certainty flag, and the combined function, both from u2
void ddm_bm_fast_n(const double* u2, double* s, double* c, unsigned char* ok, long n) {
  for (long i = 0; i < n; ++i) {
    bool o;
    bo::ddm::sincos_bm_fast(u2[i], s + i, c + i, &o);
    ok[i] = o;
  }
}
void ddm_bm_cr_n(const double* u2, double* s, double* c, long n) {
  for (long i = 0; i < n; ++i) bo::ddm::sincos_bm_cr(u2[i], s + i, c + i);
}
void ddm_log_n(const double* x, double* y, long n) {
  for (long i = 0; i < n; ++i) y[i] = bo::ddm::log_rn(x[i]);
}
void ddm_sincos_n(const double* a, double* s, double* c, long n) {
  for (long i = 0; i < n; ++i) bo::ddm::sincos_rn(a[i], s + i, c + i);
}
void glibc_log_n(const double* x, double* y, long n) {
  for (long i = 0; i < n; ++i) y[i] = std::log(x[i]);
}
void glibc_sincos_n(const double* a, double* s, double* c, long n) {
  for (long i = 0; i < n; ++i) {
    s[i] = std::sin(a[i]);
    c[i] = std::cos(a[i]);
  }
}
// Box-Muller pairs from std::mt19937_64(seed) exactly as rng.hpp:37-49 draws
// them; which = 0: glibc log/sin/cos (the reference), 1: bo_ddmath
void box_muller_n(uint64_t seed, long npairs, int which, double* out) {
  std::mt19937_64 g(seed);
  for (long t = 0; t < npairs; ++t) {
    const double u1 = ((double)(g() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = (double)(g() >> 11) * 0x1.0p-53;
    const double a = 6.283185307179586476925286766559 * u2;
    double lg, s, c;
    if (which == 0) {
      lg = std::log(u1);
      s = std::sin(a);
      c = std::cos(a);
    } else {
      lg = bo::ddm::log_cr(u1);
      bo::ddm::sincos_cr(a, &s, &c);
    }
    const double r = std::sqrt(-2.0 * lg);
    out[2 * t] = r * c;
    out[2 * t + 1] = r * s;
  }
}
// Gaussian sketch Theta (n x mhat, column-major, scale 1/sqrt(mhat)) as
// sketch.cpp:30-35 fills it from Rng(rng_seed), with bo_ddmath's correctly
// rounded log / sin / cos: what the device generator must reproduce bit for bit
void theta_cr(uint64_t rng_seed, long n, long mhat, double* out) {
  std::mt19937_64 g(rng_seed);
  const double scale = 1.0 / std::sqrt((double)mhat);
  const long total = n * mhat;
  for (long q = 0; q < total; q += 2) {
    const double u1 = ((double)(g() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = (double)(g() >> 11) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * bo::ddm::log_cr(u1));
    double s, c;
    bo::ddm::sincos_cr(6.283185307179586476925286766559 * u2, &s, &c);
    out[q] = scale * (r * c);
    if (q + 1 < total) out[q + 1] = scale * (r * s);
  }
}
}
