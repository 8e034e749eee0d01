// bo_cost.cpp — the reference's per-restart-cycle cost model
// (proj/include/blkorth/cost_model.hpp:9-39, proj/src/cost_model.cpp:38-111):
// exact integer evaluation of the tabulated flop / latency / volume / storage
// formulas for standard GMRES, s-step BCGS2 and the sketched schemes.  Host
// only; the comparator row of SURVEY.md §8(f)4.  Error texts are the
// reference's (InvalidScheme).
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/bo_cuda.h"

namespace bo {
namespace host {
int set_st(bo_status* st, int code, long long index, double pivot, const char* fmt, ...);
void ok_st(bo_status* st);
}  // namespace host
}  // namespace bo

namespace {

struct NotInt {
  std::string what;
};

int64_t exact_div(int64_t num, int64_t den, const char* what) {  // cost_model.cpp:30-35
  if (den == 0 || num % den != 0)
    throw NotInt{std::string("cost formula '") + what + "' does not evaluate to an integer for these parameters"};
  return num / den;
}

}  // namespace

extern "C" int bo_cost_eval(int scheme, int64_t n, int64_t m, int64_t s, int64_t shat, int64_t mhat,
                            bo_cost_result* out, bo_status* st) {
  using bo::host::set_st;
  bo::host::ok_st(st);
  *out = bo_cost_result{};
  if (scheme < BO_COST_STANDARD || scheme > BO_COST_SKETCH_EQ_M)
    return set_st(st, BO_INVALID, 0, 0.0, "unknown cost scheme");
  if (n < 1 || m < 1) return set_st(st, BO_INVALID, 0, 0.0, "need positive n and m");
  switch (scheme) {  // shat forced as in cost_model.cpp:45-51
    case BO_COST_STANDARD: shat = 1; break;
    case BO_COST_SSTEP:
    case BO_COST_SKETCH_EQ_S: shat = s; break;
    case BO_COST_SKETCH_EQ_M: shat = m; break;
    default: break;
  }
  if (mhat <= 0) mhat = 2 * (shat + 1);
  const bool s_divides = s >= 1 && s <= m && m % s == 0;
  try {
    switch (scheme) {
      case BO_COST_STANDARD:
        out->flops_total = 2 * n * m * m;
        out->flops_second = out->flops_total;
        out->latency = 4 * m;
        out->volume = n * m * (2 * m + 4);
        out->storage = n * m;
        break;
      case BO_COST_SSTEP:
      case BO_COST_SKETCH_EQ_S: {
        if (!s_divides) return set_st(st, BO_INVALID, 0, 0.0, "need s | m with 1 <= s <= m");
        const int64_t ms = exact_div(m, s, "m/s");
        out->flops_total = 2 * n * m * ms * (s + 1);
        out->flops_second = out->flops_total;
        out->latency = 4 * ms;
        out->volume = n * ms * (2 * m + 4 + 4 * s + (scheme == BO_COST_SKETCH_EQ_S ? mhat : 0));
        out->storage = scheme == BO_COST_SKETCH_EQ_S ? n * (m + mhat) : n * m;
        break;
      }
      case BO_COST_SKETCH_BETWEEN: {
        if (!(s >= 1 && s < shat && shat < m)) return set_st(st, BO_INVALID, 0, 0.0, "need 1 <= s < shat < m");
        if (shat % s != 0 || m % shat != 0) return set_st(st, BO_INVALID, 0, 0.0, "need s | shat and shat | m");
        const int64_t ms = exact_div(m, s, "m/s"), mh = exact_div(m, shat, "m/shat");
        out->flops_total = 2 * n * m * ms * (s + 1);
        out->flops_second = 2 * n * m * mh * (shat + 1);
        out->latency = ms + 3 * mh;
        out->volume = n * ms * (m + 2 + 2 * s + mhat) + n * mh * (m + 2 + 4 * shat);
        out->storage = n * (m + mhat);
        break;
      }
      case BO_COST_SKETCH_EQ_M: {
        if (!s_divides) return set_st(st, BO_INVALID, 0, 0.0, "need s | m with 1 <= s <= m");
        const int64_t ms = exact_div(m, s, "m/s");
        out->flops_total = 5 * n * m * ms * (s + 1);
        out->flops_second = 2 * n * m * m;
        out->latency = ms + 1;
        out->volume = exact_div(n * ms * (m + 2 * mhat + 4 + 4 * s), 2, "volume/2") + 2 * n * m;
        out->storage = n * (m + mhat);
        break;
      }
    }
  } catch (const NotInt& e) {
    *out = bo_cost_result{};
    return set_st(st, BO_INVALID, 0, 0.0, "%s", e.what.c_str());
  }
  return BO_OK;
}
