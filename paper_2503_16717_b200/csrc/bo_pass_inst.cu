// bo_pass_inst.cu — one instantiation unit of the streaming pass engine.
// Compiled once per combination with -DBO_INST_NT=<1|2> or -DBO_INST_KC=<6|11|13|16>
// and -DBO_INST_T=<64|128> (or -DBO_INST_EXACT), so the build runs the heavy
// template instantiations in parallel.
#include "bo_internal.h"
#include "bo_pass.cuh"
#include "bo_pass_inst.h"

#define BO_CAT_(a, b, c, d) a##b##c##d
#define BO_CAT(a, b, c, d) BO_CAT_(a, b, c, d)

namespace bo {
namespace host {

#if defined(BO_INST_EXACT)
PassFn pass_fn_exact(int nt) {
  return nt == 1 ? (PassFn)pass_kernel<1, 64, 1, false, 0, false, false, SK_NONE, true, true>
                 : (PassFn)pass_kernel<2, 64, 1, false, 0, false, false, SK_NONE, true, true>;
}
#elif defined(BO_INST_NT)
PassFn BO_CAT(pass_fn_nt, BO_INST_NT, _t, BO_INST_T)(int kind) {
  switch (kind) {
#define X(nm, a, b, c, d, e, f, g) \
  case PK_##nm:                    \
    return pass_kernel<BO_INST_NT, BO_INST_T, a, b, c, d, e, f, g, false>;
    BO_PASS_KINDS(X)
#undef X
  }
  return nullptr;
}
#elif defined(BO_INST_KC)
// triangular-solve passes specialised on the panel width (s = 5, 10, 12, 15; K = 13 is
// also the last 16-column block of the two-stage big panel at shat = 60)
PassFn BO_CAT(pass_fn_kc, BO_INST_KC, _t, BO_INST_T)(int kind) {
  constexpr int NT = BO_INST_KC <= 8 ? 1 : 2;
  switch (kind) {
#define X(nm, a, b, c, d, e, f, g)                                             \
  case PK_##nm:                                                                \
    if constexpr (a > 0 || c > 0)                                              \
      return pass_kernel<NT, BO_INST_T, a, b, c, d, e, f, g, false, BO_INST_KC>; \
    else                                                                       \
      return nullptr;
    BO_PASS_KINDS(X)
#undef X
  }
  return nullptr;
}
#else
#error "bo_pass_inst.cu needs BO_INST_EXACT, BO_INST_NT or BO_INST_KC"
#endif

}  // namespace host
}  // namespace bo
