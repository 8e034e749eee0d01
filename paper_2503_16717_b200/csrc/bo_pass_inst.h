// bo_pass_inst.h — entry points of the pass-kernel instantiation units.
// Each function returns the pass_kernel specialisation for a pass kind
// (nullptr when the combination is not instantiated).
#pragma once
#include <cuda.h>

#include "bo_common.cuh"

namespace bo {
namespace host {
typedef void (*PassFn)(const PassArgs, const CUtensorMap, const CUtensorMap, const CUtensorMap);
PassFn pass_fn_nt1_t256(int kind);
PassFn pass_fn_nt2_t256(int kind);
PassFn pass_fn_kc6_t256(int kind);
PassFn pass_fn_kc11_t256(int kind);
PassFn pass_fn_kc16_t256(int kind);
PassFn pass_fn_kc13_t256(int kind);
PassFn pass_fn_kc13_t128(int kind);
PassFn pass_fn_kc13_t64(int kind);
PassFn pass_fn_nt1_t128(int kind);
PassFn pass_fn_nt1_t64(int kind);
PassFn pass_fn_nt2_t128(int kind);
PassFn pass_fn_nt2_t64(int kind);
PassFn pass_fn_kc6_t128(int kind);
PassFn pass_fn_kc6_t64(int kind);
PassFn pass_fn_kc11_t128(int kind);
PassFn pass_fn_kc11_t64(int kind);
PassFn pass_fn_kc16_t128(int kind);
PassFn pass_fn_kc16_t64(int kind);
PassFn pass_fn_exact(int nt);
}  // namespace host
}  // namespace bo
