// mt64_jump.h — MT19937-64 jump-ahead (see mt64_jump.cpp)
#pragma once
#include <cstdint>

namespace bo {
namespace mt64 {
bool ready();
int poly_words();    // 312
int prefix_words();  // 20248: g[0 .. 19936+311]
// g[0..prefix_words()) = untempered words following the first twist
void prefix(uint64_t seed, uint64_t* g);
// x^J mod phi, poly_words() words
void jump_poly(uint64_t J, uint64_t* out);
// x^(J0 + c L) mod phi for c < count, count*poly_words() words
void jump_polys_strided(uint64_t J0, uint64_t L, uint64_t count, uint64_t* out);
// host reference: window g[J .. J+311]
void jump_window_host(uint64_t seed, uint64_t J, uint64_t* w);
}  // namespace mt64
}  // namespace bo
