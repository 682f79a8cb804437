// The INT4 -> INT8 DGQ dequantiser shared by the fused GEMM prologue and the
// standalone kernels:  W_s8 = S2 * (code - ZP)   (proj/src/format.cpp:129-130).
//
// Eight codes of one word share (S2, ZP).  Two codes are processed per 32-bit
// IMAD in separate 16-bit lanes:  code*S2 + (2048 - ZP*S2)  never exceeds
// 15*127 + 2047 < 2^16, and 2048 == 0 (mod 256), so the low byte of each lane
// is S2*(code-ZP) mod 256 — exactly the int8 value, because a valid layer keeps
// it inside [-127, 127] (clip_interval, proj/src/search.cpp:190-201).  Two
// PRMTs gather the low bytes into k order.
#pragma once
#include <cstdint>

namespace dgqk {

__device__ __forceinline__ uint32_t dq_bias2(uint32_t s2, uint32_t zp) {
  const uint32_t a = 2048u - zp * s2;
  return a | (a << 16);
}

// word nibble layout (kernels.h kNibblePos): nibble 2j = k j, nibble 2j+1 = k j+4,
// i.e. {0:k0, 1:k4, 2:k1, 3:k5, 4:k2, 5:k6, 6:k3, 7:k7}; lo = bytes k0..k3, hi = k4..k7.
__device__ __forceinline__ void dq_word(uint32_t w, uint32_t s2, uint32_t bias2, uint32_t& lo, uint32_t& hi) {
  const uint32_t m = 0x000F000Fu;
  const uint32_t v0 = (w & m) * s2 + bias2;
  const uint32_t v1 = ((w >> 4) & m) * s2 + bias2;
  const uint32_t v2 = ((w >> 8) & m) * s2 + bias2;
  const uint32_t v3 = ((w >> 12) & m) * s2 + bias2;
  lo = __byte_perm(v0, v2, 0x6240);  // (k0, k1, k2, k3)
  hi = __byte_perm(v1, v3, 0x6240);  // (k4, k5, k6, k7)
}

}  // namespace dgqk
