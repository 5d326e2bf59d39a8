// prng.cuh -- the reference's counter-based PRNG on the device.
//
// bits(seed, stream, counter) = mix(mix(mix(seed+G) ^ mix(stream+SS)) ^ mix(counter+CS))
// with mix = splitmix64's finalizer (prng.py:50-81).  The seed/stream half is
// counter independent, so every chain precomputes h_sc once (the same
// factorisation prng.py:149 uses) and a draw costs two mix64 rounds.
#pragma once
#include "dmath.cuh"

namespace fsmc {

constexpr uint64_t MIX_A = 0xBF58476D1CE4E5B9ULL;
constexpr uint64_t MIX_B = 0x94D049BB133111EBULL;
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t STREAM_SALT = 0xC2B2AE3D27D4EB4FULL;
constexpr uint64_t COUNTER_SALT = 0x165667B19E3779F9ULL;
constexpr double INV_2_53 = 1.0 / 9007199254740992.0;

// x * c mod 2^64 in three 32-bit multiplies chained into the high word
// (FSMC_MUL3; the compiler's own form adds the cross terms separately)
#ifndef FSMC_MUL3
#define FSMC_MUL3 0
#endif
FSMC_HD uint64_t mulc64(uint64_t x, uint64_t c) {
#if defined(__CUDA_ARCH__) && FSMC_MUL3
  const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
  const uint32_t cl = (uint32_t)c, ch = (uint32_t)(c >> 32);
  uint32_t rl, rh;
  asm("{\n\t"
      ".reg .u64 t;\n\t"
      "mul.wide.u32 t, %2, %4;\n\t"
      "mov.b64 {%0, %1}, t;\n\t"
      "mad.lo.u32 %1, %2, %5, %1;\n\t"
      "mad.lo.u32 %1, %3, %4, %1;\n\t"
      "}"
      : "=r"(rl), "=r"(rh)
      : "r"(xl), "r"(xh), "r"(cl), "r"(ch));
  return ((uint64_t)rh << 32) | rl;
#else
  return x * c;
#endif
}

FSMC_HD uint64_t mix64(uint64_t x) {
  x = mulc64(x ^ (x >> 30), MIX_A);
  x = mulc64(x ^ (x >> 27), MIX_B);
  return x ^ (x >> 31);
}

// counter-independent half of _bits (prng.py:64-74)
FSMC_HD uint64_t hash_seed_stream(uint64_t seed, uint64_t stream) {
  return mix64(mix64(seed + GOLDEN) ^ mix64(stream + STREAM_SALT));
}

// prng.py:75-81
FSMC_HD uint64_t bits(uint64_t hsc, uint64_t counter) {
  return mix64(hsc ^ mix64(counter + COUNTER_SALT));
}

// prng.py:97-100
FSMC_HD double uniform(uint64_t hsc, uint64_t counter) {
  return (double)(bits(hsc, counter) >> 11) * INV_2_53;
}

// prng.py:103-111: ndtri((b + 0.5) * 2^-53); the +0.5 rounds in fp64
FSMC_HD double normal(uint64_t hsc, uint64_t counter) {
  uint64_t b = bits(hsc, counter) >> 11;
  return ndtri(((double)b + 0.5) * INV_2_53);
}

// prng.py:84-94: child stream i of a parent stream
FSMC_HD uint64_t split_stream(uint64_t parent_stream, uint64_t i) {
  return mix64(parent_stream * GOLDEN + i + 1);
}

}  // namespace fsmc
