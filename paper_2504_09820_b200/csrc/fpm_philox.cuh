// Keyed Philox4x32-10 draws shared by the generators (fpm_gen.cu raw
// draws, fpm_sim.cu fused link model): Salmon et al., SC'11, key (seed low
// word, seed high word ^ context << 16 ^ point), counter (element, stream,
// trial low, trial high); uniforms from 53 bits of two outputs in (0, 1];
// normals as Box-Muller pairs (rng.py:33-39).
#pragma once
#include <stdint.h>

namespace fpm {

struct Ph4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ Ph4 philox4x32_10(Ph4 c, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = Ph4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += W0;
    k1 += W1;
  }
  return c;
}

// 53-bit uniform in (0, 1]
__device__ __forceinline__ double u01(uint32_t a, uint32_t b) {
  const uint64_t v = ((uint64_t)a << 21) ^ (uint64_t)(b >> 11);
  return ((double)(v & ((1ULL << 53) - 1)) + 1.0) * (1.0 / 9007199254740992.0);
}

// complex standard normal (re, im ~ N(0, 1)) of (stream, element) of a trial
__device__ __forceinline__ double2 cnormal(uint32_t k0, uint32_t k1, uint32_t stream, uint32_t elem, uint64_t trial) {
  const Ph4 r = philox4x32_10(Ph4{elem, stream, (uint32_t)trial, (uint32_t)(trial >> 32)}, k0, k1);
  const double u1 = u01(r.x, r.y), u2 = u01(r.z, r.w);
  const double rad = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  return make_double2(rad * c, rad * s);
}

enum { kStreamW = 1, kStreamBits = 2, kStreamNoise = 3, kStreamCsi = 4 };

// uniform payload bit `elem` of a trial (detect.py:207)
__device__ __forceinline__ uint32_t gen_bit(uint32_t k0, uint32_t k1, uint32_t elem, uint64_t trial) {
  return philox4x32_10(Ph4{elem, kStreamBits, (uint32_t)trial, (uint32_t)(trial >> 32)}, k0, k1).x >> 31;
}

}  // namespace fpm
