// GPU input generation (the reference's simulate_trials,
// detect.py:189-214, channel.py:138-161, rng.py:19-39): per-trial random
// streams on the device, keyed like the reference's substreams by
// (seed, context, point, trial), so a trial's draws do not depend on the
// batch, the chunking or the GPU it is generated on.
//
// Generator: Philox4x32-10 (Salmon et al., SC'11) with key (seed low word,
// seed high word ^ context << 16 ^ point) and counter (element, stream,
// trial low, trial high).  Uniforms use 53 bits of two 32-bit outputs, in
// (0, 1]; normals are Box-Muller pairs like rng.py:33-39.  The reference's
// NumPy Philox / libm stream is not reproduced bit for bit (SURVEY.md 8(f):
// distribution-level parity), so the Kronecker colouring and y = H s + n are
// composed on the device by the Python layer (channel.py) from these draws.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/fpmimo_b200.h"
#include "fpm_common.cuh"

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

// per trial: W (M, N) CN(0, 1/M) (channel.py:150-151), bits (nbits) uniform
// {0, 1} (detect.py:207), unit complex normals for the noise (M) and, when
// requested, for the CSI perturbation (M, N) (channel.py:206-219)
__global__ void fpm_gen_kernel(uint32_t k0, uint32_t k1, long trial0, long T, int M, int N, int nbits,
                               double2* W, uint8_t* bits, double2* noise, double2* csi) {
  const long per = (long)M * N;
  const long stride = (long)gridDim.x * blockDim.x;
  const double sc = 1.0 / sqrt(2.0 * M);
  for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < T * per; q += stride) {
    const long t = q / per;
    const uint32_t e = (uint32_t)(q - t * per);
    const double2 g = cnormal(k0, k1, kStreamW, e, (uint64_t)(trial0 + t));
    W[q] = make_double2(g.x * sc, g.y * sc);
    if (csi) csi[q] = cnormal(k0, k1, kStreamCsi, e, (uint64_t)(trial0 + t));
  }
  for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < T * M; q += stride) {
    const long t = q / M;
    noise[q] = cnormal(k0, k1, kStreamNoise, (uint32_t)(q - t * M), (uint64_t)(trial0 + t));
  }
  for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < T * nbits; q += stride) {
    const long t = q / nbits;
    const uint32_t e = (uint32_t)(q - t * nbits);
    const Ph4 r = philox4x32_10(Ph4{e, kStreamBits, (uint32_t)(trial0 + t), (uint32_t)((trial0 + t) >> 32)}, k0, k1);
    bits[q] = (uint8_t)(r.x >> 31);
  }
}

}  // namespace fpm

using namespace fpm;

extern "C" int fpm_gen_trials(uint64_t seed, int32_t context, int32_t point, int64_t trial0, int64_t T, int32_t M,
                              int32_t N, int32_t nbits, double* W, uint8_t* bits, double* noise, double* csi,
                              void* stream) {
  if (T < 0 || M < 1 || N < 1 || nbits < 0 || trial0 < 0 || (T > 0 && (!W || !noise || (nbits && !bits))))
    return FPM_EINVAL;
  if (context < 0 || context >= (1 << 12) || point < 0 || point >= (1 << 16)) return FPM_EINVAL;  // rng.py:21-26
  if (T == 0) return FPM_OK;
  const uint32_t k0 = (uint32_t)seed;
  const uint32_t k1 = (uint32_t)(seed >> 32) ^ ((uint32_t)context << 16) ^ (uint32_t)point;
  const long work = T * (long)M * N;
  const int tpb = 256;
  const long grid = std::min<long>((work + tpb - 1) / tpb, 148L * 16);
  fpm_gen_kernel<<<(unsigned)grid, tpb, 0, (cudaStream_t)stream>>>(
      k0, k1, trial0, T, M, N, nbits, reinterpret_cast<double2*>(W), bits, reinterpret_cast<double2*>(noise),
      reinterpret_cast<double2*>(csi));
  count_launch();
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}
