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
#include "fpm_philox.cuh"

namespace fpm {

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
