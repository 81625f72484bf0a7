// Convergence-study diagnostics on the device (off the detection hot path):
// the true-residual gap of every recorded sweep,
//   gap_i = || b - A x_i - r_i ||_2 / scale        (solvers.py:289-294, 375-377)
// from the iterates / residual vectors run_batch records (fpm_cg_ex), in one
// launch over all sweeps instead of a host loop of batched matvecs.
//
// One warp per (sweep, realization): the lanes split a row's columns
// (coalesced 16-byte loads of A), a butterfly sum gives every lane the row's
// A x, and lane (row % 32) keeps the row's residual entry; the 2-norm is
// linalg.py:122-134's scaled form (cgw_norm2).  Binary64 throughout, separately
// rounded; the reference forms A x with BLAS, so parity is a tolerance.
#include "../../include/fpmimo_b200.h"
#include "fpm_cgw.cuh"

namespace fpm {

__global__ void __launch_bounds__(128) fpm_gaps_kernel(const double2* __restrict__ A, const double2* __restrict__ b,
                                                       const double2* __restrict__ xit, const double2* __restrict__ rit,
                                                       const double* __restrict__ scale, long T, int N, int it1,
                                                       double* __restrict__ gaps) {
  const long w = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= (long)(it1 - 1) * T) return;
  const int i = 1 + (int)(w / T);
  const long t = w - (long)(i - 1) * T;
  const double2* At = A + t * (long)N * N;
  const double2* bt = b + t * (long)N;
  const double2* xv = xit + ((long)i * T + t) * N;
  const double2* rv = rit + ((long)i * T + t) * N;
  double2 xs[4], v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = lane + 32 * j;
    xs[j] = k < N ? xv[k] : make_double2(0.0, 0.0);
    v[j] = make_double2(0.0, 0.0);
  }
#pragma unroll 1
  for (int row = 0; row < N; ++row) {
    const double2* ar = At + (long)row * N;
    double sr = 0.0, si = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = lane + 32 * j;
      if (k < N) {
        const double2 a = ar[k];
        sr += a.x * xs[j].x - a.y * xs[j].y;
        si += a.x * xs[j].y + a.y * xs[j].x;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      sr += __shfl_xor_sync(0xffffffffu, sr, o);
      si += __shfl_xor_sync(0xffffffffu, si, o);
    }
    if ((row & 31) == lane) {
      const double2 bb = bt[row], rr = rv[row];
      const double2 e = make_double2(bb.x - sr - rr.x, bb.y - si - rr.y);
      switch (row >> 5) {  // static register indices
        case 0: v[0] = e; break;
        case 1: v[1] = e; break;
        case 2: v[2] = e; break;
        default: v[3] = e; break;
      }
    }
  }
  const double nrm = cgw_norm2<4>(v);
  if (lane == 0) gaps[(long)i * T + t] = nrm / scale[t];
}

}  // namespace fpm

extern "C" int fpm_residual_gaps(const double* A, const double* b, const double* iterates,
                                 const double* residual_vectors, const double* scale, int64_t T, int32_t N,
                                 int32_t iters, double* gaps, void* stream) {
  using namespace fpm;
  if (T < 0 || N < 1 || iters < 0 || (T > 0 && iters > 0 && (!A || !b || !iterates || !residual_vectors || !scale || !gaps)))
    return FPM_EINVAL;
  if (N > 128) return FPM_EUNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(iterates) |
       reinterpret_cast<uintptr_t>(residual_vectors)) & 15)
    return FPM_EINVAL;
  if (T == 0 || iters == 0) return FPM_OK;
  const long warps = (long)iters * T;
  const long grid = (warps + 3) / 4;
  if (grid > 0x7fffffffL) return FPM_EUNSUPPORTED;
  fpm_gaps_kernel<<<(unsigned)grid, 128, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const double2*>(A), reinterpret_cast<const double2*>(b), reinterpret_cast<const double2*>(iterates),
      reinterpret_cast<const double2*>(residual_vectors), scale, T, N, iters + 1, gaps);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}
