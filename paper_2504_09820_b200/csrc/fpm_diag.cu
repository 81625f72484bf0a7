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

// ||A||_2 = max |lambda| of a Hermitian matrix (the reference: np.linalg.norm(A, 2),
// experiments.py:246-256 / solvers.py:289-294's a_norm): one warp per matrix
// runs N Lanczos steps in binary64 (three vectors in registers, lanes own
// entries lane + 32 j; A streamed from L2 every step) and then brackets the
// extreme eigenvalues of the real tridiagonal (alpha, beta) by 32-way
// multisection on its Sturm count (one trial shift per lane).  No
// reorthogonalisation: ghost copies of converged Ritz values do not move the
// extreme ones, which is all that is read.  A start vector with every
// component non-zero and of varied phase; an exact invariant subspace
// (beta = 0) ends the recurrence early.
__global__ void __launch_bounds__(128) fpm_hnorm_kernel(const double2* __restrict__ A, long T, int N,
                                                        double* __restrict__ out) {
  __shared__ double s_al[4][128], s_be[4][128];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long t = (long)blockIdx.x * 4 + wl;
  if (t >= T) return;
  double* al = s_al[wl];
  double* be = s_be[wl];  // be[k] couples steps k-1 and k (be[0] unused)
  const double2* At = A + t * (long)N * N;
  double2 v[4], vp[4], w[4];
  double nn = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = lane + 32 * j;
    const double ph = 0.7 * k + 0.1 * k * k;  // varied phases, unit moduli
    v[j] = k < N ? make_double2(cos(ph), sin(ph)) : make_double2(0.0, 0.0);
    vp[j] = make_double2(0.0, 0.0);
    nn += v[j].x * v[j].x + v[j].y * v[j].y;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
  const double inv0 = 1.0 / sqrt(nn);
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = make_double2(v[j].x * inv0, v[j].y * inv0);
  double beta = 0.0, amax = 0.0;
  int K = 0;
#pragma unroll 1
  for (int step = 0; step < N; ++step) {
    // w = A v
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int row = 0; row < N; ++row) {
      const double2* ar = At + (long)row * N;
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = lane + 32 * j;
        if (k < N) {
          const double2 a = ar[k];
          sr += a.x * v[j].x - a.y * v[j].y;
          si += a.x * v[j].y + a.y * v[j].x;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        sr += __shfl_xor_sync(0xffffffffu, sr, o);
        si += __shfl_xor_sync(0xffffffffu, si, o);
      }
      if ((row & 31) == lane) {
        const double2 e = make_double2(sr, si);
        switch (row >> 5) {
          case 0: w[0] = e; break;
          case 1: w[1] = e; break;
          case 2: w[2] = e; break;
          default: w[3] = e; break;
        }
      }
    }
    double a = 0.0;  // alpha = Re(v^H w)
#pragma unroll
    for (int j = 0; j < 4; ++j) a += v[j].x * w[j].x + v[j].y * w[j].y;
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    double b2 = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      w[j].x -= a * v[j].x + beta * vp[j].x;
      w[j].y -= a * v[j].y + beta * vp[j].y;
      b2 += w[j].x * w[j].x + w[j].y * w[j].y;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) b2 += __shfl_xor_sync(0xffffffffu, b2, o);
    if (lane == 0) {
      al[step] = a;
      be[step] = beta;
    }
    K = step + 1;
    amax = fmax(amax, fabs(a));
    const double bn = sqrt(b2);
    if (!(bn > 1e-14 * fmax(amax, 1e-300)) || !isfinite(bn)) break;  // invariant subspace (or non-finite input)
    const double ib = 1.0 / bn;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      vp[j] = v[j];
      v[j] = make_double2(w[j].x * ib, w[j].y * ib);
    }
    beta = bn;
  }
  __syncwarp();
  // Gershgorin bracket of the tridiagonal, then multisection on the Sturm
  // count (number of eigenvalues below x) for the largest and the smallest
  double lo = 0.0, hi = 0.0;
  for (int k = lane; k < K; k += 32) {
    const double r = (k > 0 ? fabs(be[k]) : 0.0) + (k + 1 < K ? fabs(be[k + 1]) : 0.0);
    lo = (k == lane) ? al[k] - r : fmin(lo, al[k] - r);
    hi = (k == lane) ? al[k] + r : fmax(hi, al[k] + r);
  }
  if (lane >= K) {
    lo = al[0];
    hi = al[0];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  auto below = [&](double x) -> int {  // eigenvalues of the tridiagonal < x
    int c = 0;
    double d = 1.0;
    for (int k = 0; k < K; ++k) {
      const double b = k > 0 ? be[k] : 0.0;
      d = (al[k] - x) - (k > 0 ? b * b / d : 0.0);
      if (d == 0.0) d = -1e-300;
      c += d < 0.0;
    }
    return c;
  };
  double res[2];
#pragma unroll 1
  for (int which = 0; which < 2; ++which) {  // 0: largest (count(x) < K below it), 1: smallest (count(x) >= 1 above it)
    double a = lo, b = hi;
#pragma unroll 1
    for (int round = 0; round < 14; ++round) {
      const double x = a + (b - a) * (lane + 1) / 33.0;
      const int c = below(x);
      const bool left = which == 0 ? (c < K) : (c < 1);  // the wanted eigenvalue is >= x
      const unsigned m = __ballot_sync(0xffffffffu, left);
      const int nleft = __popc(m);  // monotone: the first nleft trial points lie at or below it
      const double na = nleft > 0 ? a + (b - a) * nleft / 33.0 : a;
      const double nb = nleft < 32 ? a + (b - a) * (nleft + 1) / 33.0 : b;
      a = na;
      b = nb;
    }
    res[which] = 0.5 * (a + b);
  }
  if (lane == 0) out[t] = fmax(fabs(res[0]), fabs(res[1]));
}

}  // namespace fpm

extern "C" int fpm_herm_norm2(const double* A, int64_t T, int32_t N, double* norms, void* stream) {
  using namespace fpm;
  if (T < 0 || N < 1 || (T > 0 && (!A || !norms))) return FPM_EINVAL;
  if (N > 128) return FPM_EUNSUPPORTED;
  if (reinterpret_cast<uintptr_t>(A) & 15) return FPM_EINVAL;
  if (T == 0) return FPM_OK;
  const long grid = (T + 3) / 4;
  if (grid > 0x7fffffffL) return FPM_EUNSUPPORTED;
  fpm_hnorm_kernel<<<(unsigned)grid, 128, 0, (cudaStream_t)stream>>>(reinterpret_cast<const double2*>(A), T, N, norms);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}

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
