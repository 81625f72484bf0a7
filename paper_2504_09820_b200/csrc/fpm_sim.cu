// Fused input generator: the reference's link model
// simulate_trials (detect.py:189-214) -- Kronecker channel
// H = R_r^{1/2} W R_t^{1/2} (channel.py:138-161), optional imperfect CSI
// (channel.py:206-219), Gray QAM payload (detect.py:54-67) and
// y = H s + CN(0, sigma^2) (detect.py:87-93, 210-211) -- in ONE kernel that
// writes H, y, bits (and H_est, symbols) once.
//
// Draws: the same keyed Philox4x32-10 streams as fpm_gen_trials (W, bits,
// noise, CSI; fpm_gen.cu), so every trial's draws are those of
// fpm_gen_trials and do not depend on batching, chunking or the GPU.
//
// Colouring: the reference multiplies by the symmetric square roots of the
// exponential correlation matrices [R]_ij = zeta^|i-j| (O(M^2 N + M N^2) per
// trial).  Any factor F with F F^H = R gives the same distribution of
// H = F_r W F_t^T for i.i.d. circularly-symmetric Gaussian W (vec H ~
// CN(0, (R_t (x) R_r) / M) either way), and the lower Cholesky factor of an
// exponential correlation matrix is the AR(1) recursion
//     x_0 = w_0,  x_k = zeta x_{k-1} + sqrt(1 - zeta^2) w_k,
// restarting at every user block when block_diag_users.  So the colouring is
// two first-order recursions, O(M N): along the users inside a warp (an
// affine prefix scan over lane segments) and along the antennas in each
// lane's registers.  Parity with the reference generator is distribution
// level; tests pin the draws bit for bit and the colouring
// against a host restatement.
//
// Layout: one warp per trial; lane l owns the contiguous columns
// [l*cpl, (l+1)*cpl) (cpl = ceil(N/32)) of every antenna row; rows are
// produced in order m = 0..M-1, so each warp store of a row is one
// contiguous N*16-byte segment.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/fpmimo_b200.h"
#include "fpm_common.cuh"
#include "fpm_philox.cuh"

namespace fpm {

constexpr int kSimCplMax = 4;  // N <= 128; kernels for 1, 2, 4 columns per lane
constexpr int kSimRows = 4;    // antenna rows drawn ahead of their recursions

struct SimArgs {
  uint32_t k0, k1;
  long trial0, T;
  int M, N, cpl, bps, n_ue, block_diag;
  double zr, cr, zt, ct;  // AR(1) multiplier / innovation weight, receive / transmit side
  double wscale;          // 1 / sqrt(2 M): W ~ CN(0, 1/M)
  double nscale;          // sqrt(sigma^2 / 2)
  double cscale;          // sqrt(csi_var / 2), < 0: no CSI
  double lv[8];           // Gray levels per axis index (16-QAM: 4, 64-QAM: 8)
  double2* H;
  double2* Hest;
  double2* y;
  uint8_t* bits;
  double2* sym;
};

// (A, B) affine map x -> A x + B composed over lanes: inclusive scan
__device__ __forceinline__ void affine_scan(double& A, double2& B, int lane) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double pA = __shfl_up_sync(0xffffffffu, A, off);
    const double pBx = __shfl_up_sync(0xffffffffu, B.x, off);
    const double pBy = __shfl_up_sync(0xffffffffu, B.y, off);
    if (lane >= off) {  // (A, B) after (pA, pB): x -> A (pA x + pB) + B
      B.x = fma(A, pBx, B.x);
      B.y = fma(A, pBy, B.y);
      A = A * pA;
    }
  }
}

template <int kSimMaxCpl>
__global__ void __launch_bounds__(256, kSimMaxCpl == 4 ? 2 : 3) fpm_sim_kernel(const SimArgs a) {
  const int lane = threadIdx.x & 31;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = ((long)gridDim.x * blockDim.x) >> 5;
  const int N = a.N, M = a.M, cpl = a.cpl;
  const int n0 = lane * cpl;
  for (long t = warp; t < a.T; t += nwarps) {
    const uint64_t trial = (uint64_t)(a.trial0 + t);
    // payload bits and symbols of this lane's users (detect.py:54-67, 207)
    double2 s[kSimMaxCpl];
#pragma unroll
    for (int k = 0; k < kSimMaxCpl; ++k) {
      s[k] = make_double2(0.0, 0.0);
      const int n = n0 + k;
      if (k < cpl && n < N) {
        int iv = 0, qv = 0;
        const int h = a.bps / 2;
        for (int q = 0; q < a.bps; ++q) {
          const uint32_t e = (uint32_t)(n * a.bps + q);
          const uint32_t bit = gen_bit(a.k0, a.k1, e, trial);
          a.bits[(long)t * N * a.bps + e] = (uint8_t)bit;
          if (q < h) iv = 2 * iv + (int)bit;
          else qv = 2 * qv + (int)bit;
        }
        s[k] = make_double2(a.lv[iv], a.lv[qv]);
        if (a.sym) a.sym[(long)t * N + n] = s[k];
      }
    }
    double2 hprev[kSimMaxCpl];  // H[m-1, n] of this lane's columns
#pragma unroll
    for (int k = 0; k < kSimMaxCpl; ++k) hprev[k] = make_double2(0.0, 0.0);
    double2* Ht = a.H + (long)t * M * N;
    double2* Et = a.Hest ? a.Hest + (long)t * M * N : nullptr;
    for (int m0 = 0; m0 < M; m0 += kSimRows) {
      // draws of kSimRows rows first (independent Philox / Box-Muller chains
      // in flight together), then the recursions of those rows
      double2 wv[kSimRows][kSimMaxCpl];
      double2 gn = make_double2(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < kSimRows; ++r)
#pragma unroll
        for (int k = 0; k < kSimMaxCpl; ++k) {
          const int n = n0 + k, m = m0 + r;
          wv[r][k] = make_double2(0.0, 0.0);
          if (k < cpl && n < N && m < M) {
            const double2 g = cnormal(a.k0, a.k1, kStreamW, (uint32_t)(m * N + n), trial);
            wv[r][k] = make_double2(g.x * a.wscale, g.y * a.wscale);
          }
        }
      if (lane < kSimRows && m0 + lane < M) gn = cnormal(a.k0, a.k1, kStreamNoise, (uint32_t)(m0 + lane), trial);
#pragma unroll
      for (int r = 0; r < kSimRows; ++r) {
        const int m = m0 + r;
        if (m >= M) break;
        // transmit side: x_n = at_n x_{n-1} + ct_n w_n along the users; the
        // lane folds its segment into (A, B), the warp scans the segments
        double2 xl[kSimMaxCpl];
        double A = 1.0;
        double2 B = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < kSimMaxCpl; ++k) {
          const int n = n0 + k;
          xl[k] = make_double2(0.0, 0.0);
          if (k < cpl && n < N) {
            const double2 w = wv[r][k];
            const bool start = (n == 0) || (a.block_diag && n % a.n_ue == 0);
            const double an = start ? 0.0 : a.zt, cn = start ? 1.0 : a.ct;
            B = make_double2(fma(an, B.x, cn * w.x), fma(an, B.y, cn * w.y));
            A *= an;
            xl[k] = B;  // value with a zero carry-in
          }
        }
        affine_scan(A, B, lane);
        // carry into this lane = inclusive value of the previous lane
        double2 cin = make_double2(__shfl_up_sync(0xffffffffu, B.x, 1), __shfl_up_sync(0xffffffffu, B.y, 1));
        if (lane == 0) cin = make_double2(0.0, 0.0);
        // receive side: H[m, n] = ar_m H[m-1, n] + cr_m X[m, n]
        const double ar = m == 0 ? 0.0 : a.zr, crm = m == 0 ? 1.0 : a.cr;
        double2 acc = make_double2(0.0, 0.0);  // this lane's part of (H s)[m]
        double mul = 1.0;
#pragma unroll
        for (int k = 0; k < kSimMaxCpl; ++k) {
          const int n = n0 + k;
          if (k < cpl && n < N) {
            const bool start = (n == 0) || (a.block_diag && n % a.n_ue == 0);
            mul = start ? 0.0 : mul * a.zt;  // product of the multipliers from the lane start to n
            const double2 x = make_double2(fma(mul, cin.x, xl[k].x), fma(mul, cin.y, xl[k].y));
            const double2 hv = make_double2(fma(ar, hprev[k].x, crm * x.x), fma(ar, hprev[k].y, crm * x.y));
            hprev[k] = hv;
            Ht[(long)m * N + n] = hv;
            if (Et) {
              const double2 c = cnormal(a.k0, a.k1, kStreamCsi, (uint32_t)(m * N + n), trial);
              Et[(long)m * N + n] = make_double2(fma(a.cscale, c.x, hv.x), fma(a.cscale, c.y, hv.y));
            }
            acc.x = fma(hv.x, s[k].x, fma(-hv.y, s[k].y, acc.x));
            acc.y = fma(hv.x, s[k].y, fma(hv.y, s[k].x, acc.y));
          }
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) {
          acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
          acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
        }
        if (lane == r)  // every lane holds the row sum; lane r drew row m's noise
          a.y[(long)t * M + m] = make_double2(fma(a.nscale, gn.x, acc.x), fma(a.nscale, gn.y, acc.y));
      }
    }
  }
}

}  // namespace fpm

using namespace fpm;

extern "C" int fpm_simulate(uint64_t seed, int32_t context, int32_t point, int64_t trial0, int64_t T, int32_t M,
                            int32_t N, double zeta_r, double zeta_t, int32_t n_ue, int32_t block_diag_users,
                            int32_t qam, double sigma2, double csi_var, double* H, double* H_est, double* y,
                            uint8_t* bits, double* symbols, void* stream) {
  if (T < 0 || M < 1 || N < 1 || trial0 < 0 || (T > 0 && (!H || !y || !bits))) return FPM_EINVAL;
  if (context < 0 || context >= (1 << 12) || point < 0 || point >= (1 << 16)) return FPM_EINVAL;  // rng.py:21-26
  if (!(zeta_r >= 0.0 && zeta_r < 1.0) || !(zeta_t >= 0.0 && zeta_t < 1.0)) return FPM_EINVAL;    // channel.py:109
  if (qam != 16 && qam != 64) return FPM_EINVAL;
  if (!(sigma2 >= 0.0) || n_ue < 1 || (block_diag_users && N % n_ue)) return FPM_EINVAL;
  if ((H_est != nullptr) != (csi_var >= 0.0)) return FPM_EINVAL;
  if (N > 32 * kSimCplMax) return FPM_EUNSUPPORTED;
  if (T == 0) return FPM_OK;
  SimArgs a;
  a.k0 = (uint32_t)seed;
  a.k1 = (uint32_t)(seed >> 32) ^ ((uint32_t)context << 16) ^ (uint32_t)point;
  a.trial0 = trial0;
  a.T = T;
  a.M = M;
  a.N = N;
  a.cpl = (N + 31) / 32;
  a.bps = qam == 16 ? 4 : 6;
  a.n_ue = n_ue;
  a.block_diag = block_diag_users ? 1 : 0;
  a.zr = zeta_r;
  a.cr = std::sqrt(1.0 - zeta_r * zeta_r);
  a.zt = zeta_t;
  a.ct = std::sqrt(1.0 - zeta_t * zeta_t);
  a.wscale = 1.0 / std::sqrt(2.0 * M);
  a.nscale = std::sqrt(sigma2 / 2.0);
  a.cscale = csi_var >= 0.0 ? std::sqrt(csi_var / 2.0) : -1.0;
  // Gray levels per axis (detect.py:47; 64-QAM extension), indexed by the
  // axis bits read MSB first
  if (qam == 16) {
    const double sc = 1.0 / std::sqrt(10.0), l[4] = {-3, -1, 3, 1};
    for (int i = 0; i < 4; ++i) a.lv[i] = l[i] * sc;
  } else {
    const double sc = 1.0 / std::sqrt(42.0), l[8] = {-7, -5, -1, -3, 7, 5, 1, 3};
    for (int i = 0; i < 8; ++i) a.lv[i] = l[i] * sc;
  }
  a.H = reinterpret_cast<double2*>(H);
  a.Hest = reinterpret_cast<double2*>(H_est);
  a.y = reinterpret_cast<double2*>(y);
  a.bits = bits;
  a.sym = reinterpret_cast<double2*>(symbols);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tpb = 256;
  const long grid = std::min<long>((T + tpb / 32 - 1) / (tpb / 32), (long)sms * 8);
  if (a.cpl == 1) fpm_sim_kernel<1><<<(unsigned)grid, tpb, 0, (cudaStream_t)stream>>>(a);
  else if (a.cpl == 2) fpm_sim_kernel<2><<<(unsigned)grid, tpb, 0, (cudaStream_t)stream>>>(a);
  else fpm_sim_kernel<4><<<(unsigned)grid, tpb, 0, (cudaStream_t)stream>>>(a);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}
