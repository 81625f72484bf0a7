// FP32-Gram extension (BASELINE.json config c4, "FP32 Gram"; the reference
// has no such knob -- parity unpinned, restated in oracle gram_mf_fp32):
// the Gram / matched filter of detect.py:215-218 with H and y rounded once to
// binary32 and every operation in binary32 (FMUL / FADD, no FMA): per entry
// acc = +0f; for m in order: acc.re += fl32(fl32(hr_i hr_j) + fl32(hi_i hi_j)),
// acc.im += fl32(fl32(hr_i hi_j) - fl32(hi_i hr_j)); final entries
// (G.re + delta_ij fl32(sigma^2), G.im + 0f), mirrors (G.re + 0f, 0f - G.im);
// b likewise.  Results are widened exactly to the complex128 carriers the CG
// consumes.  Runs on the FP32 pipe (twice the FP64 rate on B200).
//
// One CTA per realization; H rows staged to shared memory as binary32 in
// chunks; each thread owns up to two 4x4 jobs of the residue-class tiling
// (gram_job, R = 1) and the matched-filter chains are spread over threads.
#include <cuda_runtime.h>

#include <algorithm>

#include "../../include/fpmimo_b200.h"
#include "fpm_common.cuh"

namespace fpm {

__device__ __forceinline__ void cmac_conj32(float2& acc, float2 hi, float2 hj) {
  const float pr = __fadd_rn(__fmul_rn(hi.x, hj.x), __fmul_rn(hi.y, hj.y));
  const float pi = __fsub_rn(__fmul_rn(hi.x, hj.y), __fmul_rn(hi.y, hj.x));
  acc.x = __fadd_rn(acc.x, pr);
  acc.y = __fadd_rn(acc.y, pi);
}

constexpr int kG32Rows = 16;  // antenna rows per staged chunk
constexpr int kG32Jobs = 2;   // jobs per thread (N = 128: 512 jobs on 256 threads)

__global__ void __launch_bounds__(256) fpm_gram32_kernel(const double2* __restrict__ H, const double2* __restrict__ y,
                                                          long T, int M, int N, double sigma2, double2* __restrict__ A,
                                                          double2* __restrict__ b) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int Np = (N + 7) / 8 * 8, nb = Np / 4;
  float2* hs = reinterpret_cast<float2*>(smem);          // [kG32Rows][Np]
  float2* ysm = hs + kG32Rows * Np;                      // [kG32Rows]
  const long t = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int njobs = nb * (nb / 2 - 1) + nb;
  GramJob job[kG32Jobs];
  float2 acc[kG32Jobs][16];
#pragma unroll
  for (int s = 0; s < kG32Jobs; ++s) {
    const int q = tid + s * nt;
    job[s] = q < njobs ? gram_job(q, 1, nb) : GramJob{-1, 0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[s][k] = make_float2(0.f, 0.f);
  }
  // matched-filter chains: q in [0, 2N) -> entry n, part (0 re / 1 im)
  const bool chain = tid < 2 * N;
  const int cpart = tid / max(N, 1), cn = tid - cpart * N;
  float ca = 0.f;
  const double2* Ht = H + t * (long)M * N;
  const double2* yt = y + t * (long)M;
#pragma unroll 1
  for (int m0 = 0; m0 < M; m0 += kG32Rows) {
    const int rows = min(kG32Rows, M - m0);
    __syncthreads();
    for (int q = tid; q < rows * Np; q += nt) {
      const int r = q / Np, c = q - r * Np;
      const double2 v = c < N ? Ht[(long)(m0 + r) * N + c] : make_double2(0.0, 0.0);
      hs[q] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
    }
    for (int r = tid; r < rows; r += nt) {
      const double2 v = yt[m0 + r];
      ysm[r] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kG32Jobs; ++s) {
      const GramJob& jb = job[s];
      if (jb.g < 0) continue;
      if (!jb.half) {
#pragma unroll 1
        for (int mm = 0; mm < rows; ++mm) {
          const float2* row = hs + mm * Np;
          float2 hi[4], hj[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) hi[u] = row[jb.a + nb * u];
#pragma unroll
          for (int v = 0; v < 4; ++v) hj[v] = row[jb.c + nb * v];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) cmac_conj32(acc[s][u * 4 + v], hi[u], hj[v]);
        }
      } else {
#pragma unroll 1
        for (int mm = 0; mm < rows; ++mm) {
          const float2* row = hs + mm * Np;
          float2 hx[4], hy[2], hz[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) hx[u] = row[jb.a + nb * u];
#pragma unroll
          for (int w = 0; w < 2; ++w) hy[w] = row[jb.y + nb * (jb.yo + w)];
#pragma unroll
          for (int v = 0; v < 4; ++v) hz[v] = row[jb.c + nb * v];
          int p = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = u + 1; v < 4; ++v) cmac_conj32(acc[s][p++], hx[u], hx[v]);
#pragma unroll
          for (int w = 0; w < 2; ++w)
#pragma unroll
            for (int v = 0; v < 4; ++v) cmac_conj32(acc[s][6 + w * 4 + v], hy[w], hz[v]);
          float dg[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) dg[u] = __fadd_rn(__fmul_rn(hx[u].x, hx[u].x), __fmul_rn(hx[u].y, hx[u].y));
          acc[s][14].x = __fadd_rn(acc[s][14].x, dg[0]);
          acc[s][14].y = __fadd_rn(acc[s][14].y, dg[1]);
          acc[s][15].x = __fadd_rn(acc[s][15].x, dg[2]);
          acc[s][15].y = __fadd_rn(acc[s][15].y, dg[3]);
        }
      }
    }
    if (chain) {
#pragma unroll 1
      for (int mm = 0; mm < rows; ++mm) {
        const float2 h = hs[mm * Np + cn], yv = ysm[mm];
        // re: hr yr + hi yi ; im: hr yi - hi yr
        const float t1 = __fmul_rn(h.x, cpart ? yv.y : yv.x);
        const float t2 = __fmul_rn(h.y, cpart ? yv.x : yv.y);
        ca = __fadd_rn(ca, cpart ? __fsub_rn(t1, t2) : __fadd_rn(t1, t2));
      }
    }
  }
  // emit: final / mirror entries in binary32, widened to the fp64 carriers
  const float s2f = __double2float_rn(sigma2);
  double2* At = A + t * (long)N * N;
  auto put = [&](int i, int j, float2 G) {
    At[(long)i * N + j] = make_double2((double)__fadd_rn(G.x, 0.f), (double)__fadd_rn(G.y, 0.f));
    At[(long)j * N + i] = make_double2((double)__fadd_rn(G.x, 0.f), (double)__fsub_rn(0.f, G.y));
  };
#pragma unroll
  for (int s = 0; s < kG32Jobs; ++s) {
    const GramJob& jb = job[s];
    if (jb.g < 0) continue;
    if (!jb.half) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int i = jb.a + nb * u, j = jb.c + nb * v;
          if (i < N && j < N) put(i, j, acc[s][u * 4 + v]);
        }
    } else {
      int p = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = u + 1; v < 4; ++v) {
          const int i = jb.a + nb * u, j = jb.a + nb * v;
          if (i < N && j < N) put(i, j, acc[s][p]);
          ++p;
        }
#pragma unroll
      for (int w = 0; w < 2; ++w)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int i = jb.y + nb * (jb.yo + w), j = jb.c + nb * v;
          if (i < N && j < N) put(i, j, acc[s][6 + w * 4 + v]);
        }
      const float dg[4] = {acc[s][14].x, acc[s][14].y, acc[s][15].x, acc[s][15].y};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = jb.a + nb * u;
        if (i < N) At[(long)i * N + i] = make_double2((double)__fadd_rn(dg[u], s2f), 0.0);
      }
    }
  }
  if (chain) reinterpret_cast<double*>(b + t * N + cn)[cpart] = (double)ca;
}

int launch_gram32(const double2* H, const double2* y, long T, int M, int N, double sigma2, double2* A, double2* b,
                  cudaStream_t st) {
  const int Np = (N + 7) / 8 * 8, nb = Np / 4;
  const int njobs = nb * (nb / 2 - 1) + nb;
  const int threads = std::max(2 * N, std::min(256, (njobs + 31) / 32 * 32));
  if ((njobs + threads - 1) / threads > kG32Jobs || threads > 256) return FPM_EUNSUPPORTED;
  const int smem = (kG32Rows * Np + kG32Rows) * 8;
  fpm_gram32_kernel<<<(unsigned)T, threads, smem, st>>>(H, y, T, M, N, sigma2, A, b);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}

}  // namespace fpm
