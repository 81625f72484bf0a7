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
#include "fpm_gram32.cuh"
#include "fpm_ptx.cuh"

namespace fpm {

constexpr int kG32Rows = 16;  // antenna rows per staged chunk
constexpr int kG32Jobs = 2;   // jobs per thread (N = 128: 512 jobs on 256 threads)

template <int NB>  // nb = Np/4 at compile time (0 = run time): immediate-offset operand loads
__global__ void __launch_bounds__(256) fpm_gram32_kernel(const double2* __restrict__ H, const double2* __restrict__ y,
                                                          long T, int M, int N, double sigma2, double2* __restrict__ A,
                                                          double2* __restrict__ b, f2x k_one, f2x k_pm) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int Np = NB > 0 ? 4 * NB : (N + 7) / 8 * 8, nb = NB > 0 ? NB : Np / 4;
  const int raw_bytes = kG32Rows * N * 16 + kG32Rows * 16;  // one binary64 chunk: H rows, then y entries
  float2* hs = reinterpret_cast<float2*>(smem + 2 * raw_bytes);  // [kG32Rows][Np] binary32
  float2* ysm = hs + kG32Rows * Np;                             // [kG32Rows]
  uint64_t* full = reinterpret_cast<uint64_t*>(ysm + kG32Rows);  // one per raw buffer
  const long t = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int njobs = nb * (nb / 2 - 1) + nb;
  const Cj32 cj{k_one, k_pm};
  GramJob job[kG32Jobs];
  f2x acc[kG32Jobs][16];
#pragma unroll
  for (int s = 0; s < kG32Jobs; ++s) {
    const int q = tid + s * nt;
    job[s] = q < njobs ? gram_job(q, 1, nb) : GramJob{-1, 0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[s][k] = 0ull;
  }
  // matched-filter chains: q in [0, 2N) -> entry n, part (0 re / 1 im)
  const bool chain = tid < 2 * N;
  const int cpart = tid / max(N, 1), cn = tid - cpart * N;
  float ca = 0.f;
  const double2* Ht = H + t * (long)M * N;
  const double2* yt = y + t * (long)M;
  const int nch = (M + kG32Rows - 1) / kG32Rows;
  // chunk c (binary64, as it lies in HBM) -> raw buffer c & 1, one bulk copy each for H and y
  auto issue = [&](int c) {
    const int m0 = c * kG32Rows, rows = min(kG32Rows, M - m0);
    unsigned char* dst = smem + (c & 1) * raw_bytes;
    mbar_expect_tx(full + (c & 1), (uint32_t)(rows * N * 16 + rows * 16));
    bulk_g2s(dst, Ht + (long)m0 * N, (uint32_t)(rows * N * 16), full + (c & 1));
    bulk_g2s(dst + kG32Rows * N * 16, yt + m0, (uint32_t)(rows * 16), full + (c & 1));
  };
  if (tid == 0) {
    mbar_init(full, 1);
    mbar_init(full + 1, 1);
    fence_mbar_init();
    issue(0);
  }
#pragma unroll 1
  for (int c = 0; c < nch; ++c) {
    const int m0 = c * kG32Rows, rows = min(kG32Rows, M - m0);
    __syncthreads();  // chunk c-1 accumulated by all: hs free, raw buffer (c+1)&1 long converted
    if (tid == 0 && c + 1 < nch) issue(c + 1);  // lands while chunk c is converted and accumulated
    mbar_wait(full + (c & 1), (uint32_t)((c >> 1) & 1));
    const double2* raw = reinterpret_cast<const double2*>(smem + (c & 1) * raw_bytes);
    for (int q = tid; q < rows * Np; q += nt) {
      const int r = q / Np, cc = q - r * Np;
      const double2 v = cc < N ? raw[r * N + cc] : make_double2(0.0, 0.0);
      hs[q] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
    }
    if (tid < rows) {
      const double2 v = raw[kG32Rows * N + tid];
      ysm[tid] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
    }
    __syncthreads();
    (void)m0;
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
            for (int v = 0; v < 4; ++v) cj.mac(acc[s][u * 4 + v], hi[u], hj[v]);
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
            for (int v = u + 1; v < 4; ++v) cj.mac(acc[s][p++], hx[u], hx[v]);
#pragma unroll
          for (int w = 0; w < 2; ++w)
#pragma unroll
            for (int v = 0; v < 4; ++v) cj.mac(acc[s][6 + w * 4 + v], hy[w], hz[v]);
          // diagonal: (|h_a|^2, |h_a+nb|^2) and (|h_a+2nb|^2, |h_a+3nb|^2)
          const f2x q0 = mul2(pk2(hx[0].x, hx[1].x), pk2(hx[0].x, hx[1].x));
          const f2x q1 = mul2(pk2(hx[0].y, hx[1].y), pk2(hx[0].y, hx[1].y));
          const f2x q2 = mul2(pk2(hx[2].x, hx[3].x), pk2(hx[2].x, hx[3].x));
          const f2x q3 = mul2(pk2(hx[2].y, hx[3].y), pk2(hx[2].y, hx[3].y));
          acc[s][14] = fma2(fma2(q1, cj.one, q0), cj.one, acc[s][14]);
          acc[s][15] = fma2(fma2(q3, cj.one, q2), cj.one, acc[s][15]);
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
  auto put = [&](int i, int j, f2x Gp) {
    const float2 G = upk2(Gp);
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
      const float2 d01 = upk2(acc[s][14]), d23 = upk2(acc[s][15]);
      const float dg[4] = {d01.x, d01.y, d23.x, d23.y};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = jb.a + nb * u;
        if (i < N) At[(long)i * N + i] = make_double2((double)__fadd_rn(dg[u], s2f), 0.0);
      }
    }
  }
  if (chain) reinterpret_cast<double*>(b + t * N + cn)[cpart] = (double)ca;
}

static const f2x g32_one = kG32One, g32_pm = kG32Pm;

int launch_gram32(const double2* H, const double2* y, long T, int M, int N, double sigma2, double2* A, double2* b,
                  cudaStream_t st) {
  const int Np = (N + 7) / 8 * 8, nb = Np / 4;
  const int njobs = nb * (nb / 2 - 1) + nb;
  const int threads = std::max(2 * N, std::min(256, (njobs + 31) / 32 * 32));
  if ((njobs + threads - 1) / threads > kG32Jobs || threads > 256) return FPM_EUNSUPPORTED;
  const int smem = 2 * (kG32Rows * N * 16 + kG32Rows * 16) + (kG32Rows * Np + kG32Rows) * 8 + 16;
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(fpm_gram32_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(fpm_gram32_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(fpm_gram32_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  }
  if (nb == 32)
    fpm_gram32_kernel<32><<<(unsigned)T, threads, smem, st>>>(H, y, T, M, N, sigma2, A, b, g32_one, g32_pm);
  else if (nb == 16)
    fpm_gram32_kernel<16><<<(unsigned)T, threads, smem, st>>>(H, y, T, M, N, sigma2, A, b, g32_one, g32_pm);
  else
    fpm_gram32_kernel<0><<<(unsigned)T, threads, smem, st>>>(H, y, T, M, N, sigma2, A, b, g32_one, g32_pm);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}

}  // namespace fpm
