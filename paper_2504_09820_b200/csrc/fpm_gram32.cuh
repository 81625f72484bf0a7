// Packed binary32 arithmetic of the FP32-Gram extension, shared by the
// standalone kernel (fpm_gram32.cu) and the fused detector's Gram warps
// (fpm_detect_ws.cuh, DetectorSpec(gram="fp32")).
#pragma once
#include <stdint.h>

#include "fpm_gram.cuh"

namespace fpm {

// Packed binary32 pairs (FMUL2 / FFMA2, f32x2 PTX, sm_100a): two lanes per
// instruction, each an IEEE binary32 op rounded to nearest.  ptxas contracts
// even explicit-.rn f32x2 mul/add pairs into FFMA2, so every add is written
// as fma(x, k, y) with k = (1, 1) or (1, -1) passed in at run time: k is
// opaque to the compiler, x*k is exact, and the fma rounds once -- the same
// bits as add.rn / sub.rn, and nothing left to contract.
typedef unsigned long long f2x;
__device__ __forceinline__ f2x pk2(float a, float b) {
  f2x r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk2(f2x r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ f2x mul2(f2x a, f2x b) {
  f2x d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) {
  f2x d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// acc += conj(h_i) h_j:  P1 = (hr_i hr_j, hr_i hi_j), P2 = (hi_i hi_j, hi_i hr_j),
// (pr, pi) = P1 + (1, -1) P2, acc = acc + (pr, pi)
struct Cj32 {
  f2x one, pm;  // (1, 1), (1, -1) -- run-time values
  __device__ __forceinline__ void mac(f2x& acc, float2 hi, float2 hj) const {
    const f2x p1 = mul2(pk2(hi.x, hi.x), pk2(hj.x, hj.y));
    const f2x p2 = mul2(pk2(hi.y, hi.y), pk2(hj.y, hj.x));
    acc = fma2(fma2(p2, pm, p1), one, acc);
  }
};

// (1, 1) and (1, -1) as binary32 pairs, lane 0 in the low word (passed to
// kernels as run-time values so they stay opaque to the compiler)
constexpr f2x kG32One = 0x3F8000003F800000ull, kG32Pm = 0xBF8000003F800000ull;

// final reference-style entries of a binary32 Gram job, widened exactly to
// binary64: f(i, j, v_ij, v_ji) for i != j, d(i, v_ii) on the diagonal
// (G.re + 0f, G.im + 0f), mirrors (G.re + 0f, 0f - G.im), diagonal
// (G + fl32(sigma^2), 0)
template <class F, class D>
__device__ __forceinline__ void gram32_entries(const GramJob& job, const f2x (&acc)[16], int nb, int N, float s2f,
                                               F&& f, D&& d) {
  auto fin = [](f2x Gp) {
    const float2 G = upk2(Gp);
    return make_double2((double)__fadd_rn(G.x, 0.f), (double)__fadd_rn(G.y, 0.f));
  };
  auto mir = [](f2x Gp) {
    const float2 G = upk2(Gp);
    return make_double2((double)__fadd_rn(G.x, 0.f), (double)__fsub_rn(0.f, G.y));
  };
  if (!job.half) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = job.a + nb * u, j = job.c + nb * v;
        if (i < N && j < N) f(i, j, fin(acc[u * 4 + v]), mir(acc[u * 4 + v]));
      }
  } else {
    int p = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = u + 1; v < 4; ++v) {
        const int i = job.a + nb * u, j = job.a + nb * v;
        if (i < N && j < N) f(i, j, fin(acc[p]), mir(acc[p]));
        ++p;
      }
#pragma unroll
    for (int w = 0; w < 2; ++w)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = job.y + nb * (job.yo + w), j = job.c + nb * v;
        if (i < N && j < N) f(i, j, fin(acc[6 + w * 4 + v]), mir(acc[6 + w * 4 + v]));
      }
    const float2 d01 = upk2(acc[14]), d23 = upk2(acc[15]);
    const float dg[4] = {d01.x, d01.y, d23.x, d23.y};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = job.a + nb * u;
      if (i < N) d(i, make_double2((double)__fadd_rn(dg[u], s2f), 0.0));
    }
  }
}

// one antenna row of a binary32 Gram job (operands from the row's binary32 copy)
__device__ __forceinline__ void gram32_row(const GramJob& jb, const float2* row, int nb, const Cj32& cj, f2x (&acc)[16]) {
  if (!jb.half) {
    float2 hi[4], hj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) hi[u] = row[jb.a + nb * u];
#pragma unroll
    for (int v = 0; v < 4; ++v) hj[v] = row[jb.c + nb * v];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) cj.mac(acc[u * 4 + v], hi[u], hj[v]);
  } else {
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
      for (int v = u + 1; v < 4; ++v) cj.mac(acc[p++], hx[u], hx[v]);
#pragma unroll
    for (int w = 0; w < 2; ++w)
#pragma unroll
      for (int v = 0; v < 4; ++v) cj.mac(acc[6 + w * 4 + v], hy[w], hz[v]);
    // diagonal: (|h_a|^2, |h_a+nb|^2) and (|h_a+2nb|^2, |h_a+3nb|^2)
    const f2x q0 = mul2(pk2(hx[0].x, hx[1].x), pk2(hx[0].x, hx[1].x));
    const f2x q1 = mul2(pk2(hx[0].y, hx[1].y), pk2(hx[0].y, hx[1].y));
    const f2x q2 = mul2(pk2(hx[2].x, hx[3].x), pk2(hx[2].x, hx[3].x));
    const f2x q3 = mul2(pk2(hx[2].y, hx[3].y), pk2(hx[2].y, hx[3].y));
    acc[14] = fma2(fma2(q1, cj.one, q0), cj.one, acc[14]);
    acc[15] = fma2(fma2(q3, cj.one, q2), cj.one, acc[15]);
  }
}

}  // namespace fpm
