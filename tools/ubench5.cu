// Sequential-sum latency variants (dev tool).
#include <cstdio>
#include "../paper_2504_09820_b200/csrc/fpm_cg.cuh"
using namespace fpm;

__device__ __noinline__ __half2 sum_pre(const __half2* t) {
  // all 64 terms loaded first (16 x LDS.128), then the dependent chain
  __half2 v[64];
  const uint4* q = reinterpret_cast<const uint4*>(t);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    uint4 u = q[i];
    v[4 * i] = u2h(u.x); v[4 * i + 1] = u2h(u.y); v[4 * i + 2] = u2h(u.z); v[4 * i + 3] = u2h(u.w);
  }
  __half2 s = v[0];
#pragma unroll
  for (int i = 1; i < 64; ++i) s = __hadd2_rn(s, v[i]);
  return s;
}

__device__ __noinline__ __half2 sum_pipe(const __half2* t) {
  // 16-term blocks, next block's loads issued before this block's adds
  const uint4* q = reinterpret_cast<const uint4*>(t);
  uint4 a0 = q[0], a1 = q[1], a2 = q[2], a3 = q[3];
  __half2 s = u2h(a0.x);
  bool first = true;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    uint4 n0, n1, n2, n3;
    if (b < 3) { n0 = q[4 * b + 4]; n1 = q[4 * b + 5]; n2 = q[4 * b + 6]; n3 = q[4 * b + 7]; }
    unsigned w[16] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w, a3.x, a3.y, a3.z, a3.w};
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (first && i == 0) continue;
      s = __hadd2_rn(s, u2h(w[i]));
    }
    first = false;
    if (b < 3) { a0 = n0; a1 = n1; a2 = n2; a3 = n3; }
  }
  return s;
}

__global__ void k(long long* out, int reps, int which) {
  __shared__ __align__(16) __half2 t[64 * 66];
  for (int i = threadIdx.x; i < 64 * 66; i += blockDim.x) t[i] = __floats2half2_rn(1e-3f * (i % 97), 2e-3f * (i % 13));
  __syncthreads();
  if (threadIdx.x != 0) return;
  FmtP f{};
  float acc = 0;
  for (int r = 0; r < reps; ++r) {
    long long c0 = clock64();
    __half2 s;
    if (which == 0) s = __floats2half2_rn(chain_sum<FK_F16>(t + 4 * r, 64, f).x, 0.f);
    else if (which == 1) s = sum_pre(t + 4 * r);
    else s = sum_pipe(t + 4 * r);
    acc += __low2float(s);
    long long c1 = clock64();
    out[r] = c1 - c0;
  }
  if (acc == 12345.f) out[0] = 0;
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  const char* nm[3] = {"chain_sum (8-batch)", "preload 64 + chain", "pipelined 16-blocks"};
  for (int w = 0; w < 3; ++w) {
    k<<<1, 128>>>(d, 6, w);
    cudaDeviceSynchronize();
    long long h[8];
    cudaMemcpy(h, d, 6 * sizeof(long long), cudaMemcpyDeviceToHost);
    printf("%-24s", nm[w]);
    for (int r = 0; r < 6; ++r) printf(" %lld", h[r]);
    printf("\n");
  }
  return 0;
}
