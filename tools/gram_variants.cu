// Gram inner-loop variants on smem-resident rows (dev tool; measures the DP
// pipe efficiency of the per-thread 4x4 Gram job shapes).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -Xptxas -v -o tools/gram_variants tools/gram_variants.cu
#include <cstdio>

__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  double pr = __dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y));
  double pi = __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x));
  acc.x = __dadd_rn(acc.x, pr);
  acc.y = __dadd_rn(acc.y, pi);
}

constexpr int NB = 16, NP = 64, ROWS = 32;

// V0: runtime nb, all 8 operands loaded up front (current library shape)
__global__ void __launch_bounds__(512, 1) v0(double2* out, int reps, int nb) {
  __shared__ double2 H[ROWS * NP];
  for (int i = threadIdx.x; i < ROWS * NP; i += blockDim.x) H[i] = make_double2(1e-3 * i, 2e-3 * (i & 7));
  __syncthreads();
  const int t = threadIdx.x % 120;
  const int d = 1 + t / 16, a = t % 16, c = (a + d) % 16;
  double2 acc[16];
  for (int k = 0; k < 16; ++k) acc[k] = make_double2(0, 0);
  for (int r = 0; r < reps; ++r)
    for (int m = 0; m < ROWS; ++m) {
      const double2* row = H + m * NP;
      double2 hi[4], hj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) hi[u] = row[a + nb * u];
#pragma unroll
      for (int v = 0; v < 4; ++v) hj[v] = row[c + nb * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) cmac(acc[u * 4 + v], hi[u], hj[v]);
    }
  double2 s = make_double2(0, 0);
  for (int k = 0; k < 16; ++k) { s.x += acc[k].x; s.y += acc[k].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// V1: compile-time NB (immediate offsets), same schedule
__global__ void __launch_bounds__(512, 1) v1(double2* out, int reps) {
  __shared__ double2 H[ROWS * NP];
  for (int i = threadIdx.x; i < ROWS * NP; i += blockDim.x) H[i] = make_double2(1e-3 * i, 2e-3 * (i & 7));
  __syncthreads();
  const int t = threadIdx.x % 120;
  const int d = 1 + t / 16, a = t % 16, c = (a + d) % 16;
  double2 acc[16];
  for (int k = 0; k < 16; ++k) acc[k] = make_double2(0, 0);
  const double2* pa = H + a;
  const double2* pc = H + c;
  for (int r = 0; r < reps; ++r)
#pragma unroll 2
    for (int m = 0; m < ROWS; ++m) {
      double2 hi[4], hj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) hi[u] = pa[m * NP + NB * u];
#pragma unroll
      for (int v = 0; v < 4; ++v) hj[v] = pc[m * NP + NB * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) cmac(acc[u * 4 + v], hi[u], hj[v]);
    }
  double2 s = make_double2(0, 0);
  for (int k = 0; k < 16; ++k) { s.x += acc[k].x; s.y += acc[k].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// V2: products first for a group of 4 entries (explicit ILP), then sums
__global__ void __launch_bounds__(512, 1) v2(double2* out, int reps) {
  __shared__ double2 H[ROWS * NP];
  for (int i = threadIdx.x; i < ROWS * NP; i += blockDim.x) H[i] = make_double2(1e-3 * i, 2e-3 * (i & 7));
  __syncthreads();
  const int t = threadIdx.x % 120;
  const int d = 1 + t / 16, a = t % 16, c = (a + d) % 16;
  double2 acc[16];
  for (int k = 0; k < 16; ++k) acc[k] = make_double2(0, 0);
  const double2* pa = H + a;
  const double2* pc = H + c;
  for (int r = 0; r < reps; ++r)
    for (int m = 0; m < ROWS; ++m) {
      double2 hj[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) hj[v] = pc[m * NP + NB * v];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 hi = pa[m * NP + NB * u];
        double p0[4], p1[4], q0[4], q1[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          p0[v] = __dmul_rn(hi.x, hj[v].x);
          p1[v] = __dmul_rn(hi.y, hj[v].y);
          q0[v] = __dmul_rn(hi.x, hj[v].y);
          q1[v] = __dmul_rn(hi.y, hj[v].x);
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          acc[u * 4 + v].x = __dadd_rn(acc[u * 4 + v].x, __dadd_rn(p0[v], p1[v]));
          acc[u * 4 + v].y = __dadd_rn(acc[u * 4 + v].y, __dsub_rn(q0[v], q1[v]));
        }
      }
    }
  double2 s = make_double2(0, 0);
  for (int k = 0; k < 16; ++k) { s.x += acc[k].x; s.y += acc[k].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// V3: like V1 plus next-row operand prefetch (register double buffer)
__global__ void __launch_bounds__(512, 1) v3(double2* out, int reps) {
  __shared__ double2 H[ROWS * NP];
  for (int i = threadIdx.x; i < ROWS * NP; i += blockDim.x) H[i] = make_double2(1e-3 * i, 2e-3 * (i & 7));
  __syncthreads();
  const int t = threadIdx.x % 120;
  const int d = 1 + t / 16, a = t % 16, c = (a + d) % 16;
  double2 acc[16];
  for (int k = 0; k < 16; ++k) acc[k] = make_double2(0, 0);
  const double2* pa = H + a;
  const double2* pc = H + c;
  for (int r = 0; r < reps; ++r) {
    double2 hj[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) hj[v] = pc[NB * v];
    for (int m = 0; m < ROWS; ++m) {
      double2 hi[4], nj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) hi[u] = pa[m * NP + NB * u];
      const int mn = (m + 1 < ROWS) ? m + 1 : m;
#pragma unroll
      for (int v = 0; v < 4; ++v) nj[v] = pc[mn * NP + NB * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) cmac(acc[u * 4 + v], hi[u], hj[v]);
#pragma unroll
      for (int v = 0; v < 4; ++v) hj[v] = nj[v];
    }
  }
  double2 s = make_double2(0, 0);
  for (int k = 0; k < 16; ++k) { s.x += acc[k].x; s.y += acc[k].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// V4: 4x2 tile (8 accumulators, 6 operands) -> more warps per SM (2 CTAs x 512)
__global__ void __launch_bounds__(512, 2) v4(double2* out, int reps) {
  __shared__ double2 H[ROWS * NP];
  for (int i = threadIdx.x; i < ROWS * NP; i += blockDim.x) H[i] = make_double2(1e-3 * i, 2e-3 * (i & 7));
  __syncthreads();
  const int t = threadIdx.x % 240;
  const int d = 1 + (t >> 1) / 16, a = (t >> 1) % 16, c = (a + d) % 16, h = t & 1;
  double2 acc[8];
  for (int k = 0; k < 8; ++k) acc[k] = make_double2(0, 0);
  const double2* pa = H + a;
  const double2* pc = H + c + NB * 2 * h;
  for (int r = 0; r < reps; ++r)
    for (int m = 0; m < ROWS; ++m) {
      double2 hi[4], hj[2];
#pragma unroll
      for (int u = 0; u < 4; ++u) hi[u] = pa[m * NP + NB * u];
#pragma unroll
      for (int v = 0; v < 2; ++v) hj[v] = pc[m * NP + NB * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) cmac(acc[u * 2 + v], hi[u], hj[v]);
    }
  double2 s = make_double2(0, 0);
  for (int k = 0; k < 8; ++k) { s.x += acc[k].x; s.y += acc[k].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// V5: 4x2 tiles, 512 threads per CTA (16 warps = 4 per SM sub-partition),
// one CTA per SM, register cap 128 (as the v1 sweep)
__global__ void __launch_bounds__(512, 1) v5(double2* out, int reps) {
  __shared__ double2 H[ROWS * NP];
  for (int i = threadIdx.x; i < ROWS * NP; i += blockDim.x) H[i] = make_double2(1e-3 * i, 2e-3 * (i & 7));
  __syncthreads();
  const int t = threadIdx.x % 240;
  const int d = 1 + (t >> 1) / 16, a = (t >> 1) % 16, c = (a + d) % 16, h = t & 1;
  double2 acc[8];
  for (int k = 0; k < 8; ++k) acc[k] = make_double2(0, 0);
  const double2* pa = H + a;
  const double2* pc = H + c + NB * 2 * h;
  for (int r = 0; r < reps; ++r)
#pragma unroll 2
    for (int m = 0; m < ROWS; ++m) {
      double2 hi[4], hj[2];
#pragma unroll
      for (int u = 0; u < 4; ++u) hi[u] = pa[m * NP + NB * u];
#pragma unroll
      for (int v = 0; v < 2; ++v) hj[v] = pc[m * NP + NB * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) cmac(acc[u * 2 + v], hi[u], hj[v]);
    }
  double2 s = make_double2(0, 0);
  for (int k = 0; k < 8; ++k) { s.x += acc[k].x; s.y += acc[k].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double2* d;
  cudaMalloc(&d, (size_t)148 * 8 * 512 * sizeof(double2));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 200;
  cudaFuncSetAttribute(v1, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  for (int thr : {128, 256, 384, 512}) {
    const int blocks = 148 * 4 * 512 / thr;
    v1<<<blocks, thr, 150 * 1024>>>(d, reps);  // 150 KB dynamic smem: one CTA per SM
    cudaEventRecord(e0);
    v1<<<blocks, thr, 150 * 1024>>>(d, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * thr * reps * ROWS * 128.0;
    printf("v1 %3d threads/CTA (1 CTA/SM resident): %6.2f TFLOP/s\n", thr, ops / (ms * 1e-3) / 1e12);
  }
  cudaFuncSetAttribute(v5, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  for (int thr : {256, 512}) {
    const int blocks = 148 * 4 * 512 / thr;
    v5<<<blocks, thr, 150 * 1024>>>(d, reps);
    cudaEventRecord(e0);
    v5<<<blocks, thr, 150 * 1024>>>(d, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * thr * reps * ROWS * 64.0;
    printf("v5 (4x2) %3d threads/CTA: %6.2f TFLOP/s\n", thr, ops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
