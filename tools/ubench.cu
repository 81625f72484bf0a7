// Latency microbenchmarks for the CG critical path on sm_100a (dev tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/ubench tools/ubench.cu
#include <cuda_fp16.h>
#include <cstdio>

__global__ void lat_dadd(double* out, long n, double a) {
  double x = a;
  long long t0 = clock64();
  for (long i = 0; i < n; ++i) x = __dadd_rn(x, 1e-300);
  long long t1 = clock64();
  out[0] = x;
  out[1] = (double)(t1 - t0) / n;
}
__global__ void lat_dmul(double* out, long n, double a) {
  double x = a;
  long long t0 = clock64();
  for (long i = 0; i < n; ++i) x = __dmul_rn(x, 1.0000000001);
  long long t1 = clock64();
  out[0] = x;
  out[1] = (double)(t1 - t0) / n;
}
__global__ void lat_ddiv(double* out, long n, double a) {
  double x = a;
  long long t0 = clock64();
  for (long i = 0; i < n; ++i) x = __ddiv_rn(1.0000001, x);
  long long t1 = clock64();
  out[0] = x;
  out[1] = (double)(t1 - t0) / n;
}
__global__ void lat_dsqrt(double* out, long n, double a) {
  double x = a;
  long long t0 = clock64();
  for (long i = 0; i < n; ++i) x = __dsqrt_rn(x + 1.0);
  long long t1 = clock64();
  out[0] = x;
  out[1] = (double)(t1 - t0) / n;
}
__global__ void lat_hadd2(double* out, long n, float a) {
  __half2 x = __floats2half2_rn(a, a), d = __floats2half2_rn(1e-3f, 1e-3f);
  long long t0 = clock64();
  for (long i = 0; i < n; ++i) x = __hadd2_rn(x, d);
  long long t1 = clock64();
  out[0] = __low2float(x);
  out[1] = (double)(t1 - t0) / n;
}
__global__ void lat_f2f(double* out, long n, double a) {
  double x = a;
  long long t0 = clock64();
  for (long i = 0; i < n; ++i) x = (double)__half2float(__double2half(x)) + 1.0;
  long long t1 = clock64();
  out[0] = x;
  out[1] = (double)(t1 - t0) / n;
}
__global__ void lat_lds(double* out, long n) {
  __shared__ int buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (long i = 0; i < n; ++i) p = buf[p];
  long long t1 = clock64();
  out[0] = p;
  out[1] = (double)(t1 - t0) / n;
}
__global__ void lat_bar(double* out, long n) {
  long long t0 = clock64();
  for (long i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  __shared__ int s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  if (threadIdx.x == 0) out[1] = (double)(t1 - t0) / n;
}
// barrier round trip with a dependent smem value (forces real release)
__global__ void lat_bar_dep(double* out, long n) {
  __shared__ volatile int v[2];
  if (threadIdx.x == 0) v[0] = 0;
  __syncthreads();
  long long t0 = clock64();
  for (long i = 0; i < n; ++i) {
    if (threadIdx.x == (i & 255)) v[0] = v[0] + 1;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = v[0]; out[1] = (double)(t1 - t0) / n; }
}
// DP throughput per SM with k independent chains per thread, `warps` warps
template <int K>
__global__ void thr_dp(double* out, long n) {
  double a[K];
  for (int k = 0; k < K; ++k) a[k] = 1.0 + threadIdx.x + k;
  long long t0 = clock64();
  for (long i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = __dadd_rn(a[k], 1e-300);
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < K; ++k) s += a[k];
  if (threadIdx.x == 0) { out[0] = s; out[1] = (double)(t1 - t0) / n; }
}

int main() {
  double* d;
  cudaMalloc(&d, 16 * sizeof(double));
  double h[2];
  const long n = 100000;
#define RUN(name, launch)                                          \
  launch;                                                          \
  cudaMemcpy(h, d, 2 * sizeof(double), cudaMemcpyDeviceToHost);   \
  printf("%-28s %8.2f cycles\n", name, h[1]);
  RUN("dadd latency", (lat_dadd<<<1, 1>>>(d, n, 1.0)));
  RUN("dmul latency", (lat_dmul<<<1, 1>>>(d, n, 1.0)));
  RUN("ddiv latency", (lat_ddiv<<<1, 1>>>(d, n / 10, 1.5)));
  RUN("dsqrt latency", (lat_dsqrt<<<1, 1>>>(d, n / 10, 1.5)));
  RUN("hadd2 latency", (lat_hadd2<<<1, 1>>>(d, n, 1.0f)));
  RUN("f64->f16->f32->f64 +1", (lat_f2f<<<1, 1>>>(d, n, 1.0)));
  RUN("lds latency", (lat_lds<<<1, 32>>>(d, n)));
  RUN("bar.sync 512 thr (no dep)", (lat_bar<<<1, 512>>>(d, n)));
  RUN("bar.sync 512 thr (dep)", (lat_bar_dep<<<1, 512>>>(d, n)));
  RUN("bar.sync 128 thr (dep)", (lat_bar_dep<<<1, 128>>>(d, n)));
  for (int w : {1, 2, 4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "dadd x8 chains, %d warps/SM", w);
    RUN(nm, (thr_dp<8><<<1, 32 * w>>>(d, n / 10)));
    printf("    -> %.3f warp-DADD per cycle per SM\n", 8.0 * w / h[1]);
  }
  return 0;
}
