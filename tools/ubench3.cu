// chain_sum / wdiv from the library headers, timed in isolation (dev tool)
#include <cstdio>
#include "../paper_2504_09820_b200/csrc/fpm_cg.cuh"
using namespace fpm;
__global__ void k(long long* out, int reps) {
  __shared__ __half2 t[64];
  __shared__ FmtP f;
  if (threadIdx.x < 64) t[threadIdx.x] = __floats2half2_rn(1e-3f * threadIdx.x, 1e-2f);
  if (threadIdx.x == 0) { f.sig = 53; f.qmin = -1074; f.sub = 1; f.native = 1; f.xmax = 1e308; f.xmin = 1e-308; }
  __syncthreads();
  if (threadIdx.x == blockDim.x - 1) {
    double2 acc = make_double2(0, 0);
    for (int r = 0; r < reps; ++r) {
      long long c0 = clock64();
      double2 s = chain_sum<FK_F16>(t, 64, f);
      long long c1 = clock64();
      double2 q = wdiv<FK_F64>(make_double2(1.0 + s.x, 0.5 + r), make_double2(2.0 + s.y, 0.25), f);
      long long c2 = clock64();
      acc.x += q.x; acc.y += q.y;
      out[2 * r] = c1 - c0; out[2 * r + 1] = c2 - c1;
    }
    if (acc.x == 12345.0) out[0] = 0;
  }
}
int main() {
  long long* d; cudaMalloc(&d, 64 * 8);
  long long h[16];
  for (int thr : {32, 512}) {
    k<<<1, thr>>>(d, 6);
    cudaMemcpy(h, d, 12 * 8, cudaMemcpyDeviceToHost);
    printf("threads %d chain_sum:", thr); for (int r = 0; r < 6; ++r) printf(" %lld", h[2*r]);
    printf(" | wdiv:"); for (int r = 0; r < 6; ++r) printf(" %lld", h[2*r+1]); printf("\n");
  }
  return 0;
}
