#include <algorithm>
// Generic emulation of any (sig, exp) format: fp64 work with generic
// matvec/inner formats, and everything generic (work coarser than fp64).
#include "fpm_detect_ws.cuh"
namespace fpm {
int launch_detect_gen(const DetectArgs& a, int threads, int nb, int lb, cudaStream_t st) {
  return launch_detect_t<FK_F64, FK_GEN, 0, 0>(a, threads, st);
}
int launch_cg_gen(const CgArgs& a, int smem, int lb, cudaStream_t st) {
  return launch_cg_t<FK_F64, FK_GEN, 0>(a, smem, st);
}
int launch_detect_gen_w(const DetectArgs& a, int threads, int nb, int lb, cudaStream_t st) {
  return launch_detect_t<FK_GEN, FK_GEN, 0, 0>(a, threads, st);
}
int launch_cg_gen_w(const CgArgs& a, int smem, int lb, cudaStream_t st) {
  return launch_cg_t<FK_GEN, FK_GEN, 0>(a, smem, st);
}
int launch_detect_ws_gen(const DetectArgs& a, const WsLayout& sl, int grid, int nb, int lb, cudaStream_t st) {
  return launch_detect_ws_t<FK_F64, FK_GEN, 0, 0>(a, sl, grid, st);
}
int launch_detect_ws_gen_w(const DetectArgs& a, const WsLayout& sl, int grid, int nb, int lb, cudaStream_t st) {
  return launch_detect_ws_t<FK_GEN, FK_GEN, 0, 0>(a, sl, grid, st);
}
__global__ void fpm_round_mv_gen_kernel(const double2* __restrict__ A, double2* __restrict__ out, long n, FmtP f) {
  for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (long)gridDim.x * blockDim.x)
    out[q] = Ar<FK_GEN>::rnd(A[q], f);
}
int launch_round_mv_gen(const double2* A, double2* out, long n, FmtP f, cudaStream_t st) {
  const long grid = std::min<long>((n + 255) / 256, 148L * 16);
  fpm_round_mv_gen_kernel<<<(unsigned)grid, 256, 0, st>>>(A, out, n, f);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}
}  // namespace fpm
