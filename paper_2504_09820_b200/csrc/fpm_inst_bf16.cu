// fp64 work, bfloat16 matvec / inner products.  Specialisations: c2-p7 (N=32, plain), c3 / c5 shapes at p = 7 (N=64, L=4; warp-specialised kernel).
#include "fpm_detect_ws.cuh"
namespace fpm {
int launch_detect_bf16(const DetectArgs& a, int threads, int nb, int lb, cudaStream_t st) {
  if (nb == 8 && lb == 0) return launch_detect_t<FK_F64, FK_BF16, 8, 0>(a, threads, st);
  return launch_detect_t<FK_F64, FK_BF16, 0, 0>(a, threads, st);
}
int launch_cg_bf16(const CgArgs& a, int smem, int lb, cudaStream_t st) {
  return launch_cg_t<FK_F64, FK_BF16, 0>(a, smem, st);
}
int launch_detect_ws_bf16(const DetectArgs& a, const WsLayout& sl, int grid, int nb, int lb, cudaStream_t st) {
  if (nb == 8 && lb == 0) return launch_detect_ws_t<FK_F64, FK_BF16, 8, 0>(a, sl, grid, st);
  if (nb == 16 && lb == 4) return launch_detect_ws_t<FK_F64, FK_BF16, 16, 4>(a, sl, grid, st);  // c3 / c5 shapes at p = 7
  return launch_detect_ws_t<FK_F64, FK_BF16, 0, 0>(a, sl, grid, st);
}
}  // namespace fpm
