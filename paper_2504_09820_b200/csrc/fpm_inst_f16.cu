// fp64 work, fp16 matvec / inner products.  Specialisations: c3/c5
// (N=64, L=4), c4 (N=128, L=8), c2 (N=32, plain).
#include "fpm_detect_ws.cuh"
namespace fpm {
int launch_detect_f16(const DetectArgs& a, int threads, int nb, int lb, cudaStream_t st) {
  if (nb == 16 && lb == 4) return launch_detect_t<FK_F64, FK_F16, 16, 4>(a, threads, st);
  if (nb == 32 && lb == 8) return launch_detect_t<FK_F64, FK_F16, 32, 8>(a, threads, st);
  if (nb == 8 && lb == 0) return launch_detect_t<FK_F64, FK_F16, 8, 0>(a, threads, st);
  return launch_detect_t<FK_F64, FK_F16, 0, 0>(a, threads, st);
}
int launch_cg_f16(const CgArgs& a, int smem, int lb, cudaStream_t st) {
  if (lb == 4) return launch_cg_t<FK_F64, FK_F16, 4>(a, smem, st);
  return launch_cg_t<FK_F64, FK_F16, 0>(a, smem, st);
}
int launch_detect_ws_f16(const DetectArgs& a, const WsLayout& sl, int grid, int nb, int lb, cudaStream_t st) {
  if (nb == 16 && lb == 4) return launch_detect_ws_t<FK_F64, FK_F16, 16, 4>(a, sl, grid, st);
  if (nb == 8 && lb == 0) return launch_detect_ws_t<FK_F64, FK_F16, 8, 0>(a, sl, grid, st);
  if (nb == 32 && lb == 8) return launch_detect_ws_t<FK_F64, FK_F16, 32, 8>(a, sl, grid, st);
  return launch_detect_ws_t<FK_F64, FK_F16, 0, 0>(a, sl, grid, st);
}
}  // namespace fpm
