// fp64 work, fp32 matvec / inner products (generic geometry).
#include "fpm_detect_ws.cuh"
namespace fpm {
int launch_detect_f32(const DetectArgs& a, int threads, int nb, int lb, cudaStream_t st) {
  return launch_detect_t<FK_F64, FK_F32, 0, 0>(a, threads, st);
}
int launch_cg_f32(const CgArgs& a, int smem, int lb, cudaStream_t st) {
  return launch_cg_t<FK_F64, FK_F32, 0>(a, smem, st);
}
int launch_detect_ws_f32(const DetectArgs& a, const WsLayout& sl, int grid, int nb, int lb, cudaStream_t st) {
  return launch_detect_ws_t<FK_F64, FK_F32, 0, 0>(a, sl, grid, st);
}
}  // namespace fpm
