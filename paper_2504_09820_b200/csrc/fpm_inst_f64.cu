// fp64 throughout.  Specialisations: c1 (N=16, plain), c5-fp64 (N=64, L=4).
#include "fpm_detect_ws.cuh"
namespace fpm {
int launch_detect_f64(const DetectArgs& a, int threads, int nb, int lb, cudaStream_t st) {
  if (nb == 4 && lb == 0) return launch_detect_t<FK_F64, FK_F64, 4, 0>(a, threads, st);
  if (nb == 16 && lb == 4) return launch_detect_t<FK_F64, FK_F64, 16, 4>(a, threads, st);
  return launch_detect_t<FK_F64, FK_F64, 0, 0>(a, threads, st);
}
int launch_cg_f64(const CgArgs& a, int smem, int lb, cudaStream_t st) {
  if (lb == 4) return launch_cg_t<FK_F64, FK_F64, 4>(a, smem, st);
  return launch_cg_t<FK_F64, FK_F64, 0>(a, smem, st);
}
int launch_detect_ws_f64(const DetectArgs& a, const WsLayout& sl, int grid, int nb, int lb, cudaStream_t st) {
  if (nb == 4 && lb == 0) return launch_detect_ws_t<FK_F64, FK_F64, 4, 0>(a, sl, grid, st);
  if (nb == 16 && lb == 4) return launch_detect_ws_t<FK_F64, FK_F64, 16, 4>(a, sl, grid, st);
  return launch_detect_ws_t<FK_F64, FK_F64, 0, 0>(a, sl, grid, st);
}
}  // namespace fpm
