// Warp-per-realization CG (fpm_cgw.cuh) instances for the f32 matvec / inner kind.
#include "fpm_cgw.cuh"
namespace fpm {
int launch_cgw_f32(const CgArgs& a, cudaStream_t st) { return launch_cgw_k<FK_F32>(a, st); }
}  // namespace fpm
