// Warp-per-realization CG (fpm_cgw.cuh) instances for the f16 matvec / inner kind.
#include "fpm_cgw.cuh"
namespace fpm {
int launch_cgw_f16(const CgArgs& a, cudaStream_t st) { return launch_cgw_k<FK_F16>(a, st); }
}  // namespace fpm
