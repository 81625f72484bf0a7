// Warp-per-realization CG (fpm_cgw.cuh) instances for the f64 matvec / inner kind.
#include "fpm_cgw.cuh"
namespace fpm {
int launch_cgw_f64(const CgArgs& a, cudaStream_t st) { return launch_cgw_k<FK_F64>(a, st); }
}  // namespace fpm
