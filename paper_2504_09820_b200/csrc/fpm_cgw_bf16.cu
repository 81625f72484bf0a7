// Warp-per-realization CG (fpm_cgw.cuh) instances for the bf16 matvec / inner kind.
#include "fpm_cgw.cuh"
namespace fpm {
int launch_cgw_bf16(const CgArgs& a, cudaStream_t st) { return launch_cgw_k<FK_BF16>(a, st); }
}  // namespace fpm
