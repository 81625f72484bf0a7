// Block-Jacobi setup: Hermitian-PD inverse of one Lk x Lk diagonal block.
//
// The reference (solvers.py:232-253) checks PD with a Cholesky
// (np.linalg.cholesky, :246-249), inverts with LAPACK zgesv against the
// identity (:250-251) and symmetrizes 0.5(inv + inv^H) (:252).  LAPACK bits
// are not portable, so this is an fp64 Cholesky-based inverse with the same
// PD test; parity is a tolerance (or the inverses are injected).  The result
// is exactly Hermitian (upper computed, lower mirrored, real diagonal), as
// the reference's symmetrization makes it.
//
// Layout: input block entry (i,j) at B[(i*Lk+j)*sb], scratch at
// C[(i*Lk+j)*sc] -- interleaved across the threads that each own one block,
// so every shared-memory access is conflict-free; output column-major
// (entry (i,j) at out[j*Lk+i]) for the CG's block apply.  LB > 0 fixes the
// block size at compile time (fully unrolled).
#pragma once
#include <cuda_runtime.h>

namespace fpm {

template <int LB>
__device__ __forceinline__ bool hpd_inverse(const double2* B, int sb, double2* C, int sc, double2* out, int Lk_rt) {
  const int Lk = LB > 0 ? LB : Lk_rt;
#define FPM_B(i, j) B[((i) * Lk + (j)) * sb]
#define FPM_C(i, j) C[((i) * Lk + (j)) * sc]
  // Cholesky B = L L^H (lower), reciprocal pivots kept on the diagonal
#pragma unroll
  for (int j = 0; j < Lk; ++j) {
    double d = FPM_B(j, j).x;
#pragma unroll
    for (int k = 0; k < j; ++k) {
      const double2 c = FPM_C(j, k);
      d = d - (c.x * c.x + c.y * c.y);
    }
    if (!(d > 0.0)) return false;
    const double rs = 1.0 / sqrt(d);
    FPM_C(j, j) = make_double2(rs, 0.0);
#pragma unroll
    for (int i = j + 1; i < Lk; ++i) {
      double2 s = FPM_B(i, j);
#pragma unroll
      for (int k = 0; k < j; ++k) {
        const double2 a = FPM_C(i, k), b = FPM_C(j, k);  // s -= a * conj(b)
        s.x -= a.x * b.x + a.y * b.y;
        s.y -= a.y * b.x - a.x * b.y;
      }
      FPM_C(i, j) = make_double2(s.x * rs, s.y * rs);
    }
  }
  // Linv = L^-1 in place, columns right to left, rows bottom up:
  //   Linv(i,j) = -Linv(j,j) * sum_{k=j+1}^{i} Linv(i,k) L(k,j)
#pragma unroll
  for (int j = Lk - 1; j >= 0; --j) {
    const double rj = FPM_C(j, j).x;
#pragma unroll
    for (int i = Lk - 1; i > j; --i) {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = j + 1; k <= i; ++k) {
        const double2 a = FPM_C(i, k), b = FPM_C(k, j);
        s.x += a.x * b.x - a.y * b.y;
        s.y += a.x * b.y + a.y * b.x;
      }
      FPM_C(i, j) = make_double2(-s.x * rj, -s.y * rj);
    }
  }
  // Minv = Linv^H Linv: upper computed, mirrored, diagonal real
#pragma unroll
  for (int i = 0; i < Lk; ++i)
#pragma unroll
    for (int j = i; j < Lk; ++j) {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = j; k < Lk; ++k) {
        const double2 a = FPM_C(k, i), b = FPM_C(k, j);  // conj(a) * b
        s.x += a.x * b.x + a.y * b.y;
        s.y += a.x * b.y - a.y * b.x;
      }
      if (i == j) {
        out[i * Lk + i] = make_double2(s.x, 0.0);
      } else {
        out[j * Lk + i] = s;                        // (i,j)
        out[i * Lk + j] = make_double2(s.x, -s.y);  // (j,i)
      }
    }
#undef FPM_B
#undef FPM_C
  return true;
}

}  // namespace fpm
