// Lockstep mixed-precision (BJ-)CG over the R realizations resident in one
// CTA, entirely in shared memory.  Restates run_batch (solvers.py:262-393):
//
//   x = 0, r = b, p = BJ ? M r @u_W : r
//   carry = r^H r (plain) | r^H p (BJ textbook)           @u_IP
//   for i = 1..iters:
//     w    = A p                                          @u_MV (A, p rounded once)
//     phi  = p^H w                                        @u_IP
//     rho0 = carry (plain/textbook) | r^H p (BJ as_written)
//     stall = rho0 == 0; breakdown = live & !stall & Re(phi) <= 0
//     alpha = rho0 / phi (NumPy Smith), rounded to u_W
//     xn = x + alpha p ; rn = r + (-alpha) w              @u_W
//     non-finite -> diverged (freeze at the last finite iterate)
//     BJ: z = M r; rho1 = r^H z; beta = rho1/rho0; p = z + beta p
//     plain: rho1 = r^H r;       beta = rho1/rho0; p = r + beta p
//   frozen lanes never resume (so per-lane early exit is exact).
//
// Sequential accumulation order is part of the contract (linalg.py:65-68,
// 94-95): every dot product is ONE dependent chain in one thread, every
// matvec row is one chain; parallelism comes from rows and realizations.
#pragma once
#include "fpm_arith.cuh"

namespace fpm {

template <int MVK>
struct CgSmem {
  typedef typename Ar<MVK>::C MC;
  int R, N, L, nblk, ldA;
  MC* At;          // R * N * ldA, transposed: entry (i,k) at k*ldA + i
  MC* pmv;         // R * N   p rounded to u_MV
  double2* minv;   // R * N*L block inverses (block kb at kb*L*L, row-major Lk x Lk), on the u_W grid
  double2 *b, *x, *r, *p, *z, *w, *xn, *rn;  // R * N each
  double2* sc;     // R * 8 : alpha, beta, phi, rho0, carry, rho1
  int* fl;         // R * 4 : live, nonfinite, breakdown_at, diverged_at
};

// Owner thread of dot product `which` (0/1) of slot g: prefer threads past
// the matvec rows, one per warp, so the chains run in parallel.
__device__ __forceinline__ int dot_owner(int g, int which, int R, int rows, int nthreads) {
  int k = g * 2 + which;
  int cand = nthreads - 1 - 32 * k;
  if (cand >= rows && cand >= 0) return cand;
  return (nthreads - 1 - k) % nthreads;
}

// u^H v over n entries, products and sums at the IP format (dot_fp).
template <int IPK>
__device__ __forceinline__ double2 dot_ip(const double2* u, const double2* v, int n, const FmtP& f) {
  typedef Ar<IPK> A;
  typename A::C s = A::mulc(A::rnd(u[0], f), A::rnd(v[0], f), f);
  for (int k = 1; k < n; ++k) s = A::add(s, A::mulc(A::rnd(u[k], f), A::rnd(v[k], f), f), f);
  double2 d = A::wide(s);
  return assemble(d.x, d.y);
}

// one row of the block-diagonal apply M r (solvers.py:222-225) at u_W
template <int WK>
__device__ __forceinline__ double2 bj_row(const double2* minv, const double2* r, int j, int L, int N,
                                          const FmtP& w) {
  typedef Ar<WK> A;
  const int kb = j / L, jl = j - kb * L;
  const int s0 = kb * L;
  const int Lk = min(L, N - s0);
  const double2* M = minv + kb * L * L + jl * Lk;
  double2 s = A::mul(M[0], A::rnd(r[s0], w), w);
  for (int l = 1; l < Lk; ++l) s = A::add(s, A::mul(M[l], A::rnd(r[s0 + l], w), w), w);
  return assemble(s.x, s.y);
}

template <int WK, int MVK, int IPK>
__device__ void cg_team(CgSmem<MVK>& S, int Rv, int iters, bool bj, bool textbook, const Prec& pr,
                        int nthreads, int tid) {
  typedef Ar<MVK> MV;
  const int N = S.N;
  const int RN = Rv * N;
  const FmtP& fw = pr.work;
  const FmtP& fm = pr.mv;
  const FmtP& fi = pr.ip;

  // ---- init (solvers.py:297-328) ----
  for (int q = tid; q < RN; q += nthreads) {
    S.x[q] = make_double2(0.0, 0.0);
    S.r[q] = S.b[q];
  }
  for (int g = tid; g < Rv; g += nthreads) {
    S.fl[g * 4 + 1] = 0;
    S.fl[g * 4 + 2] = -1;
    S.fl[g * 4 + 3] = -1;
    // fl[g*4+0] (live) is set by the caller (0 if setup failed)
  }
  __syncthreads();
  for (int q = tid; q < RN; q += nthreads) {
    const int g = q / N, i = q - g * N;
    double2 pv = bj ? bj_row<WK>(S.minv + (long)g * N * S.L, S.r + g * N, i, S.L, N, fw) : S.r[q];
    S.p[q] = pv;
    S.pmv[q] = MV::rnd(pv, fm);
  }
  __syncthreads();
  if (!bj || textbook) {
    for (int g = 0; g < Rv; ++g)
      if (tid == dot_owner(g, 0, Rv, RN, nthreads))
        S.sc[g * 8 + 4] = dot_ip<IPK>(S.r + g * N, bj ? S.p + g * N : S.r + g * N, N, fi);
  }
  __syncthreads();

  for (int it = 1; it <= iters; ++it) {
    // ---- w = A p (u_MV), and for BJ as_written rho0 = r^H p ----
    for (int q = tid; q < RN; q += nthreads) {
      const int g = q / N, i = q - g * N;
      if (!S.fl[g * 4]) continue;
      const typename MV::C* col = S.At + (long)g * N * S.ldA + i;
      const typename MV::C* pv = S.pmv + g * N;
      typename MV::C s = MV::mul(col[0], pv[0], fm);
      for (int k = 1; k < N; ++k) s = MV::add(s, MV::mul(col[(long)k * S.ldA], pv[k], fm), fm);
      double2 d = MV::wide(s);
      S.w[q] = assemble(d.x, d.y);
    }
    if (bj && !textbook) {
      for (int g = 0; g < Rv; ++g)
        if (tid == dot_owner(g, 1, Rv, RN, nthreads) && S.fl[g * 4])
          S.sc[g * 8 + 3] = dot_ip<IPK>(S.r + g * N, S.p + g * N, N, fi);
    }
    __syncthreads();
    // ---- phi, flags, alpha ----
    for (int g = 0; g < Rv; ++g) {
      if (tid != dot_owner(g, 0, Rv, RN, nthreads) || !S.fl[g * 4]) continue;
      double2 phi = dot_ip<IPK>(S.p + g * N, S.w + g * N, N, fi);
      double2 rho0 = (bj && !textbook) ? S.sc[g * 8 + 3] : S.sc[g * 8 + 4];
      S.sc[g * 8 + 3] = rho0;
      bool stall = (rho0.x == 0.0) && (rho0.y == 0.0);
      if (!stall && phi.x <= 0.0) S.fl[g * 4 + 2] = it;  // breakdown
      if (stall || phi.x <= 0.0) S.fl[g * 4] = 0;
      S.sc[g * 8 + 0] = wdiv<WK>(rho0, phi, fw);
    }
    __syncthreads();
    // ---- x, r updates (u_W) + finiteness ----
    for (int q = tid; q < RN; q += nthreads) {
      const int g = q / N;
      if (!S.fl[g * 4]) continue;
      const double2 al = S.sc[g * 8 + 0];
      const double2 xn = axpy1<WK>(al, S.p[q], S.x[q], fw);
      const double2 rn = axpy1<WK>(make_double2(-al.x, -al.y), S.w[q], S.r[q], fw);
      S.xn[q] = xn;
      S.rn[q] = rn;
      if (!(finite2(xn) && finite2(rn))) S.fl[g * 4 + 1] = 1;
    }
    __syncthreads();
    for (int q = tid; q < RN; q += nthreads) {  // commit (same thread wrote xn/rn)
      const int g = q / N;
      if (S.fl[g * 4] && !S.fl[g * 4 + 1]) {
        S.x[q] = S.xn[q];
        S.r[q] = S.rn[q];
      }
    }
    __syncthreads();
    if (bj) {
      for (int q = tid; q < RN; q += nthreads) {
        const int g = q / N, i = q - g * N;
        if (S.fl[g * 4] && !S.fl[g * 4 + 1])
          S.z[q] = bj_row<WK>(S.minv + (long)g * N * S.L, S.r + g * N, i, S.L, N, fw);
      }
      __syncthreads();
    }
    // ---- rho1, beta, flags ----
    for (int g = 0; g < Rv; ++g) {
      if (tid != dot_owner(g, 0, Rv, RN, nthreads) || !S.fl[g * 4]) continue;
      if (S.fl[g * 4 + 1]) {  // non-finite update: diverged, frozen
        S.fl[g * 4 + 3] = it;
        S.fl[g * 4] = 0;
        continue;
      }
      double2 rho1 = dot_ip<IPK>(S.r + g * N, bj ? S.z + g * N : S.r + g * N, N, fi);
      S.sc[g * 8 + 1] = wdiv<WK>(rho1, S.sc[g * 8 + 3], fw);
      S.sc[g * 8 + 4] = rho1;
    }
    __syncthreads();
    // ---- p = (z|r) + beta p ; pmv = rnd(p) ----
    int any = 0;
    for (int q = tid; q < RN; q += nthreads) {
      const int g = q / N;
      if (!S.fl[g * 4]) continue;
      any = 1;
      double2 pn = axpy1<WK>(S.sc[g * 8 + 1], S.p[q], bj ? S.z[q] : S.r[q], fw);
      S.p[q] = pn;
      S.pmv[q] = MV::rnd(pn, fm);
    }
    if (!__syncthreads_or(any)) break;
  }
  __syncthreads();
}

}  // namespace fpm
