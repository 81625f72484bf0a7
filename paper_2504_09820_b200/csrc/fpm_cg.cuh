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
// 94-95).  Latency design: the product terms of every dot product are
// formed in parallel by the row threads (each is an independent rounded
// complex multiply), and only the left-to-right SUM runs as one dependent
// chain in one thread per realization; matvec rows are chains in parallel.
// Six CTA barriers per iteration.
#pragma once
#include "fpm_arith.cuh"

namespace fpm {

template <int MVK, int IPK>
struct CgSmem {
  typedef typename Ar<MVK>::C MC;
  typedef typename Ar<IPK>::C IC;
  int R, N, L, ldA;
  MC* At;          // R * N * ldA, transposed: entry (i,k) at k*ldA + i
  MC* pmv;         // R * N   p rounded to u_MV
  IC *tphi, *trho, *tr1;  // R * N product terms of p^H w, r^H p, r^H z (or r^H r)
  double2* minv;   // R * N*L block inverses (block kb at kb*L*L, row-major Lk x Lk), on the u_W grid
  double2 *b, *x, *r, *p, *z, *w, *xn, *rn;  // R * N each
  double2* sc;     // R * 8 : 0 alpha, 1 beta, 3 rho0, 4 carry
  int* fl;         // R * 4 : live, nonfinite, breakdown_at, diverged_at
};

// Owner of the sequential sums of slot g: past the matvec rows when possible,
// one warp apart so the R chains run in parallel.
__device__ __forceinline__ int dot_owner(int g, int which, int rows, int nthreads) {
  int k = g * 2 + which;
  int cand = nthreads - 1 - 32 * k;
  if (cand >= rows && cand >= 0) return cand;
  return (nthreads - 1 - k) % nthreads;
}

// left-to-right sum t_0 + t_1 + ... (dot_fp's accumulation, linalg.py:94-95)
template <int IPK>
__device__ __forceinline__ double2 chain_sum(const typename Ar<IPK>::C* t, int n, const FmtP& f) {
  typedef Ar<IPK> A;
  typename A::C s = t[0];
  int k = 1;
  for (; k + 8 <= n; k += 8) {
    typename A::C v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = t[k + j];
#pragma unroll
    for (int j = 0; j < 8; ++j) s = A::add(s, v[j], f);
  }
  for (; k < n; ++k) s = A::add(s, t[k], f);
  double2 d = A::wide(s);
  return assemble(d.x, d.y);
}

// conj(u) * v term at the IP format (inputs rounded into it, dot_fp)
template <int IPK>
__device__ __forceinline__ typename Ar<IPK>::C ip_term(double2 u, double2 v, const FmtP& f) {
  typedef Ar<IPK> A;
  return A::mulc(A::rnd(u, f), A::rnd(v, f), f);
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

// w_i = sum_k A(i,k) p_k at u_MV (matvec_fp), A column-major in shared memory
template <int MVK>
__device__ __forceinline__ double2 mv_row(const typename Ar<MVK>::C* col, const typename Ar<MVK>::C* pv, int N,
                                          int ldA, const FmtP& f) {
  typedef Ar<MVK> A;
  typename A::C s = A::mul(col[0], pv[0], f);
  int k = 1;
  for (; k + 8 <= N; k += 8) {
    typename A::C t[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) t[j] = A::mul(col[(long)(k + j) * ldA], pv[k + j], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) s = A::add(s, t[j], f);
  }
  for (; k < N; ++k) s = A::add(s, A::mul(col[(long)k * ldA], pv[k], f), f);
  double2 d = A::wide(s);
  return assemble(d.x, d.y);
}

// phase timestamps (diagnostic): thread 0 of CTA 0 writes clock64 values
#define FPM_STAMP(tr, k)                                      \
  do {                                                        \
    if ((tr) && tid == 0) (tr)[(k)] = (long long)clock64();   \
  } while (0)

template <int WK, int MVK, int IPK>
__device__ void cg_team(CgSmem<MVK, IPK>& S, int Rv, int iters, bool bj, bool textbook, const Prec& pr,
                        int nthreads, int tid, long long* tr = nullptr) {
  typedef Ar<MVK> MV;
  const int N = S.N;
  const int RN = Rv * N;
  const FmtP& fw = pr.work;
  const FmtP& fm = pr.mv;
  const FmtP& fi = pr.ip;
  const bool rho_fresh = bj && !textbook;  // as_written: rho0 = r^H p every sweep

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
    const double2 rv = S.r[q];
    const double2 pv = bj ? bj_row<WK>(S.minv + (long)g * N * S.L, S.r + g * N, i, S.L, N, fw) : rv;
    S.p[q] = pv;
    S.pmv[q] = MV::rnd(pv, fm);
    S.tr1[q] = ip_term<IPK>(rv, (bj && textbook) ? pv : rv, fi);  // carry terms
    if (rho_fresh) S.trho[q] = ip_term<IPK>(rv, pv, fi);
  }
  __syncthreads();
  if (!rho_fresh) {
    for (int g = 0; g < Rv; ++g)
      if (tid == dot_owner(g, 0, RN, nthreads)) S.sc[g * 8 + 4] = chain_sum<IPK>(S.tr1 + g * N, N, fi);
  }
  __syncthreads();

  for (int it = 1; it <= iters; ++it) {
    // ---- A: w = A p (u_MV) + phi terms;  rho0 = sum r^H p (BJ as_written) ----
    for (int q = tid; q < RN; q += nthreads) {
      const int g = q / N, i = q - g * N;
      if (!S.fl[g * 4]) continue;
      const double2 wv = mv_row<MVK>(S.At + (long)g * N * S.ldA + i, S.pmv + g * N, N, S.ldA, fm);
      S.w[q] = wv;
      S.tphi[q] = ip_term<IPK>(S.p[q], wv, fi);
    }
    if (rho_fresh) {
      for (int g = 0; g < Rv; ++g)
        if (tid == dot_owner(g, 1, RN, nthreads) && S.fl[g * 4])
          S.sc[g * 8 + 3] = chain_sum<IPK>(S.trho + g * N, N, fi);
    }
    __syncthreads();
    if (it == 1) FPM_STAMP(tr, 0);
    // ---- B: phi, flags, alpha ----
    for (int g = 0; g < Rv; ++g) {
      if (tid != dot_owner(g, 0, RN, nthreads) || !S.fl[g * 4]) continue;
      const double2 phi = chain_sum<IPK>(S.tphi + g * N, N, fi);
      const double2 rho0 = rho_fresh ? S.sc[g * 8 + 3] : S.sc[g * 8 + 4];
      S.sc[g * 8 + 3] = rho0;
      const bool stall = (rho0.x == 0.0) && (rho0.y == 0.0);
      if (!stall && phi.x <= 0.0) S.fl[g * 4 + 2] = it;  // breakdown
      if (stall || phi.x <= 0.0) S.fl[g * 4] = 0;
      S.sc[g * 8 + 0] = wdiv<WK>(rho0, phi, fw);
    }
    __syncthreads();
    if (it == 1) FPM_STAMP(tr, 1);
    // ---- C: x, r updates (u_W) + finiteness ----
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
    if (it == 1) FPM_STAMP(tr, 2);
    // ---- D: commit; z = M r_new; rho1 terms ----
    for (int q = tid; q < RN; q += nthreads) {
      const int g = q / N, i = q - g * N;
      if (!S.fl[g * 4] || S.fl[g * 4 + 1]) continue;
      const double2 rn = S.rn[q];
      S.x[q] = S.xn[q];
      S.r[q] = rn;
      if (bj) {
        const double2 zv = bj_row<WK>(S.minv + (long)g * N * S.L, S.rn + g * N, i, S.L, N, fw);
        S.z[q] = zv;
        S.tr1[q] = ip_term<IPK>(rn, zv, fi);
      } else {
        S.tr1[q] = ip_term<IPK>(rn, rn, fi);
      }
    }
    __syncthreads();
    if (it == 1) FPM_STAMP(tr, 3);
    // ---- E: rho1, beta, divergence flag ----
    for (int g = 0; g < Rv; ++g) {
      if (tid != dot_owner(g, 0, RN, nthreads) || !S.fl[g * 4]) continue;
      if (S.fl[g * 4 + 1]) {  // non-finite update: diverged, frozen at the last finite iterate
        S.fl[g * 4 + 3] = it;
        S.fl[g * 4] = 0;
        continue;
      }
      const double2 rho1 = chain_sum<IPK>(S.tr1 + g * N, N, fi);
      S.sc[g * 8 + 1] = wdiv<WK>(rho1, S.sc[g * 8 + 3], fw);
      S.sc[g * 8 + 4] = rho1;
    }
    __syncthreads();
    if (it == 1) FPM_STAMP(tr, 4);
    // ---- F: p = (z|r) + beta p ; pmv = rnd(p) ; next rho0 terms ----
    int any = 0;
    for (int q = tid; q < RN; q += nthreads) {
      const int g = q / N;
      if (!S.fl[g * 4]) continue;
      any = 1;
      const double2 pn = axpy1<WK>(S.sc[g * 8 + 1], S.p[q], bj ? S.z[q] : S.r[q], fw);
      S.p[q] = pn;
      S.pmv[q] = MV::rnd(pn, fm);
      if (rho_fresh) S.trho[q] = ip_term<IPK>(S.r[q], pn, fi);
    }
    const int more = __syncthreads_or(any);
    if (it == 1) FPM_STAMP(tr, 5);
    if (!more) break;
  }
  __syncthreads();
  FPM_STAMP(tr, 6);
}

}  // namespace fpm
