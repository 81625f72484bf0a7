// Solver warps of the warp-specialised detector (template SW of
// fpm_detect_ws_kernel): instead of one CG group advancing the group's
// realizations in lockstep behind named barriers, each solver warp owns ONE
// realization from the hand-off slot to the write-back, with the arithmetic of
// the warp-per-realization run_batch kernel (fpm_cgw.cuh; solvers.py:262-393):
//
//   * lane l owns rows l, l + 32: x, r, p and its block-inverse rows live in
//     registers; every step is warp-synchronous (no named barrier);
//   * a matvec row is one left-to-right chain in its lane (linalg.py:65-68);
//     for a dot product every lane writes its rows' terms to shared memory and
//     every lane runs the same left-to-right chain (linalg.py:94-95);
//   * freeze semantics (solvers.py:342-357) are an early exit of the warp.
//
// The sequential sums of a realization then cost one warp's issue slots
// instead of an owner thread's with five other warps parked at a barrier, and
// the CG side issues ~40 % fewer instructions per realization: the Gram
// warps, which share the SM sub-partitions' issue ports with it, lose less of
// the FP64 pipe.  A sits in the slot in the run_batch kernel's layout
// (unpadded, 16-byte units XOR-swizzled by row: CgwLayout::at), written there
// by the Gram warps.  u_MV == u_IP native 32-bit (fp16 / bf16), fp64 work.
#pragma once
#include "fpm_bj.cuh"
#include "fpm_cgw.cuh"

namespace fpm {

// per-solver-warp scratch (bytes): the CG's term buffers and binary64 r; the
// block-inverse scratch (Cholesky factors, interleaved over the blocks) and
// its output alias them in time (the inverse rows move to registers first)
template <int K, int NC, int LB>
struct SwScratch {
  typedef typename Ar<K>::C C;
  typedef typename Ar<K>::P P;
  static constexpr int off_pmv = 0;
  static constexpr int off_t0 = off_pmv + NC * (int)sizeof(P);
  static constexpr int off_t1 = off_t0 + NC * (int)sizeof(C);
  static constexpr int off_rv = (off_t1 + NC * (int)sizeof(C) + 15) / 16 * 16;
  static constexpr int cg_bytes = off_rv + (LB > 0 ? NC * 16 : 0);
  static constexpr int inv_bytes = LB > 0 ? 2 * NC * LB * 16 : 0;  // factors + output
  static constexpr int bytes = ((cg_bytes > inv_bytes ? cg_bytes : inv_bytes) + 127) / 128 * 128;
};

// (BJ-)CG of one realization by one warp: At = the realization's A at u_MV
// (CgwLayout::at), bv = its matched filter, m = the lane's block-inverse rows.
// Same operations, in the same order, as fpm_cgw_kernel's sweeps.
template <int K, int NC, int LB>
__device__ __forceinline__ void sw_solve(const typename Ar<K>::C* At, const double2* bv,
                                         const double2 (&m)[NC / 32][LB > 0 ? LB : 1], unsigned char* scr, int iters,
                                         bool textbook, const Prec& pr, int l, double2 (&x)[NC / 32], int& brk,
                                         int& dvg) {
  typedef Ar<K> A;
  typedef typename A::C C;
  typedef typename A::P P;
  typedef SwScratch<K, NC, LB> Lay;
  constexpr int RPL = NC / 32;
  constexpr bool BJ = LB > 0;
  const FmtP& fm = pr.mv;
  const FmtP& fi = pr.ip;
  const FmtP fw{};  // work = binary64 (identity rounding)
  P* pmv = reinterpret_cast<P*>(scr + Lay::off_pmv);
  C* tb0 = reinterpret_cast<C*>(scr + Lay::off_t0);  // rho0 = r^H p terms (as_written BJ) / rho1, carry terms
  C* tb1 = reinterpret_cast<C*>(scr + Lay::off_t1);  // phi = p^H w terms
  C* tb2 = tb0;
  double2* rv = reinterpret_cast<double2*>(scr + Lay::off_rv);
  const bool rho_fresh = BJ && !textbook;  // as_written: rho0 = r^H p every sweep
  double2 r[RPL], p[RPL];
  C pm[RPL];
  auto zrow = [&](int j) -> double2 {
    const int i = l + 32 * j;
    return bj_z<(LB > 0 ? LB : 1)>(m[j], rv, i - i % (LB > 0 ? LB : 1));
  };
  // ---- init (solvers.py:297-328): p = M r | r; carry = r^H r | r^H p ----
#pragma unroll
  for (int j = 0; j < RPL; ++j) {
    x[j] = make_double2(0.0, 0.0);
    r[j] = bv[l + 32 * j];
  }
  if constexpr (BJ) {
#pragma unroll
    for (int j = 0; j < RPL; ++j) rv[l + 32 * j] = r[j];
    __syncwarp();
  }
#pragma unroll
  for (int j = 0; j < RPL; ++j) {
    if constexpr (BJ) p[j] = zrow(j);
    else p[j] = r[j];
  }
#pragma unroll
  for (int j = 0; j < RPL; ++j) {
    const int i = l + 32 * j;
    pm[j] = A::rnd(p[j], fm);
    pmv[i] = A::prep(pm[j]);
    const C ri = A::rnd(r[j], fi);
    tb0[i] = A::mulc(ri, (BJ && (textbook || rho_fresh)) ? pm[j] : ri, fi);
  }
  __syncwarp();
  double2 carry = make_double2(0.0, 0.0);
  if (!rho_fresh) carry = wsum<K, NC>(tb2, fi);
#pragma unroll 1
  for (int it = 1; it <= iters; ++it) {
    // ---- w = A p (u_MV) ; rho0 (as_written BJ) ; phi = p^H w (u_IP) ----
    C wc[RPL];
    double2 rho0 = carry;
    mv_rows<K, NC, RPL, 32>(At, pmv, l, wc, fm);
    if (rho_fresh) rho0 = wsum<K, NC>(tb0, fi);
#pragma unroll
    for (int j = 0; j < RPL; ++j) tb1[l + 32 * j] = A::mulc(pm[j], wc[j], fi);
    __syncwarp();
    const double2 phi = wsum<K, NC>(tb1, fi);
    // stall / breakdown freeze the realization (solvers.py:342-345)
    const bool stall = (rho0.x == 0.0) && (rho0.y == 0.0);
    if (!stall && phi.x <= 0.0) brk = it;
    if (stall || phi.x <= 0.0) break;
    const double2 al = cgw_div<K>(rho0, phi);
    const double2 nal = make_double2(-al.x, -al.y);
    // ---- x, r updates at u_W; non-finite -> diverged (solvers.py:346-354) ----
    double2 xn[RPL], rn[RPL];
    bool bad = false;
#pragma unroll
    for (int j = 0; j < RPL; ++j) {
      xn[j] = axpy1<FK_F64>(al, p[j], x[j], fw);
      rn[j] = axpy1<FK_F64>(nal, A::wide(wc[j]), r[j], fw);
      bad |= !(finite2(xn[j]) && finite2(rn[j]));
    }
    if (__any_sync(0xffffffffu, bad)) {
      dvg = it;
      break;
    }
#pragma unroll
    for (int j = 0; j < RPL; ++j) {
      x[j] = xn[j];
      r[j] = rn[j];
    }
    // ---- z = M r ; rho1 = r^H z | r^H r ; beta = rho1 / rho0 ----
    double2 z[RPL];
    if constexpr (BJ) {
#pragma unroll
      for (int j = 0; j < RPL; ++j) rv[l + 32 * j] = r[j];
      __syncwarp();
#pragma unroll
      for (int j = 0; j < RPL; ++j) z[j] = zrow(j);
    }
    C ri[RPL];
#pragma unroll
    for (int j = 0; j < RPL; ++j) {
      ri[j] = A::rnd(r[j], fi);
      tb2[l + 32 * j] = A::mulc(ri[j], BJ ? A::rnd(z[j], fi) : ri[j], fi);
    }
    __syncwarp();
    const double2 rho1 = wsum<K, NC>(tb2, fi);
    const double2 be = cgw_div<K>(rho1, rho0);
    carry = rho1;
    __syncwarp();  // every lane's rho1 chain has read tb2 (= tb0's storage)
    // ---- p = (z | r) + beta p ; prepared p and next rho0 terms ----
#pragma unroll
    for (int j = 0; j < RPL; ++j) {
      const int i = l + 32 * j;
      p[j] = axpy1<FK_F64>(be, p[j], BJ ? z[j] : r[j], fw);
      pm[j] = A::rnd(p[j], fm);
      pmv[i] = A::prep(pm[j]);
      if (rho_fresh) tb0[i] = A::mulc(ri[j], pm[j], fi);
    }
    __syncwarp();
  }
}

}  // namespace fpm
