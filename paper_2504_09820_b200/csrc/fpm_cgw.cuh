// Warp-per-realization (BJ-)CG: the run_batch boundary's fast path
// (solvers.py:262-393, same arithmetic contract as cg_group in fpm_cg.cuh).
//
// One warp owns one realization for its whole life: it streams the
// realization's complex128 A from HBM (coalesced 16-byte loads, many in
// flight), rounds it ONCE to u_MV into its private shared-memory matrix
// (formats.py:110-146 via cvt.rn / native ops, linalg.py:60-61), then runs
// every sweep with warp-synchronous steps only (__syncwarp, no CTA barriers):
//
//   * lane l owns rows l, l+32, ... (RPL = N/32 rows): x, r, p, w and its
//     block-Jacobi inverse rows live in registers;
//   * a matvec row is one left-to-right chain in its lane (linalg.py:65-68);
//   * a dot product u^H v: every lane forms the product terms of its rows,
//     writes them to shared memory, and then EVERY lane runs the same
//     left-to-right chain over all N terms (broadcast loads,
//     linalg.py:94-95), so the scalar is warp-uniform with no broadcast step
//     and the freeze / stall / breakdown decisions are warp-uniform branches;
//   * alpha, beta: NumPy's Smith division in binary64 (solvers.py:256-259).
//
// Freeze semantics (solvers.py:342-357) become an early exit of the warp.
// CTAs are one warp, so the block scheduler refills an SM as soon as any
// realization finishes and loading (HBM latency) overlaps other warps' sweeps.
// Work format fp64 and u_MV == u_IP native (fp64 / fp32 / fp16 / bf16), N in
// {32, 64}, plain CG or block-Jacobi with L in {1, 2, 4, 8} (with or without
// the run_batch histories); everything else runs fpm_cg_kernel.
#pragma once
#include "../../include/fpmimo_b200.h"
#include "fpm_common.cuh"
#include "fpm_ptx.cuh"

#include <cstdlib>


namespace fpm {

#ifndef FPM_CGW_PREFETCH
#define FPM_CGW_PREFETCH 1
#endif
// alpha / beta: NumPy's Smith division at u_W = binary64 (the rounding to
// u_W is the identity).  Inline for 32-bit u_MV (c5 fp16 55.6 -> 56.5 M/s);
// the shared __noinline__ wdiv for 16-byte u_MV, whose kernels are
// register-bound (inline measured 13.5 -> 13.1 M/s at fp64).
template <int K>
__device__ __forceinline__ double2 cgw_div(double2 n, double2 d) {
  if constexpr (sizeof(typename Ar<K>::C) >= 16) return wdiv<FK_F64>(n, d, FmtP{});
  else return cdiv(n, d);
}
#define CGW_DIV(n, d) cgw_div<K>((n), (d))
#ifndef FPM_CGW_LOADS
#define FPM_CGW_LOADS 16
#endif

// Per-realization shared-memory region.  A is unpadded (N*N entries at
// u_MV) with an XOR swizzle on its 16-byte units, unit u of row i stored at
// u ^ (i & 7): the 8 rows one LDS.128 quarter-warp phase reads fall on 8
// distinct bank groups.  Scratch after A: the prepared p, the rho0 / rho1
// term buffer (live ranges [p update, matvec] and [r update, rho1] are
// disjoint, so one buffer), the phi terms and the binary64 r that z = M r
// reads.  N = 64 fp16: 18,432 B (12 warps / SM).
template <int K, int NC, int LB>
struct CgwLayout {
  typedef typename Ar<K>::C C;
  typedef typename Ar<K>::P P;
  static constexpr int EPU = 16 / (int)sizeof(C);  // entries per 16-byte unit
  static constexpr int UPR = NC / EPU;             // units per row (>= 8)
  static_assert(UPR % 8 == 0, "swizzle needs >= 8 units per row");
  static constexpr int a_bytes = NC * NC * (int)sizeof(C);
  static constexpr int off_pmv = a_bytes;
  static constexpr int off_t0 = off_pmv + NC * (int)sizeof(P);
  static constexpr int off_t1 = off_t0 + NC * (int)sizeof(C);
  static constexpr int off_t2 = off_t0;
  static constexpr int off_rv = (off_t1 + NC * (int)sizeof(C) + 15) / 16 * 16;
  // block-inverse rows: registers unless a lane would hold more than 8
  static constexpr bool MS = (NC / 32) * LB > 8;
  static constexpr int off_ms = off_rv + (LB > 0 ? NC * 16 : 0);
  static constexpr int bytes = off_ms + (MS ? NC * LB * 16 : 0);
  // element offset of A(i, k)
  static __device__ __forceinline__ int at(int i, int k) {
    return (i * UPR + ((k / EPU) ^ (i & 7))) * EPU + k % EPU;
  }
};

// w_i = sum_k A(i,k) p_k (matvec_fp, linalg.py:45-69) for the lane's RPL
// rows: one left-to-right chain per row, the rows' chains interleaved block
// by block; the prepared p block is shared by the rows.  (Folding the
// as-written rho0 = r^H p chain into this loop as one more chain measured
// 1.5 % slower at fp16 and 13 % at fp64: register pressure.)
template <int K, int NC, int RPL, int LPR>
__device__ __forceinline__ void mv_rows(const typename Ar<K>::C* At, const typename Ar<K>::P* pv, int lane,
                                        typename Ar<K>::C (&out)[RPL], const FmtP& f) {
  typedef Ar<K> A;
  typedef typename A::C C;
  typedef typename A::P P;
  constexpr int B = V16<C>::n;  // entries per 16-byte unit (= per block)
  constexpr int NB = NC / B;
  static_assert(B == 16 / (int)sizeof(C), "one 16-byte unit per block");
  const C* row[RPL];
  int sw[RPL];
#pragma unroll
  for (int j = 0; j < RPL; ++j) {
    const int i = lane + LPR * j;
    row[j] = At + i * NC;
    sw[j] = i & 7;
  }
  C s[RPL];
#pragma unroll
  for (int kb = 0; kb < NB; ++kb) {
    P p[B];
    ld_blk<B>(pv + kb * B, p);
#pragma unroll
    for (int j = 0; j < RPL; ++j) {
      C a[B];
      ld_blk<B>(row[j] + (kb ^ sw[j]) * B, a);
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const C t = A::mulp(a[u], p[u], f);
        s[j] = (kb + u == 0) ? t : A::add(s[j], t, f);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < RPL; ++j) out[j] = A::asmc(s[j]);
}

// left-to-right sum of the NC terms in shared memory (dot_fp's
// accumulation, linalg.py:94-95), run identically by every lane
template <int K, int NC>
__device__ __forceinline__ double2 wsum(const typename Ar<K>::C* t, const FmtP& f) {
  typedef Ar<K> A;
  typedef typename A::C C;
  constexpr int B = V16<C>::n;
  constexpr int NB = NC / B;
  C s;
#pragma unroll
  for (int kb = 0; kb < NB; ++kb) {
    C v[B];
    ld_blk<B>(t + kb * B, v);
#pragma unroll
    for (int u = 0; u < B; ++u) s = (kb + u == 0) ? v[u] : A::add(s, v[u], f);
  }
  return A::wide(A::asmc(s));
}

// z_i = sum_l Minv(i, l) r_(block start + l) at u_W = fp64 (_BatchBlocks.apply,
// solvers.py:222-225 -> matvec_fp at u_W), r from shared memory
template <int LB>
__device__ __forceinline__ double2 bj_z(const double2 (&m)[LB], const double2* rv, int s0) {
  typedef Ar<FK_F64> W;
  const FmtP f{};
  double2 s = W::mul(m[0], rv[s0], f);
#pragma unroll
  for (int l = 1; l < LB; ++l) s = W::add(s, W::mul(m[l], rv[s0 + l], f), f);
  return assemble(s.x, s.y);
}

// ---- tensor memory (TMEM) as the matrix store -----------------------------
// 32x32b shapes: lane l of the warp reads / writes TMEM lane (32 * (warp % 4)
// + l), consecutive 32-bit columns.  tcgen05.ld / st complete asynchronously;
// tm_wait_ld / tm_wait_st wait for all of this thread's outstanding ones, and
// tm_launder makes the loaded registers' consumers depend on the wait (the
// compiler sees the ld's outputs as defined at the ld itself).
__device__ __forceinline__ void tm_ld8(uint32_t (&v)[8], uint32_t taddr) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tm_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_launder(uint32_t (&v)[8]) {
  asm volatile("" : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]));
}

// w = A p for rows l and l+32 with A in TMEM (row l: columns [0, 64), row
// l+32: [64, 128), one 32-bit u_MV complex per column): 8-column blocks, the
// next block's tcgen05.ld in flight while this block's products and sums run.
template <int K>
__device__ __forceinline__ void mv_rows_tm(uint32_t ta, const typename Ar<K>::P* pv, typename Ar<K>::C (&out)[2],
                                           const FmtP& f) {
  typedef Ar<K> A;
  typedef typename A::C C;
  typedef typename A::P P;
  static_assert(sizeof(C) == 4, "TMEM matvec: 32-bit complex entries");
  uint32_t ra[2][2][8];
  tm_ld8(ra[0][0], ta);
  tm_ld8(ra[0][1], ta + 64);
  tm_wait_ld();
  tm_launder(ra[0][0]);
  tm_launder(ra[0][1]);
  C s[2];
#pragma unroll
  for (int kb = 0; kb < 8; ++kb) {
    const int cur = kb & 1;
    if (kb < 7) {
      tm_ld8(ra[cur ^ 1][0], ta + 8 * (kb + 1));
      tm_ld8(ra[cur ^ 1][1], ta + 64 + 8 * (kb + 1));
    }
    P p[8];
    ld_blk<8>(pv + 8 * kb, p);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        uint32_t w = ra[cur][j][u];
        const C t = A::mulp(*reinterpret_cast<C*>(&w), p[u], f);
        s[j] = (kb + u == 0) ? t : A::add(s[j], t, f);
      }
    }
    if (kb < 7) {
      tm_wait_ld();
      tm_launder(ra[cur ^ 1][0]);
      tm_launder(ra[cur ^ 1][1]);
    }
  }
  out[0] = A::asmc(s[0]);
  out[1] = A::asmc(s[1]);
}

// Block-inverse rows in shared memory (when they do not fit in registers:
// RPL * L > 8, and in the TMEM variant): row i's entry k at unit
// ms_unit(i, k) of its L-unit row, so 8 lanes reading 8 consecutive rows'
// entry k hit 8 distinct 16-byte bank groups.
template <int LB>
__device__ __forceinline__ int ms_unit(int i, int k) {
  if constexpr (LB >= 8) return (k + i) & (LB - 1);
  else if constexpr (LB == 4) return (k + (i >> 1)) & 3;
  else if constexpr (LB == 2) return (k + (i >> 2)) & 1;
  else return 0;
}

template <int LB>
__device__ __forceinline__ double2 bj_z_s(const double2* ms, int i, const double2* rv, int s0) {
  static_assert((LB & (LB - 1)) == 0, "power-of-two block size");
  typedef Ar<FK_F64> W;
  const FmtP f{};
  const double2* mr = ms + i * LB;
  double2 s = W::mul(mr[ms_unit<LB>(i, 0)], rv[s0], f);
#pragma unroll
  for (int k = 1; k < LB; ++k) s = W::add(s, W::mul(mr[ms_unit<LB>(i, k)], rv[s0 + k], f), f);
  return assemble(s.x, s.y);
}

// One warp (= one CTA) per realization; the block scheduler refills an SM as
// soon as any realization finishes, so one warp's HBM load phase overlaps the
// other resident warps' sweeps.  (A persistent grid that bulk-prefetches each
// warp's next A into L2 -- cp.async.bulk.prefetch.L2 -- measured slower at c5
// fp16, 48.3 M vs 51.7 M/s: one fewer resident warp per SM, and the
// L2-sourced load phase still took ~11 K cycles.)
// norm2 (linalg.py:122-134) of the realization's vector held two rows per
// lane: scale = max |v_k| (NaN-propagating; 1 if not a finite positive
// number), scale * sqrt(sum (|v_k| / scale)^2), inf if any |v_k| is inf.  The
// sum runs as a warp tree (NumPy's pairwise sum and the lockstep kernel's
// sequential sum differ from it, and from each other, in the last bits only).
template <int RPL>
__device__ __forceinline__ double cgw_norm2(const double2 (&v)[RPL]) {
  double h[RPL], scale = 0.0;
  bool nan = false, inf = false;
#pragma unroll
  for (int j = 0; j < RPL; ++j) {
    h[j] = hypot(v[j].x, v[j].y);
    nan |= isnan(h[j]);
    inf |= isinf(h[j]);
    scale = h[j] > scale ? h[j] : scale;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, scale, o);
    scale = u > scale ? u : scale;
  }
  nan = __any_sync(0xffffffffu, nan);
  inf = __any_sync(0xffffffffu, inf);
  if (nan || !isfinite(scale) || !(scale > 0.0)) scale = 1.0;
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < RPL; ++j) {
    const double q = __ddiv_rn(h[j], scale);
    s = __dadd_rn(s, __dmul_rn(q, q));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  const double out = __dmul_rn(scale, __dsqrt_rn(s));
  return inf ? __longlong_as_double(0x7ff0000000000000LL) : out;
}

// TM = false: one warp per CTA, A at u_MV in shared memory (CgwLayout).
// TM = true (N = 64, 32-bit u_MV entries, L in {0, 4}; opt-in, see
// launch_cgw_t): four warps per CTA,
// each warp's A in its TMEM lane quarter (128 columns per CTA), the
// block-inverse rows in shared memory: the shared-memory footprint drops from
// 18 KB to 6 KB per realization, so registers, not shared memory, bound the
// resident warps (16 per SM at <= 128 registers).
template <int K, int NC, int LB, bool TM>
struct CgwTmLayout {
  typedef typename Ar<K>::C C;
  typedef typename Ar<K>::P P;
  static constexpr int off_pmv = 0;
  static constexpr int off_t0 = off_pmv + NC * (int)sizeof(P);
  static constexpr int off_t1 = off_t0 + NC * (int)sizeof(C);
  static constexpr int off_t2 = off_t0;
  static constexpr int off_rv = (off_t1 + NC * (int)sizeof(C) + 15) / 16 * 16;
  static constexpr int off_ms = off_rv + (LB > 0 ? NC * 16 : 0);
  static constexpr int bytes_ = off_ms + NC * LB * 16;
  static constexpr int stage = NC * 16 * 4;  // 16-column staging tile (aliases rv / ms)
  static constexpr int bytes = off_rv + stage > bytes_ ? off_rv + stage : bytes_;
  static constexpr int head = 128;  // TMEM address slot
  static constexpr int cta_bytes = head + 4 * bytes;
};

template <int K, int NC, int LB, bool TM, bool HIST>
__global__ void __launch_bounds__(TM ? 128 : 32, TM ? 4 : 1) fpm_cgw_kernel(const CgArgs args) {
  extern __shared__ __align__(128) unsigned char smem[];
  typedef Ar<K> A;
  typedef typename A::C C;
  typedef typename A::P P;
  typedef CgwLayout<K, NC, LB> Lay;
  typedef CgwTmLayout<K, NC, LB, TM> TLay;
  constexpr int RPL = NC / 32;  // rows per lane
  constexpr bool BJ = LB > 0;
  constexpr int NN = NC * NC;
  static_assert(!TM || (NC == 64 && sizeof(C) == 4 && (LB == 0 || LB == 4)), "TMEM variant: N = 64, 32-bit u_MV");
  const int l = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long t = TM ? (long)blockIdx.x * 4 + wid : (long)blockIdx.x;
  const bool valid = t < args.T;
  const FmtP& fm = args.pr.mv;
  const FmtP& fi = args.pr.ip;
  const FmtP fw{};  // work = binary64 (identity rounding)
  unsigned char* base = TM ? smem + TLay::head + wid * TLay::bytes : smem;
  C* At = reinterpret_cast<C*>(smem);
  P* pmv = reinterpret_cast<P*>(base + (TM ? TLay::off_pmv : Lay::off_pmv));
  C* tb0 = reinterpret_cast<C*>(base + (TM ? TLay::off_t0 : Lay::off_t0));  // rho0 = r^H p terms (as_written BJ)
  C* tb1 = reinterpret_cast<C*>(base + (TM ? TLay::off_t1 : Lay::off_t1));  // phi = p^H w terms
  C* tb2 = reinterpret_cast<C*>(base + (TM ? TLay::off_t2 : Lay::off_t2));  // rho1 / carry terms (tb0's storage)
  double2* rv = reinterpret_cast<double2*>(base + (TM ? TLay::off_rv : Lay::off_rv));
  constexpr bool MS = TM || Lay::MS;  // block-inverse rows in shared memory
  double2* ms = reinterpret_cast<double2*>(base + (TM ? TLay::off_ms : Lay::off_ms));
  const bool rho_fresh = BJ && !args.textbook;  // as_written: rho0 = r^H p every sweep
  uint32_t ta = 0;  // TM: this warp's TMEM base (lane quarter wid, 128 columns)
  if constexpr (TM) {
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem);
    if (wid == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    ta = *slot + ((uint32_t)(32 * wid) << 16);
  }

  if (valid) {
    long long* trc = diag_trace(args.trace) ? diag_trace(args.trace) + 4 * t : nullptr;  // diagnostic per-realization clocks
    if (trc && l == 0) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      trc[0] = clock64();
      trc[3] = sm;
    }
    // ---- A (complex128, row-major) -> u_MV, one rounding per entry ----
    // One bulk L2 prefetch of the whole matrix first: HBM sees all of this
    // realization's bytes requested at once (memory-level parallelism without
    // registers), the loads below then mostly wait on L2, not on HBM.
#if FPM_CGW_PREFETCH
    if (l == 0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(args.A + t * NN), "r"(NN * 16) : "memory");
#endif
    if constexpr (TM) {
      // 16-column chunks of all 64 rows: coalesced loads (two 256-byte row
      // segments per warp load), rounded into a shared-memory staging tile
      // (16-byte unit v of row i at v ^ ((i >> 1) & 3): conflict-free both
      // ways), then lane l moves rows l and l+32 into its TMEM lane.  The
      // staging tile aliases rv / ms, which are first written after this.
      constexpr int U = FPM_CGW_LOADS;
      uint32_t* stg = reinterpret_cast<uint32_t*>(base + TLay::off_rv);
      const double2* Ag = args.A + t * NN;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
#pragma unroll 1
        for (int q0 = l; q0 < 1024; q0 += 32 * U) {
          double2 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int q = q0 + 32 * u;
            v[u] = __ldcs(Ag + (q >> 4) * NC + 16 * c + (q & 15));
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int q = q0 + 32 * u, i = q >> 4, k = q & 15;
            const C h = A::rnd(v[u], fm);
            stg[i * 16 + ((((k >> 2) ^ (i >> 1)) & 3) << 2) + (k & 3)] = *reinterpret_cast<const uint32_t*>(&h);
          }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = l + 32 * j;
          uint32_t u[16];
#pragma unroll
          for (int w4 = 0; w4 < 4; ++w4) {
            const uint4 q = *reinterpret_cast<const uint4*>(stg + i * 16 + (((w4 ^ (i >> 1)) & 3) << 2));
            u[4 * w4] = q.x;
            u[4 * w4 + 1] = q.y;
            u[4 * w4 + 2] = q.z;
            u[4 * w4 + 3] = q.w;
          }
          tm_st16(ta + 64 * j + 16 * c, u);
        }
        __syncwarp();
      }
      tm_wait_st();
    } else {
      constexpr int U = FPM_CGW_LOADS;
      const double2* Ag = args.A + t * NN;
#pragma unroll 1
      for (int q0 = l; q0 < NN; q0 += 32 * U) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (q0 + 32 * u < NN) v[u] = __ldcs(Ag + q0 + 32 * u);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int q = q0 + 32 * u;
          if (q < NN) At[Lay::at(q / NC, q % NC)] = A::rnd(v[u], fm);
        }
      }
    }
    double2 x[RPL], r[RPL], p[RPL];
    C pm[RPL];
    double2 m[RPL][(LB > 0 && !MS) ? LB : 1];
#pragma unroll
    for (int j = 0; j < RPL; ++j) {
      const int i = l + 32 * j;
      x[j] = make_double2(0.0, 0.0);
      r[j] = args.b[t * NC + i];  // run_batch copies b (solvers.py:297-298)
      if constexpr (BJ && !MS) {
#pragma unroll
        for (int k = 0; k < LB; ++k) m[j][k] = args.minv[(t * NC + i) * LB + k];  // row i of its block
      }
      if constexpr (BJ && MS) {
#pragma unroll
        for (int k = 0; k < LB; ++k) ms[i * LB + ms_unit<LB>(i, k)] = args.minv[(t * NC + i) * LB + k];
      }
    }
    auto zrow = [&](int j) -> double2 {
      const int i = l + 32 * j;
      if constexpr (MS && BJ) return bj_z_s<LB>(ms, i, rv, i - i % LB);
      else if constexpr (!MS) return bj_z<(LB > 0 ? LB : 1)>(m[j], rv, i - i % (LB > 0 ? LB : 1));
      else return rv[i];  // unused (plain CG)
    };
    if (trc) {
      __syncwarp();
      if (l == 0) trc[1] = clock64();
    }
    // ---- init (solvers.py:297-328): p = M r | r; carry = r^H r | r^H p ----
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
      // as_written BJ: rho0 terms (tb0); otherwise the carry's terms (tb2, same storage)
      tb0[i] = A::mulc(ri, (BJ && (args.textbook || rho_fresh)) ? pm[j] : ri, fi);
    }
    __syncwarp();
    double2 carry = make_double2(0.0, 0.0);
    if (!rho_fresh) carry = wsum<K, NC>(tb2, fi);
    int brk = -1, dvg = -1;
    // ---- run_batch histories (solvers.py:306-319, 369-381); fpm_cg_ex only ----
    const CgHist& Hh = args.h;
    constexpr bool hist = HIST;  // compiled out of the plain fpm_cg kernel (registers)
    const bool hnorm = hist && (Hh.res || Hh.xn || Hh.conv);
    double h_bn = 0.0, h_res = 0.0, h_xn = 0.0;
    int h_conv = -1, last = args.iters;
    auto h_rows = [&](int i) {  // iterates / residual vectors of sweep i
#pragma unroll
      for (int j = 0; j < RPL; ++j) {
        const long o = ((long)i * Hh.T + t) * NC + l + 32 * j;
        if (Hh.xit) Hh.xit[o] = x[j];
        if (Hh.rit) Hh.rit[o] = r[j];
      }
    };
    auto h_norms = [&](int i, bool fresh) {  // res_hist[i], xn_hist[i] (solvers.py:373-374)
      if (!hnorm) return;
      if (fresh) {
        h_res = cgw_norm2<RPL>(r);
        h_xn = i ? cgw_norm2<RPL>(x) : 0.0;
        if (i == 0) h_bn = h_res;
      }
      // converged_at: first sweep whose (possibly frozen) residual is small
      if (i > 0 && h_conv < 0 && h_res <= Hh.rtol * fmax(h_bn, 1e-300)) h_conv = i;
      if (l == 0) {
        if (Hh.res) Hh.res[(long)i * Hh.T + t] = h_res;
        if (Hh.xn) Hh.xn[(long)i * Hh.T + t] = h_xn;
      }
    };
    auto h_ab = [&](int i, double2 al, double2 be) {  // alphas / betas[i - 1] (solvers.py:371)
      if (hist && l == 0) {
        if (Hh.al) Hh.al[(long)(i - 1) * Hh.T + t] = al;
        if (Hh.be) Hh.be[(long)(i - 1) * Hh.T + t] = be;
      }
    };
    if (hist) {
      h_norms(0, true);
      h_rows(0);
    }
    long long* ph = (trc && t == 0 && l == 0) ? args.trace + 4 * args.T : nullptr;  // phase clocks, realization 0
#define CGW_ST(k, dep)                                                             \
  do {                                                                             \
    if (ph) ph[(it - 1) * 10 + (k)] = clock64() + ((dep) == 1.2345e300 ? 1 : 0);   \
  } while (0)

#pragma unroll 1
    for (int it = 1; it <= args.iters; ++it) {
      // ---- w = A p (u_MV) ; rho0 (as_written BJ) ; phi = p^H w (u_IP) ----
      C wc[RPL];
      double2 rho0 = carry;
      if constexpr (TM) {
        mv_rows_tm<K>(ta, pmv, wc, fm);
      } else {
        mv_rows<K, NC, RPL, 32>(At, pmv, l, wc, fm);
      }
      if (rho_fresh) rho0 = wsum<K, NC>(tb0, fi);
      CGW_ST(0, A::wide(wc[RPL - 1]).x);
      CGW_ST(1, rho0.x);
#pragma unroll
      for (int j = 0; j < RPL; ++j) tb1[l + 32 * j] = A::mulc(pm[j], wc[j], fi);
      __syncwarp();
      const double2 phi = wsum<K, NC>(tb1, fi);
      CGW_ST(2, phi.x);
      // stall / breakdown freeze the realization (solvers.py:342-345)
      const bool stall = (rho0.x == 0.0) && (rho0.y == 0.0);
      if (!stall && phi.x <= 0.0) brk = it;
      if (stall || phi.x <= 0.0) {
        // alphas records alpha where the lane broke down, 0 on a stall
        if (hist) h_ab(it, stall ? make_double2(0.0, 0.0) : CGW_DIV(rho0, phi), make_double2(0.0, 0.0));
        last = it - 1;
        break;
      }
      const double2 al = CGW_DIV(rho0, phi);
      CGW_ST(3, al.x);
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
        if (hist) h_ab(it, al, make_double2(0.0, 0.0));
        last = it - 1;
        break;
      }
#pragma unroll
      for (int j = 0; j < RPL; ++j) {
        x[j] = xn[j];
        r[j] = rn[j];
      }
      CGW_ST(4, r[RPL - 1].x);
      // ---- z = M r ; rho1 = r^H z | r^H r ; beta = rho1 / rho0 ----
      double2 z[RPL];
      if constexpr (BJ) {
#pragma unroll
        for (int j = 0; j < RPL; ++j) rv[l + 32 * j] = r[j];
        __syncwarp();
#pragma unroll
        for (int j = 0; j < RPL; ++j) z[j] = zrow(j);
      }
      CGW_ST(5, BJ ? z[RPL - 1].x : r[0].x);
      C ri[RPL];
#pragma unroll
      for (int j = 0; j < RPL; ++j) {
        ri[j] = A::rnd(r[j], fi);
        tb2[l + 32 * j] = A::mulc(ri[j], BJ ? A::rnd(z[j], fi) : ri[j], fi);
      }
      __syncwarp();
      const double2 rho1 = wsum<K, NC>(tb2, fi);
      CGW_ST(6, rho1.x);
      const double2 be = CGW_DIV(rho1, rho0);
      CGW_ST(7, be.x);
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
      CGW_ST(8, p[RPL - 1].x);
      if (hist) {
        h_ab(it, al, be);
        h_norms(it, true);
        h_rows(it);
      }
    }
#undef CGW_ST
    if (hist) {
      // frozen before the last sweep: the remaining sweeps record the frozen
      // state (unchanged norms and vectors; zero alphas / betas after the
      // freezing sweep, whose alpha was recorded above)
#pragma unroll 1
      for (int i = last + 1; i <= args.iters; ++i) {
        if (i > last + 1) h_ab(i, make_double2(0.0, 0.0), make_double2(0.0, 0.0));
        h_norms(i, false);
        h_rows(i);
      }
      if (Hh.conv && l == 0) Hh.conv[t] = h_conv;
    }
    if (trc && l == 0) trc[2] = clock64();
#pragma unroll
    for (int j = 0; j < RPL; ++j) args.x[t * NC + l + 32 * j] = x[j];
    if (l == 0) {
      args.brk[t] = brk;
      args.div[t] = dvg;
    }
  }
  if constexpr (TM) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (wid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(ta) : "memory");
    }
  }
}

// One realization per warp.  (Two realizations per warp -- a half-warp each -- was measured slower at c5
// fp16: 35.9 M vs 51.7 M/s, half the warps per SM and twice the serial load
// phase per warp.)
template <int K, int NC, int LB, bool TM, bool HIST>
inline int launch_cgw_k2(const CgArgs& a, cudaStream_t st) {
  auto k = fpm_cgw_kernel<K, NC, LB, TM, HIST>;
  constexpr int smem = TM ? CgwTmLayout<K, NC, LB, true>::cta_bytes : CgwLayout<K, NC, LB>::bytes;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return FPM_ECUDA;
  if (TM) k<<<(unsigned)((a.T + 3) / 4), 128, smem, st>>>(a);
  else k<<<(unsigned)a.T, 32, smem, st>>>(a);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}

template <int K, int NC, int LB>
inline int launch_cgw_t(const CgArgs& a, cudaStream_t st) {
  constexpr bool tm_ok = NC == 64 && sizeof(typename Ar<K>::C) == 4 && (LB == 0 || LB == 4);
  if constexpr (tm_ok) {
    // opt-in (FPM_CGW_TMEM=1): measured slower than the shared-memory kernel
    // at c5 fp16 (50.4 M vs 55.5 M det/s): 15 resident warps instead of 12,
    // but the transposing load phase is twice as long and the sweeps slow
    // down under the extra contention
    const char* e = knob("FPM_CGW_TMEM");
    if (e && e[0] == '1' && !a.h.on) return launch_cgw_k2<K, NC, LB, true, false>(a, st);
  }
  return a.h.on ? launch_cgw_k2<K, NC, LB, false, true>(a, st) : launch_cgw_k2<K, NC, LB, false, false>(a, st);
}

template <int K, int NC>
inline int launch_cgw_n(const CgArgs& a, cudaStream_t st) {
  if (!a.bj) return launch_cgw_t<K, NC, 0>(a, st);
  switch (a.L) {
    case 1: return launch_cgw_t<K, NC, 1>(a, st);
    case 2: return launch_cgw_t<K, NC, 2>(a, st);
    case 4: return launch_cgw_t<K, NC, 4>(a, st);
    case 8: return launch_cgw_t<K, NC, 8>(a, st);
    default: return FPM_EUNSUPPORTED;
  }
}

template <int K>
inline int launch_cgw_k(const CgArgs& a, cudaStream_t st) {
  if (a.N == 64) return launch_cgw_n<K, 64>(a, st);
  if (a.N == 32) return launch_cgw_n<K, 32>(a, st);
  // N = 128 stays on the CTA-lockstep kernel: with 64 KB of fp16 A per warp
  // only two warps fit per SM and each lane chains four rows; measured at c4
  // (fp16, L = 8) 23.4 ms vs 20.8 ms per 8192 realizations
  return FPM_EUNSUPPORTED;
}

}  // namespace fpm
