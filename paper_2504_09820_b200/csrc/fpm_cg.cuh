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
// 94-95).  Latency design: the product terms of every dot product are formed
// in parallel by the row threads (each an independent rounded complex
// multiply) and only the left-to-right SUM runs as one dependent chain in one
// "owner" thread per realization; matvec rows are chains in parallel.  Six
// group barriers per sweep.  The matvec and inner-product formats are the same
// kind K (the host only builds native kernels for u_MV == u_IP; any other
// pair runs the generic emulation kind, with separate runtime parameters).
//
// I-cache: each step runs once per sweep on a few warps, so latency is
// dominated by instruction fetch unless the code is small and shared; the
// heavy helpers are __noinline__ (one hot copy) and thread roles are
// computed once.
#pragma once
#include "fpm_arith.cuh"
#include "fpm_ptx.cuh"

namespace fpm {

// run_batch history outputs (fpm_cg_history); null pointers are skipped
struct CgHist {
  double* res;    // (iters+1, T)
  double* xn;     // (iters+1, T)
  double2* al;    // (iters, T)
  double2* be;    // (iters, T)
  int* conv;      // (T,)
  double rtol;
  double2* xit;   // (iters+1, T, N)
  double2* rit;   // (iters+1, T, N)
  long T;         // leading stride of the histories
  long t0;        // first realization of this CTA
  int on;         // any output requested
};

template <int K>
struct CgSmem {
  typedef typename Ar<K>::C C;
  typedef typename Ar<K>::P P;
  int R, N, L, ldA;
  C* At;                  // R * N * ldA, row-major: entry (i,k) at i*ldA + k (ldA = lda_for), u_MV grid
  P* pmv;                 // R * N   p rounded to u_MV, prepared for the matvec
  C *tphi, *trho, *tr1;   // R * N   product terms of p^H w, r^H p, r^H z (or r^H r), u_IP
  C* rip;                 // R * N   r rounded to u_IP
  double2* minv;          // R * N*L block inverses: block kb at kb*L*L, column-major Lk x Lk, u_W grid
  double2 *b, *x, *r, *p, *z, *w, *xn, *rn;  // R * N each (u_W values, binary64 carriers)
  double2* sc;            // R * 8 : 0 alpha, 1 beta, 3 rho0, 4 carry
  int* fl;                // R * 4 : live, nonfinite, breakdown_at, diverged_at
  const CgHist* h = nullptr;  // run_batch histories (standalone CG kernel only)
  int dbg = 0;                // diagnostic bits (FPM_DEBUG): 16 skip matvec rows, 64 skip owner sums
};

// Owner of the sequential sums of slot g (which = 0: phi/rho1/carry,
// 1: as_written rho0).  One warp apart and past the matvec rows when all
// 2*Rv owners fit that way, else the last 2*Rv threads; distinct threads in
// both cases (a thread owns at most one chain; 2*Rv <= nthreads).
__device__ __forceinline__ int dot_owner(int g, int which, int rows, int nthreads, int Rv) {
  const int k = g * 2 + which;
  if (nthreads - 1 - 32 * (2 * Rv - 1) >= rows) return nthreads - 1 - 32 * k;
  return nthreads - 1 - k;
}

// 16-byte shared-memory vector loads of consecutive elements: V16<T>::n
// elements per LDS.128 (16-byte aligned source).
template <class T> struct V16;
template <> struct V16<__half2> {
  static constexpr int n = 4;
  static __device__ __forceinline__ void ld(const __half2* p, __half2* d) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    d[0] = u2h(u.x); d[1] = u2h(u.y); d[2] = u2h(u.z); d[3] = u2h(u.w);
  }
};
template <> struct V16<__nv_bfloat162> {
  static constexpr int n = 4;
  static __device__ __forceinline__ void ld(const __nv_bfloat162* p, __nv_bfloat162* d) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    d[0] = u2b(u.x); d[1] = u2b(u.y); d[2] = u2b(u.z); d[3] = u2b(u.w);
  }
};
template <> struct V16<Ar<FK_F16>::P> {
  static constexpr int n = 2;
  static __device__ __forceinline__ void ld(const Ar<FK_F16>::P* p, Ar<FK_F16>::P* d) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    d[0].v1 = u2h(u.x); d[0].v2 = u2h(u.y); d[1].v1 = u2h(u.z); d[1].v2 = u2h(u.w);
  }
};
template <> struct V16<Ar<FK_BF16>::P> {
  static constexpr int n = 2;
  static __device__ __forceinline__ void ld(const Ar<FK_BF16>::P* p, Ar<FK_BF16>::P* d) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    d[0].v1 = u2b(u.x); d[0].v2 = u2b(u.y); d[1].v1 = u2b(u.z); d[1].v2 = u2b(u.w);
  }
};
template <> struct V16<float2> {
  static constexpr int n = 2;
  static __device__ __forceinline__ void ld(const float2* p, float2* d) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    d[0] = make_float2(u.x, u.y); d[1] = make_float2(u.z, u.w);
  }
};
template <> struct V16<double2> {
  static constexpr int n = 1;
  static __device__ __forceinline__ void ld(const double2* p, double2* d) { d[0] = *p; }
};

template <int B, class T>
__device__ __forceinline__ void ld_blk(const T* p, T (&d)[B]) {
  constexpr int n = V16<T>::n;
  static_assert(B % n == 0, "block must be whole 16-byte vectors");
#pragma unroll
  for (int i = 0; i < B / n; ++i) V16<T>::ld(p + i * n, d + i * n);
}

__device__ __forceinline__ bool al16(const void* a, const void* b = nullptr) {
  return ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
}

// left-to-right sum t_0 + t_1 + ... (dot_fp's accumulation, linalg.py:94-95).
// Latency: the dependent adds are the only serial part, so the terms arrive
// in 64-byte blocks loaded one block AHEAD of the chain (a batch-then-add
// loop exposes the load latency every block: 2.3x slower, tools/ubench5.cu).
template <int K>
__device__ __noinline__ double2 chain_sum(const typename Ar<K>::C* t, int n, const FmtP& f) {
  typedef Ar<K> A;
  typedef typename A::C C;
  constexpr int B = sizeof(C) >= 16 ? 2 : 64 / sizeof(C);
  typename A::C s = t[0];
  if (n % B == 0 && al16(t)) {
    C v[B], nv[B];
    ld_blk<B>(t, v);
#pragma unroll 1
    for (int k = 0; k < n; k += B) {
      const bool more = k + B < n;
      if (more) ld_blk<B>(t + k + B, nv);
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (k + j > 0) s = A::add(s, v[j], f);
#pragma unroll
      for (int j = 0; j < B; ++j) v[j] = nv[j];
    }
    return A::wide(A::asmc(s));
  }
#pragma unroll 1
  for (int k = 1; k < n; ++k) s = A::add(s, t[k], f);
  return A::wide(A::asmc(s));
}

// w_i = sum_k A(i,k) p_k at u_MV (matvec_fp) over one row of A (row-major,
// pitch lda_for), returned assembled (`sr + 1j*si`) in-format.  The products
// of a block are independent; the block's operands are loaded one block
// ahead of the sequential sum.
template <int K>
__device__ __noinline__ typename Ar<K>::C mv_row(const typename Ar<K>::C* row, const typename Ar<K>::P* pv, int N,
                                               const FmtP& f) {
  typedef Ar<K> A;
  typedef typename A::C C;
  typedef typename A::P P;
  constexpr int B = sizeof(C) >= 16 ? 2 : (sizeof(C) >= 8 ? 4 : 8);
  if (N % B == 0 && al16(row, pv)) {
    C a[B], na[B];
    P p[B], np[B];
    ld_blk<B>(row, a);
    ld_blk<B>(pv, p);
    C s = A::mulp(a[0], p[0], f);
#pragma unroll 1
    for (int k = 0; k < N; k += B) {
      const bool more = k + B < N;
      if (more) {
        ld_blk<B>(row + k + B, na);
        ld_blk<B>(pv + k + B, np);
      }
      C t[B];
#pragma unroll
      for (int j = 0; j < B; ++j) t[j] = A::mulp(a[j], p[j], f);
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (k + j > 0) s = A::add(s, t[j], f);
#pragma unroll
      for (int j = 0; j < B; ++j) {
        a[j] = na[j];
        p[j] = np[j];
      }
    }
    return A::asmc(s);
  }
  C s = A::mulp(row[0], pv[0], f);
#pragma unroll 1
  for (int k = 1; k < N; ++k) s = A::add(s, A::mulp(row[k], pv[k], f), f);
  return A::asmc(s);
}

// binary64 complex sums in program order (volatile PTX: ptxas keeps the
// order, so the in-flight depth -- and the register footprint -- is the one
// written here; the fully unrolled C++ versions hoist every load and spill
// under the CG warps' register budget of the warp-specialised kernel).
// Each dependent add is separated from the previous one by independent
// loads / products, so the serial chain runs at the DADD latency.
namespace v64 {
__device__ __forceinline__ double2 ld(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ double add(double a, double b) {
  double r;
  asm volatile("add.rn.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
  return r;
}
__device__ __forceinline__ double sub(double a, double b) {
  double r;
  asm volatile("sub.rn.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
  return r;
}
__device__ __forceinline__ double mul(double a, double b) {
  double r;
  asm volatile("mul.rn.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
  return r;
}
// _cmul at binary64 (Ar<FK_F64>::mul): (fl(fl(ar pr) - fl(ai pi)), fl(fl(ar pi) + fl(ai pr)))
__device__ __forceinline__ double2 cmul(double2 a, double2 p) {
  const double rr = mul(a.x, p.x), ii = mul(a.y, p.y), ri = mul(a.x, p.y), ir = mul(a.y, p.x);
  return make_double2(sub(rr, ii), add(ri, ir));
}
}  // namespace v64

// left-to-right sum of NC binary64 complex terms (chain_sum at u_IP = fp64);
// terms requested kD ahead of their add
#ifndef FPM_F64_DOT_RING  // binary64 terms in flight in a dot chain
#define FPM_F64_DOT_RING 6
#endif
#ifndef FPM_F64_MV_RING  // (A, p) pairs in flight in a binary64 matvec row
#define FPM_F64_MV_RING 5
#endif
template <int NC>
__device__ __noinline__ double2 chain_sum_f64(const double2* t) {
  constexpr int kD = FPM_F64_DOT_RING;
  const uint32_t a0 = smem_u32(t);
  double2 v[kD];
#pragma unroll
  for (int j = 0; j < kD && j < NC; ++j) v[j] = v64::ld(a0 + 16 * j);
  double2 s = v[0];
#pragma unroll
  for (int k = 1; k < NC; ++k) {
    if (k - 1 + kD < NC) v[(k - 1) % kD] = v64::ld(a0 + 16 * (k - 1 + kD));
    s = make_double2(v64::add(s.x, v[k % kD].x), v64::add(s.y, v[k % kD].y));
  }
  return assemble(s.x, s.y);
}

// one matvec row at binary64 (mv_row at u_MV = fp64): the (A, p) operands of
// term q + kD are requested when term q's product is formed, and products run
// kP terms ahead of their add
template <int NC>
__device__ __noinline__ double2 mv_row_f64(const double2* row, const double2* pv) {
  constexpr int kD = FPM_F64_MV_RING, kP = 2;
  static_assert(NC >= kD, "row shorter than the operand ring");
  const uint32_t ra = smem_u32(row), pa = smem_u32(pv);
  double2 a[kD], p[kD], t[kP];
#pragma unroll
  for (int j = 0; j < kD; ++j) {
    a[j] = v64::ld(ra + 16 * j);
    p[j] = v64::ld(pa + 16 * j);
  }
#pragma unroll
  for (int j = 0; j < kP; ++j) {
    t[j] = v64::cmul(a[j], p[j]);
    if (j + kD < NC) {
      a[j] = v64::ld(ra + 16 * (j + kD));
      p[j] = v64::ld(pa + 16 * (j + kD));
    }
  }
  double2 s = t[0];
#pragma unroll
  for (int k = 1; k < NC; ++k) {
    const int q = k - 1 + kP;  // term whose product is formed in this step
    if (q < NC) {
      t[q % kP] = v64::cmul(a[q % kD], p[q % kD]);
      if (q + kD < NC) {
        a[q % kD] = v64::ld(ra + 16 * (q + kD));
        p[q % kD] = v64::ld(pa + 16 * (q + kD));
      }
    }
    s = make_double2(v64::add(s.x, t[k % kP].x), v64::add(s.y, t[k % kP].y));
  }
  return assemble(s.x, s.y);
}

// one matvec row at binary64 with the row in TENSOR MEMORY (the fused
// kernel's fp64 A, one row per TMEM lane, entry k at columns 4k..4k+3 from
// ta): 4-entry chunks by tcgen05.ld 32x32b.x16, the next chunk in flight
// while this chunk's products and adds run; p from shared memory in a ring
// of kD terms (same order of operations as mv_row_f64).  Warp-collective:
// every lane of the warp calls it.
template <int NC>
__device__ __noinline__ double2 mv_row_tm64(uint32_t ta, const double2* pv) {
  constexpr int kD = 5;
  static_assert(NC % 4 == 0 && NC >= 8, "TMEM row: whole 4-entry chunks");
  const uint32_t pa = smem_u32(pv);
  uint32_t cur[16], nxt[16];
  tmx_ld16(cur, ta);
  double2 p[kD];
#pragma unroll
  for (int j = 0; j < kD; ++j) p[j] = v64::ld(pa + 16 * j);
  tmx_wait_ld();
  tmx_launder(cur);
  double2 s = make_double2(0.0, 0.0);
#pragma unroll
  for (int c = 0; c < NC / 4; ++c) {
    if (c + 1 < NC / 4) tmx_ld16(nxt, ta + 16 * (c + 1));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = 4 * c + j;
      const double2 a = make_double2(__hiloint2double(cur[4 * j + 1], cur[4 * j]),
                                     __hiloint2double(cur[4 * j + 3], cur[4 * j + 2]));
      const double2 t = v64::cmul(a, p[k % kD]);
      if (k + kD < NC) p[k % kD] = v64::ld(pa + 16 * (k + kD));
      s = k == 0 ? t : make_double2(v64::add(s.x, t.x), v64::add(s.y, t.y));
    }
    if (c + 1 < NC / 4) {
      tmx_wait_ld();
      tmx_launder(nxt);
#pragma unroll
      for (int j = 0; j < 16; ++j) cur[j] = nxt[j];
    }
  }
  return assemble(s.x, s.y);
}

// where a CG group finds the fused kernel's fp64 A in tensor memory: base =
// TMEM address of the hand-off slot (lane field 0), qw0 = CTA warp index of
// the group's first warp, nw = its warps.  Row q = g*N + i lives in TMEM lane
// q % 128 at columns base + (q / 128) * 4N.
struct TmRows {
  uint32_t base;
  int qw0, nw;
};

// Compile-time N (NC > 0): the whole sum is one basic block, so the
// scheduler overlaps every load and product with the dependent add chain
// (the loop versions above issue in order: a block's adds stall the next
// block's loads / products).
template <int K, int NC>
__device__ __noinline__ double2 chain_sum_n(const typename Ar<K>::C* t, const FmtP& f) {
  typedef Ar<K> A;
  typedef typename A::C C;
  constexpr int n16 = V16<C>::n;
  if constexpr (K == FK_F64 && NC >= 8) {
    return chain_sum_f64<NC>(t);
  } else if constexpr (NC % n16 == 0 && NC * sizeof(C) <= 256) {
    C v[NC];
#pragma unroll
    for (int i = 0; i < NC / n16; ++i) V16<C>::ld(t + i * n16, v + i * n16);
    C s = v[0];
#pragma unroll
    for (int j = 1; j < NC; ++j) s = A::add(s, v[j], f);
    return A::wide(A::asmc(s));
  } else if constexpr (NC % 8 == 0 && NC <= 128) {
    // wide terms: 8-term blocks, each loaded two blocks ahead of its adds
    C v0[8], v1[8], v2[8];
    ld_blk<8>(t, v0);
    if (NC > 8) ld_blk<8>(t + 8, v1);
    C s = v0[0];
#pragma unroll
    for (int k = 0; k < NC; k += 8) {
      if (k + 16 < NC) ld_blk<8>(t + k + 16, v2);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (k + j > 0) s = A::add(s, v0[j], f);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v0[j] = v1[j];
        v1[j] = v2[j];
      }
    }
    return A::wide(A::asmc(s));
  } else {
    return chain_sum<K>(t, NC, f);
  }
}

template <int K, int NC>
__device__ __noinline__ typename Ar<K>::C mv_row_n(const typename Ar<K>::C* row, const typename Ar<K>::P* pv,
                                                 const FmtP& f) {
  typedef Ar<K> A;
  typedef typename A::C C;
  typedef typename A::P P;
  constexpr int B = sizeof(C) >= 16 ? 2 : (sizeof(C) >= 8 ? 4 : 8);
  if constexpr (K == FK_F64 && NC >= 8) {
    if (__isShared(row)) return mv_row_f64<NC>(row, pv);  // (A stays in HBM when it does not fit: fpm_cg)
    return mv_row<K>(row, pv, NC, f);
  } else if constexpr (NC % B == 0 && NC * sizeof(C) <= 256) {
    C s;
#pragma unroll
    for (int k = 0; k < NC; k += B) {
      C a[B];
      P p[B];
      ld_blk<B>(row + k, a);
      ld_blk<B>(pv + k, p);
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const C t = A::mulp(a[j], p[j], f);
        s = (k + j == 0) ? t : A::add(s, t, f);
      }
    }
    return A::asmc(s);
  } else if constexpr (NC % 4 == 0 && NC <= 128) {
    // wide terms: 4-term blocks loaded two blocks ahead; the products of a
    // block are formed before its adds so they overlap the add chain
    C a0[4], a1[4], a2[4];
    P p0[4], p1[4], p2[4];
    ld_blk<4>(row, a0);
    ld_blk<4>(pv, p0);
    if (NC > 4) {
      ld_blk<4>(row + 4, a1);
      ld_blk<4>(pv + 4, p1);
    }
    C s;
#pragma unroll
    for (int k = 0; k < NC; k += 4) {
      if (k + 8 < NC) {
        ld_blk<4>(row + k + 8, a2);
        ld_blk<4>(pv + k + 8, p2);
      }
      C t[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = A::mulp(a0[j], p0[j], f);
#pragma unroll
      for (int j = 0; j < 4; ++j) s = (k + j == 0) ? t[0] : A::add(s, t[j], f);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        a0[j] = a1[j];
        a1[j] = a2[j];
        p0[j] = p1[j];
        p1[j] = p2[j];
      }
    }
    return A::asmc(s);
  } else {
    return mv_row<K>(row, pv, NC, f);
  }
}

// row jl of block-diagonal apply from the block's r values already in
// registers (rl[0..LB-1], on the u_W grid): same operations as bj_row
template <int WK, int LB>
__device__ __forceinline__ double2 bj_row_reg(const double2* Mblk, const double2 (&rl)[LB], int jl, const FmtP& w) {
  typedef Ar<WK> A;
  const double2* M = Mblk + jl;  // column-major block
  double2 s = A::mul(M[0], rl[0], w);
#pragma unroll
  for (int l = 1; l < LB; ++l) s = A::add(s, A::mul(M[l * LB], rl[l], w), w);
  return assemble(s.x, s.y);
}

// one row of the block-diagonal apply M r (solvers.py:222-225) at u_W
template <int WK, int LB>
__device__ __noinline__ double2 bj_row(const double2* minv, const double2* r, int j, int L_rt, int N, const FmtP& w) {
  typedef Ar<WK> A;
  const int L = LB > 0 ? LB : L_rt;
  const int kb = j / L, jl = j - kb * L;
  const int s0 = kb * L;
  const int Lk = LB > 0 ? LB : min(L, N - s0);
  const double2* M = minv + kb * L * L + jl;  // column-major block
  double2 s = A::mul(M[0], A::rnd(r[s0], w), w);
#pragma unroll
  for (int l = 1; l < Lk; ++l) s = A::add(s, A::mul(M[l * Lk], A::rnd(r[s0 + l], w), w), w);
  return assemble(s.x, s.y);
}

// norm2 (linalg.py:122-134): scale = max|v_k| (NaN-propagating, 1 if not a
// finite positive number), scale * sqrt(sum (|v_k|/scale)^2), inf if any
// |v_k| is inf.  |v| is hypot; the sum runs left to right (NumPy's pairwise
// sum and libm hypot may differ in the last bits).
static __device__ __noinline__ double norm2_c(const double2* v, int n) {
  double scale = 0.0;
  bool nan = false, inf = false;
#pragma unroll 1
  for (int k = 0; k < n; ++k) {
    const double m = hypot(v[k].x, v[k].y);
    nan |= isnan(m);
    inf |= isinf(m);
    scale = m > scale ? m : scale;
  }
  if (nan || !isfinite(scale) || !(scale > 0.0)) scale = 1.0;
  double s = 0.0;
#pragma unroll 1
  for (int k = 0; k < n; ++k) {
    const double q = __ddiv_rn(hypot(v[k].x, v[k].y), scale);
    s = __dadd_rn(s, __dmul_rn(q, q));
  }
  const double out = __dmul_rn(scale, __dsqrt_rn(s));
  return inf ? __longlong_as_double(0x7ff0000000000000LL) : out;
}

// phase timestamps (diagnostic): thread 0 of CTA 0 writes clock64 values
// (a volatile shared-memory read first forces the deferred-blocking barrier
// to actually release before the clock is sampled)
#define FPM_STAMP(tr, k)                                                      \
  do {                                                                        \
    if ((tr) && tid == 0) {                                                   \
      __shared__ int _fpm_dummy;                                              \
      int _v = *(volatile int*)&_fpm_dummy;                                   \
      (tr)[(k)] = (long long)clock64() + (_v == 0x7fffffff ? 1 : 0);          \
    }                                                                         \
  } while (0)


// Group barriers: the whole CTA, or a named hardware barrier over `count`
// threads (warp-specialised kernel; ids 1..15, count a multiple of 32).
struct CtaBar {
  __device__ __forceinline__ void sync() { __syncthreads(); }
  __device__ __forceinline__ int any(int v) { return __syncthreads_or(v); }
};
struct NamedBar {
  int id, count;
  __device__ __forceinline__ void sync() { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory"); }
  __device__ __forceinline__ int any(int v) {
    int out;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.s32 p, %1, 0;\n\t"
        "bar.red.or.pred q, %2, %3, p;\n\t"
        "selp.s32 %0, 1, 0, q;\n}"
        : "=r"(out)
        : "r"(v), "r"(id), "r"(count)
        : "memory");
    return out;
  }
};

// Group-level CG: the nthreads threads of one synchronisation group (the
// whole CTA, or a named-barrier warp group in the warp-specialised kernel)
// advance all Rv resident realizations in lockstep.  Rows are spread over
// the group; each realization's sequential sums run in an "owner" thread,
// placed past the row threads when the group has spare lanes.  bar.sync()
// is the group barrier, bar.any(v) a barrier that ORs v over the group.
//
// Five group barriers per sweep: A (matvec, phi terms) | B (phi, alpha) |
// C (x, r updates + z = M r + rho1 terms, each thread recomputing the r
// updates of its own diagonal block so z needs no extra barrier) | E (rho1,
// beta, divergence) | F (commit x, r; p update).  NC > 0: N known at
// compile time (fully unrolled sums).  Ragged blocks (LB == 0 with BJ)
// take one more barrier between the r updates and z.
template <int WK, int K, int LB, int NC = 0, bool TM = false, class Bar>
__device__ void cg_group(CgSmem<K>& S, int Rv, int iters, bool bj, bool textbook, const Prec& pr, int nthreads,
                         int tid, Bar& bar, long long* tr = nullptr, TmRows tmr = TmRows{0, 0, 0}) {
  static_assert(!TM || (K == FK_F64 && NC > 0), "A in tensor memory: binary64 matvec, compile-time N");
  typedef Ar<K> A;
  typedef typename A::C C;
  const int N = NC > 0 ? NC : S.N;
  const int RN = Rv * N;
  const FmtP& fw = pr.work;
  const FmtP& fm = pr.mv;
  const FmtP& fi = pr.ip;
  const bool rho_fresh = bj && !textbook;  // as_written: rho0 = r^H p every sweep
  const bool merged = !bj || LB > 0;       // z from registers (no barrier between r and z)
  // roles, once
  const int nrow = RN > tid ? (RN - tid + nthreads - 1) / nthreads : 0;
  int og = -1, ow = 0;
#pragma unroll 1
  for (int g = 0; g < Rv; ++g) {
    if (dot_owner(g, 0, RN, nthreads, Rv) == tid) og = g, ow = 0;
    if (dot_owner(g, 1, RN, nthreads, Rv) == tid) og = g, ow = 1;
  }
  // u_IP value of a binary64 (work) value / of a value already on the u_MV grid
  // (native kinds: u_IP == u_MV, so the matvec's rounding of p is reused)
  auto ipr = [&](double2 v) -> C { return A::rnd(v, fi); };
  auto mv_to_ip = [&](C v) -> C { return K == FK_GEN ? A::rnd(A::wide(v), fi) : v; };
  auto csum = [&](const C* t) -> double2 {
    if constexpr (NC > 0) return chain_sum_n<K, NC>(t, fi);
    else return chain_sum<K>(t, N, fi);
  };

  // ---- init (solvers.py:297-328) ----
#pragma unroll 1
  for (int k = 0; k < nrow; ++k) {
    const int q = tid + k * nthreads;
    S.x[q] = make_double2(0.0, 0.0);
    S.r[q] = S.b[q];
  }
#pragma unroll 1
  for (int g = tid; g < Rv; g += nthreads) {
    S.fl[g * 4 + 1] = 0;
    S.fl[g * 4 + 2] = -1;
    S.fl[g * 4 + 3] = -1;
    // fl[g*4+0] (live) is set by the caller (0 if setup failed)
  }
  bar.sync();
#pragma unroll 1
  for (int k = 0; k < nrow; ++k) {
    const int q = tid + k * nthreads;
    const int g = q / N, i = q - g * N;
    const double2 rv = S.r[q];
    const double2 pv = bj ? bj_row<WK, LB>(S.minv + g * N * S.L, S.r + g * N, i, S.L, N, fw) : rv;
    S.p[q] = pv;
    const C pm = A::rnd(pv, fm);
    S.pmv[q] = A::prep(pm);
    const C ri = ipr(rv);
    S.rip[q] = ri;
    const C pi = K == FK_GEN ? ipr(pv) : pm;
    S.tr1[q] = A::mulc(ri, (bj && textbook) ? pi : ri, fi);  // carry terms
    if (rho_fresh) S.trho[q] = A::mulc(ri, pi, fi);
  }
  bar.sync();
  if (!rho_fresh && og >= 0 && ow == 0) S.sc[og * 8 + 4] = csum(S.tr1 + og * N);
  // ---- run_batch histories (solvers.py:306-319; standalone kernel only) ----
  const CgHist* H = S.h;
  double h_bn = 0.0, h_res = 0.0, h_xn = 0.0;
  int h_conv = -1;
  auto h_at = [&](int i, int g) -> long { return (long)i * H->T + H->t0 + g; };
  auto h_rows = [&](int i) {  // iterates / residual vectors of sweep i, every row
#pragma unroll 1
    for (int k = 0; k < nrow; ++k) {
      const int q = tid + k * nthreads;
      const int g = q / N, row = q - g * N;
      if (H->xit) H->xit[h_at(i, g) * N + row] = S.x[q];
      if (H->rit) H->rit[h_at(i, g) * N + row] = S.r[q];
    }
  };
  auto h_norms = [&](int i) {  // res_hist[i], xn_hist[i] (solvers.py:373-374)
    h_res = norm2_c(S.r + og * N, N);
    h_xn = i ? norm2_c(S.x + og * N, N) : 0.0;
    if (i == 0) h_bn = h_res;
    if (H->res) H->res[h_at(i, og)] = h_res;
    if (H->xn) H->xn[h_at(i, og)] = h_xn;
    if (i > 0 && h_conv < 0 && h_res <= H->rtol * fmax(h_bn, 1e-300)) h_conv = i;
  };
  if (H) {
    if (og >= 0 && ow == 1) h_norms(0);
    h_rows(0);
  }
  bar.sync();
  FPM_STAMP(tr, 0);
  int it_last = iters;

#pragma unroll 1
  for (int it = 1; it <= iters; ++it) {
    // ---- A: w = A p (u_MV) + phi terms;  rho0 = sum r^H p (BJ as_written) ----
    if constexpr (TM) {
      // rows by TMEM lane ownership: this warp reads lane quarter Q; the
      // group's warps of one quarter share its 128-row blocks
      const int wi = tid >> 5, lane = tid & 31;
      const int Q = (tmr.qw0 + wi) & 3;
      const int nQ = (tmr.nw - 1 - (wi & 3)) / 4 + 1;
      const int nRB = (S.R * N + 127) / 128;
#pragma unroll 1
      for (int RB = wi >> 2; RB < nRB; RB += nQ) {
        const int q = RB * 128 + Q * 32 + lane;
        const int g = q / N;
        const C wc = mv_row_tm64<NC>(tmr.base + ((uint32_t)(Q * 32) << 16) + (uint32_t)(RB * 4 * N), S.pmv + g * N);
        if (g < Rv && S.fl[g * 4]) {
          S.w[q] = A::wide(wc);
          const C pi = A::rnd(S.p[q], fm);
          S.tphi[q] = A::mulc(pi, mv_to_ip(wc), fi);
        }
      }
      tmx_fence_before();  // this sweep's TMEM reads precede the slot's release
    } else
#pragma unroll 1
    for (int k = 0; k < nrow; ++k) {
      const int q = tid + k * nthreads;
      const int g = q / N, i = q - g * N;
      if (!S.fl[g * 4]) continue;
      if (tr && tid == 0 && it == 2) tr[75] = clock64();
      C wc;
      if (S.dbg & 16) wc = A::rnd(make_double2(1.0, 0.0), fm);
      else if constexpr (NC > 0) wc = mv_row_n<K, NC>(S.At + (g * N + i) * S.ldA, S.pmv + g * N, fm);
      else wc = mv_row<K>(S.At + (g * N + i) * S.ldA, S.pmv + g * N, N, fm);
      if (tr && tid == 0 && it == 2) tr[76] = clock64() + (h2u(*reinterpret_cast<__half2*>(&wc)) == 12345u);
      S.w[q] = A::wide(wc);
      const C pi = K == FK_GEN ? ipr(S.p[q]) : A::rnd(S.p[q], fm);
      S.tphi[q] = A::mulc(pi, mv_to_ip(wc), fi);
      if (tr && tid == 0 && it == 2) tr[77] = clock64() + (S.w[q].x == 1.234e300);
    }
    if (rho_fresh && og >= 0 && ow == 1 && S.fl[og * 4]) S.sc[og * 8 + 3] = csum(S.trho + og * N);
    diag_jitter(S.dbg, 8, it);
    bar.sync();
    FPM_STAMP(tr, 1 + (it - 1) * 6 + 0);
    // ---- B: phi, flags, alpha ----
    if (H && H->al && og >= 0 && ow == 0 && !S.fl[og * 4]) H->al[h_at(it - 1, og)] = make_double2(0.0, 0.0);
    if (og >= 0 && ow == 0 && S.fl[og * 4]) {
      const int g = og;
      const bool st = tr && g == 0 && it == 2;
      if (st) tr[78] = clock64();
      const double2 phi = (S.dbg & 64) ? make_double2(1.0, 0.0) : csum(S.tphi + g * N);
      if (st) tr[79] = clock64() + (phi.x == 1.234e300);
      const double2 rho0 = rho_fresh ? S.sc[g * 8 + 3] : S.sc[g * 8 + 4];
      S.sc[g * 8 + 3] = rho0;
      const bool stall = (rho0.x == 0.0) && (rho0.y == 0.0);
      if (!stall && phi.x <= 0.0) S.fl[g * 4 + 2] = it;  // breakdown
      if (stall || phi.x <= 0.0) S.fl[g * 4] = 0;
      const double2 al = wdiv<WK>(rho0, phi, fw);
      if (st) tr[80] = clock64() + (al.x == 1.234e300);
      S.sc[g * 8 + 0] = al;
      // alphas[i-1] = alpha where active | newly_bad | broke (solvers.py:371)
      if (H && H->al) H->al[h_at(it - 1, g)] = stall ? make_double2(0.0, 0.0) : al;
    }
    diag_jitter(S.dbg, 9, it);
    bar.sync();
    FPM_STAMP(tr, 1 + (it - 1) * 6 + 1);
    // ---- C: x, r updates (u_W) + finiteness; z = M r and rho1 terms ----
#pragma unroll 1
    for (int k = 0; k < nrow; ++k) {
      const int q = tid + k * nthreads;
      const int g = q / N, i = q - g * N;
      if (!S.fl[g * 4]) continue;
      const bool st = tr && tid == 0 && it == 2;
      if (st) tr[70] = clock64();
      const double2 al = S.sc[g * 8 + 0];
      const double2 nal = make_double2(-al.x, -al.y);
      const double2 xn = axpy1<WK>(al, S.p[q], S.x[q], fw);
      const double2 rn = axpy1<WK>(nal, S.w[q], S.r[q], fw);
      S.xn[q] = xn;
      S.rn[q] = rn;
      if (st) tr[71] = clock64() + (rn.x == 1.234e300);
      if (!(finite2(xn) && finite2(rn))) S.fl[g * 4 + 1] = 1;
      if (merged) {
        const C ri = ipr(rn);
        if (bj) {
          if constexpr (LB > 0) {
            // this thread recomputes its block's r updates (same bits as the
            // owning threads) so z = M r needs no barrier
            const int kb = i / LB, jl = i - kb * LB, s0 = g * N + kb * LB;
            double2 rl[LB];
#pragma unroll
            for (int l = 0; l < LB; ++l)  // branch-free: row jl recomputes rn bit-identically
              rl[l] = Ar<WK>::rnd(axpy1<WK>(nal, S.w[s0 + l], S.r[s0 + l], fw), fw);
            if (st) tr[72] = clock64() + (rl[LB - 1].x == 1.234e300);
            const double2 zv = bj_row_reg<WK, LB>(S.minv + g * N * S.L + kb * LB * LB, rl, jl, fw);
            if (st) tr[73] = clock64() + (zv.x == 1.234e300);
            S.z[q] = zv;
            S.tr1[q] = A::mulc(ri, ipr(zv), fi);
            if (st) tr[74] = clock64() + (h2u(*reinterpret_cast<__half2*>(&S.tr1[q])) == 12345u);
          }
        } else {
          S.tr1[q] = A::mulc(ri, ri, fi);
        }
      }
    }
    if (!merged) {  // ragged block-Jacobi: z after a barrier
      bar.sync();
#pragma unroll 1
      for (int k = 0; k < nrow; ++k) {
        const int q = tid + k * nthreads;
        const int g = q / N, i = q - g * N;
        if (!S.fl[g * 4] || S.fl[g * 4 + 1]) continue;
        const double2 zv = bj_row<WK, LB>(S.minv + g * N * S.L, S.rn + g * N, i, S.L, N, fw);
        S.z[q] = zv;
        S.tr1[q] = A::mulc(ipr(S.rn[q]), ipr(zv), fi);
      }
    }
    diag_jitter(S.dbg, 10, it);
    bar.sync();
    FPM_STAMP(tr, 1 + (it - 1) * 6 + 2);
    // ---- E: rho1, beta, divergence flag ----
    if (H && H->be && og >= 0 && ow == 0 && !S.fl[og * 4]) H->be[h_at(it - 1, og)] = make_double2(0.0, 0.0);
    if (og >= 0 && ow == 0 && S.fl[og * 4]) {
      const int g = og;
      if (S.fl[g * 4 + 1]) {  // non-finite update: diverged, frozen at the last finite iterate
        S.fl[g * 4 + 3] = it;
        S.fl[g * 4] = 0;
        if (H && H->be) H->be[h_at(it - 1, g)] = make_double2(0.0, 0.0);
      } else {
        const double2 rho1 = (S.dbg & 64) ? make_double2(1.0, 0.0) : csum(S.tr1 + g * N);
        const double2 be = wdiv<WK>(rho1, S.sc[g * 8 + 3], fw);
        S.sc[g * 8 + 1] = be;
        S.sc[g * 8 + 4] = rho1;
        if (H && H->be) H->be[h_at(it - 1, g)] = be;  // betas: where(active, beta, 0)
      }
    }
    diag_jitter(S.dbg, 11, it);
    bar.sync();
    FPM_STAMP(tr, 1 + (it - 1) * 6 + 3);
    // ---- F: commit x, r; p = (z|r) + beta p ; pmv = rnd(p) ; next rho0 terms ----
    int any = 0;
#pragma unroll 1
    for (int k = 0; k < nrow; ++k) {
      const int q = tid + k * nthreads;
      const int g = q / N;
      if (!S.fl[g * 4]) continue;
      any = 1;
      const double2 rn = S.rn[q];
      S.x[q] = S.xn[q];
      S.r[q] = rn;
      const C ri = ipr(rn);
      S.rip[q] = ri;
      const double2 pn = axpy1<WK>(S.sc[g * 8 + 1], S.p[q], bj ? S.z[q] : rn, fw);
      S.p[q] = pn;
      const C pm = A::rnd(pn, fm);
      S.pmv[q] = A::prep(pm);
      if (rho_fresh) S.trho[q] = A::mulc(ri, K == FK_GEN ? ipr(pn) : pm, fi);
    }
    const int more = bar.any(any);
    FPM_STAMP(tr, 1 + (it - 1) * 6 + 5);
    // x, r are stable until the next F: record this sweep without a barrier
    if (H) {
      if (og >= 0 && ow == 1) h_norms(it);
      h_rows(it);
    }
    if (!more) {
      it_last = it;
      break;
    }
  }
  bar.sync();
  if (H) {
    // every lane frozen early: the remaining sweeps record frozen values
    // (alphas / betas 0, unchanged norms and vectors)
#pragma unroll 1
    for (int i = it_last + 1; i <= iters; ++i) {
      if (og >= 0 && ow == 0) {
        if (H->al) H->al[h_at(i - 1, og)] = make_double2(0.0, 0.0);
        if (H->be) H->be[h_at(i - 1, og)] = make_double2(0.0, 0.0);
      }
      if (og >= 0 && ow == 1) {
        if (H->res) H->res[h_at(i, og)] = h_res;
        if (H->xn) H->xn[h_at(i, og)] = h_xn;
      }
      h_rows(i);
    }
    if (og >= 0 && ow == 1 && H->conv) H->conv[H->t0 + og] = h_conv;
    bar.sync();
  }
}

}  // namespace fpm
