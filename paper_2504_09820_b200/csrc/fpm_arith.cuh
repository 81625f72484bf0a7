// Finite-precision complex arithmetic that reproduces the reference's
// software emulation bit for bit on sm_100a.
//
// Reference semantics (all paths relative to /root/reference/pkg/src/fpmimo):
//   * FloatFormat.round            formats.py:110-139  RNE onto a (sig, exp) grid,
//                                   subnormals kept, overflow -> inf
//   * _cmul / _cadd                formats.py:218-227  schoolbook complex ops, every
//                                   real op rounded
//   * `sr + 1j*si` assembly         linalg.py:69, 97, 119; formats.py:146
//   * complex128 division (Smith)   solvers.py:256-259 via NumPy
//
// Native formats (fp64 / fp32 / fp16 / bf16) use the hardware's correctly
// rounded non-fused ops (__dmul_rn, __fadd_rn, __hmul2_rn, ...): for two
// operands on a p-bit grid the binary64-then-round emulation equals one
// correctly rounded p-bit op (exact products; double rounding innocuous for
// sums since 53 >= 2p + 2).  Any other (sig, exp) runs the generic path:
// binary64 op followed by an integer-exact RNE rounding (FK_GEN).
// Nothing here may contract into FMA: every op is an explicit _rn intrinsic
// and the library is built with -fmad=false.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace fpm {

// Diagnostics (phase clock traces, FPM_DEBUG skip bits for attribution) exist
// only in diagnostic builds (-DFPM_DIAG, tools/); in the product library the
// trace pointer and the skip bits are compile-time null / zero.
#ifdef FPM_DIAG
constexpr bool kDiag = true;
#else
constexpr bool kDiag = false;
#endif
__host__ __device__ __forceinline__ long long* diag_trace(long long* p) { return kDiag ? p : nullptr; }
__host__ __device__ __forceinline__ int diag_bits(int d) { return kDiag ? d : 0; }

// Row pitch (elements) of the u_MV matrix in shared memory: the smallest
// ldA >= N whose row is an odd number of 16-byte units, so rows start
// 16-byte aligned (LDS.128) and 8 consecutive rows fall on 8 distinct
// bank quads (conflict-free quarter-warp phases).
__host__ __device__ constexpr int lda_for(int N, int csize) {
  return (((N * csize + 15) / 16) | 1) * 16 / csize;
}

enum FmtKind : int { FK_F64 = 0, FK_F32 = 1, FK_F16 = 2, FK_BF16 = 3, FK_GEN = 4 };

// Runtime description of a format (generic path); mirrors FloatFormat.
struct FmtP {
  int sig;      // significand bits incl. hidden bit
  int qmin;     // smallest quantum exponent (formats.py:91)
  int sub;      // subnormals enabled
  int native;   // == binary64 (rounding is the identity)
  double xmax;  // largest finite value
  double xmin;  // smallest normal value
};

struct Prec {
  FmtP work, mv, ip;
};

// ------------------------------------------------------------------------
// Generic RNE rounding on the binary64 encoding (formats.py:110-139)
// ------------------------------------------------------------------------

__device__ __forceinline__ double pow2_scale(double v, int q) {
  // v * 2**q exactly (v an integer < 2**54) -- two exact power-of-two steps
  int q1 = q < -1022 ? -1022 : (q > 1023 ? 1023 : q);
  int q2 = q - q1;
  q2 = q2 < -1022 ? -1022 : (q2 > 1023 ? 1023 : q2);
  double s1 = __longlong_as_double((long long)(q1 + 1023) << 52);
  double s2 = __longlong_as_double((long long)(q2 + 1023) << 52);
  return __dmul_rn(__dmul_rn(v, s1), s2);
}

static __device__ __noinline__ double gen_round(double x, const FmtP& f) {
  if (f.native) return x;
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  unsigned long long a = b & 0x7FFFFFFFFFFFFFFFULL;
  if (a == 0ULL || a >= 0x7FF0000000000000ULL) return x;  // +-0, inf, nan
  int eb = (int)(a >> 52);
  unsigned long long mant = (a & 0x000FFFFFFFFFFFFFULL) | (eb ? 0x0010000000000000ULL : 0ULL);
  int lsb = eb ? eb - 1075 : -1074;
  int e = lsb + (64 - __clzll((long long)mant));        // frexp exponent
  int q = max(e - f.sig, f.qmin);
  int d = q - lsb;
  double y;
  if (d <= 0) {
    y = __longlong_as_double((long long)a);
  } else {
    unsigned long long r = 0ULL;
    if (d < 54) {
      r = mant >> d;
      unsigned long long rem = mant & ((1ULL << d) - 1ULL);
      unsigned long long half = 1ULL << (d - 1);
      if (rem > half || (rem == half && (r & 1ULL))) r += 1ULL;
    }
    y = pow2_scale((double)r, q);
  }
  if (y > f.xmax) y = __longlong_as_double(0x7FF0000000000000LL);
  if (!f.sub && y < f.xmin) y = 0.0;
  return (b >> 63) ? -y : y;
}

// ------------------------------------------------------------------------
// `sr + 1j*si` exactly as NumPy evaluates it: (sr + (0*si - 0), 0 + (0 + si))
// A non-finite imaginary part turns the real part into NaN; zero signs are
// normalised the same way the reference's assembly normalises them.
// ------------------------------------------------------------------------
__device__ __forceinline__ double2 assemble(double sr, double si) {
  double t = __dsub_rn(__dmul_rn(0.0, si), 0.0);
  return make_double2(__dadd_rn(sr, t), __dadd_rn(0.0, __dadd_rn(0.0, si)));
}

// NumPy complex128 division (Smith), each op separately rounded.  1/x is the
// correctly rounded reciprocal (__drcp_rn == __ddiv_rn(1.0, x) bit for bit,
// IEEE special cases included) -- a shorter dependent sequence than DDIV.
#ifndef FPM_NO_DRCP
#define FPM_RCP(v) __drcp_rn(v)
#else
#define FPM_RCP(v) __ddiv_rn(1.0, (v))
#endif
__device__ __forceinline__ double2 cdiv(double2 n, double2 d) {
  double adr = fabs(d.x), adi = fabs(d.y);
  if (adr >= adi) {
    if (adr == 0.0 && adi == 0.0)
      return make_double2(__ddiv_rn(n.x, adr), __ddiv_rn(n.y, adr));
    double rat = __ddiv_rn(d.y, d.x);
    double scl = FPM_RCP(__dadd_rn(d.x, __dmul_rn(d.y, rat)));
    return make_double2(__dmul_rn(__dadd_rn(n.x, __dmul_rn(n.y, rat)), scl),
                        __dmul_rn(__dsub_rn(n.y, __dmul_rn(n.x, rat)), scl));
  }
  double rat = __ddiv_rn(d.x, d.y);
  double scl = FPM_RCP(__dadd_rn(d.y, __dmul_rn(d.x, rat)));
  return make_double2(__dmul_rn(__dadd_rn(__dmul_rn(n.x, rat), n.y), scl),
                      __dmul_rn(__dsub_rn(__dmul_rn(n.y, rat), n.x), scl));
}

// ------------------------------------------------------------------------
// Per-format complex arithmetic.  C = the complex type in that format.
//   rnd(double2)      round a binary64 complex into the format (one rounding)
//   mul(a, b)         _cmul(ar, ai, br, bi)
//   mulc(u, v)        _cmul(ur, -ui, vr, vi)   (dot_fp's conjugated product)
//   add(a, b)         _cadd
//   wide(c)           exact binary64 value
// ------------------------------------------------------------------------
// half2 / bfloat162 lanes: .x = real (low 16 bits), .y = imag (high 16 bits)
__device__ __forceinline__ unsigned h2u(__half2 h) { return *reinterpret_cast<unsigned*>(&h); }
__device__ __forceinline__ __half2 u2h(unsigned u) { return *reinterpret_cast<__half2*>(&u); }
__device__ __forceinline__ unsigned b2u(__nv_bfloat162 h) { return *reinterpret_cast<unsigned*>(&h); }
__device__ __forceinline__ __nv_bfloat162 u2b(unsigned u) { return *reinterpret_cast<__nv_bfloat162*>(&u); }

template <int K> struct Ar;

// Extra per-format members used by the matvec / dot kernels:
//   P, prep(v)   "prepared" right operand of a matvec product (see F16)
//   mulp(a, p)   == mul(a, v) bit for bit
//   asmc(c)      the reference's `re + 1j*im` assembly applied in-format
template <> struct Ar<FK_F64> {
  typedef double2 C;
  typedef double2 P;
  static __device__ __forceinline__ P prep(C v) { return v; }
  static __device__ __forceinline__ C mulp(C a, P v, const FmtP& f) { return mul(a, v, f); }
  static __device__ __forceinline__ C asmc(C c) { return assemble(c.x, c.y); }
  static __device__ __forceinline__ C rnd(double2 v, const FmtP&) { return v; }
  static __device__ __forceinline__ C mul(C a, C b, const FmtP&) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
  }
  static __device__ __forceinline__ C mulc(C u, C v, const FmtP& f) {
    return mul(make_double2(u.x, -u.y), v, f);
  }
  static __device__ __forceinline__ C add(C a, C b, const FmtP&) {
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
  }
  static __device__ __forceinline__ double2 wide(C c) { return c; }
};

template <> struct Ar<FK_GEN> {
  typedef double2 C;
  typedef double2 P;
  static __device__ __forceinline__ P prep(C v) { return v; }
  static __device__ __forceinline__ C mulp(C a, P v, const FmtP& f) { return mul(a, v, f); }
  static __device__ __forceinline__ C asmc(C c) { return assemble(c.x, c.y); }
  static __device__ __forceinline__ C rnd(double2 v, const FmtP& f) {
    return make_double2(gen_round(v.x, f), gen_round(v.y, f));
  }
  static __device__ __forceinline__ C mul(C a, C b, const FmtP& f) {
    double rr = gen_round(__dsub_rn(gen_round(__dmul_rn(a.x, b.x), f), gen_round(__dmul_rn(a.y, b.y), f)), f);
    double ri = gen_round(__dadd_rn(gen_round(__dmul_rn(a.x, b.y), f), gen_round(__dmul_rn(a.y, b.x), f)), f);
    return make_double2(rr, ri);
  }
  static __device__ __forceinline__ C mulc(C u, C v, const FmtP& f) {
    return mul(make_double2(u.x, -u.y), v, f);
  }
  static __device__ __forceinline__ C add(C a, C b, const FmtP& f) {
    return make_double2(gen_round(__dadd_rn(a.x, b.x), f), gen_round(__dadd_rn(a.y, b.y), f));
  }
  static __device__ __forceinline__ double2 wide(C c) { return c; }
};

template <> struct Ar<FK_F32> {
  typedef float2 C;
  typedef float2 P;
  static __device__ __forceinline__ P prep(C v) { return v; }
  static __device__ __forceinline__ C mulp(C a, P v, const FmtP& f) { return mul(a, v, f); }
  static __device__ __forceinline__ C asmc(C c) {
    // (re + (0*im - 0), 0 + (0 + im)) in binary32 (exact: same rules as binary64)
    float t = __fsub_rn(__fmul_rn(0.0f, c.y), 0.0f);
    return make_float2(__fadd_rn(c.x, t), __fadd_rn(0.0f, __fadd_rn(0.0f, c.y)));
  }
  static __device__ __forceinline__ C rnd(double2 v, const FmtP&) {
    return make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
  }
  static __device__ __forceinline__ C mul(C a, C b, const FmtP&) {
    return make_float2(__fsub_rn(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)),
                       __fadd_rn(__fmul_rn(a.x, b.y), __fmul_rn(a.y, b.x)));
  }
  static __device__ __forceinline__ C mulc(C u, C v, const FmtP& f) {
    return mul(make_float2(u.x, -u.y), v, f);
  }
  static __device__ __forceinline__ C add(C a, C b, const FmtP&) {
    return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
  }
  static __device__ __forceinline__ double2 wide(C c) { return make_double2((double)c.x, (double)c.y); }
};


template <> struct Ar<FK_F16> {
  typedef __half2 C;
  // P = (v, rot(v)) with rot(v) = (-vi, vr): a*v = lo(a)*v + hi(a)*rot(v)
  // lane-wise: (ar*vr + ai*(-vi), ar*vi + ai*vr); fl(x*(-y)) = -fl(x*y), so
  // this equals _cmul's fl(fl(ar vr) - fl(ai vi)), fl(fl(ar vi) + fl(ai vr)).
  struct P {
    __half2 v1, v2;
  };
  static __device__ __forceinline__ P prep(C v) {
    P p;
    p.v1 = v;
    p.v2 = u2h(h2u(__lowhigh2highlow(v)) ^ 0x00008000u);
    return p;
  }
  static __device__ __forceinline__ C mulp(C a, P p, const FmtP&) {
    return __hadd2_rn(__hmul2_rn(__low2half2(a), p.v1), __hmul2_rn(__high2half2(a), p.v2));
  }
  static __device__ __forceinline__ C asmc(C c) {
    unsigned u = h2u(c), re = u & 0xFFFFu, im = u >> 16;
    if ((im & 0x7C00u) == 0x7C00u) re = 0x7E00u;           // non-finite imag -> NaN real
    else if (re == 0x8000u && !(im & 0x8000u)) re = 0u;    // -0 + (+0) = +0
    if (im == 0x8000u) im = 0u;                            // 0 + -0 = +0
    return u2h(re | (im << 16));
  }
  static __device__ __forceinline__ C rnd(double2 v, const FmtP&) {
    // cvt.rn.f16.f64: a single rounding (never via fp32)
    return __halves2half2(__double2half(v.x), __double2half(v.y));
  }
  static __device__ __forceinline__ C mul(C a, C b, const FmtP&) {
    // P = (ar*br, ar*bi); Q = (ai*bi, ai*br); result = (P.x - Q.x, P.y + Q.y)
    C P = __hmul2_rn(__low2half2(a), b);
    C Q = __hmul2_rn(__high2half2(a), __lowhigh2highlow(b));
    return __hadd2_rn(P, u2h(h2u(Q) ^ 0x00008000u));
  }
  static __device__ __forceinline__ C mulc(C u, C v, const FmtP& f) {
    return mul(u2h(h2u(u) ^ 0x80000000u), v, f);
  }
  static __device__ __forceinline__ C add(C a, C b, const FmtP&) { return __hadd2_rn(a, b); }
  static __device__ __forceinline__ double2 wide(C c) {
    return make_double2((double)__low2float(c), (double)__high2float(c));
  }
};

template <> struct Ar<FK_BF16> {
  typedef __nv_bfloat162 C;
  struct P {
    __nv_bfloat162 v1, v2;
  };
  static __device__ __forceinline__ P prep(C v) {
    P p;
    p.v1 = v;
    p.v2 = u2b(b2u(__lowhigh2highlow(v)) ^ 0x00008000u);
    return p;
  }
  static __device__ __forceinline__ C mulp(C a, P p, const FmtP&) {
    return __hadd2_rn(__hmul2_rn(__low2bfloat162(a), p.v1), __hmul2_rn(__high2bfloat162(a), p.v2));
  }
  static __device__ __forceinline__ C asmc(C c) {
    unsigned u = b2u(c), re = u & 0xFFFFu, im = u >> 16;
    if ((im & 0x7F80u) == 0x7F80u) re = 0x7FC0u;
    else if (re == 0x8000u && !(im & 0x8000u)) re = 0u;
    if (im == 0x8000u) im = 0u;
    return u2b(re | (im << 16));
  }
  static __device__ __forceinline__ C rnd(double2 v, const FmtP&) {
    return __halves2bfloat162(__double2bfloat16(v.x), __double2bfloat16(v.y));  // cvt.rn.bf16.f64
  }
  static __device__ __forceinline__ C mul(C a, C b, const FmtP&) {
    C P = __hmul2_rn(__low2bfloat162(a), b);
    C Q = __hmul2_rn(__high2bfloat162(a), __lowhigh2highlow(b));
    return __hadd2_rn(P, u2b(b2u(Q) ^ 0x00008000u));
  }
  static __device__ __forceinline__ C mulc(C u, C v, const FmtP& f) {
    return mul(u2b(b2u(u) ^ 0x80000000u), v, f);
  }
  static __device__ __forceinline__ C add(C a, C b, const FmtP&) { return __hadd2_rn(a, b); }
  static __device__ __forceinline__ double2 wide(C c) {
    return make_double2((double)__low2float(c), (double)__high2float(c));
  }
};

// Round into the work format and assemble like round_complex (formats.py:146)
template <int WK>
__device__ __forceinline__ double2 work_round_c(double2 q, const FmtP& w) {
  if (WK == FK_F64) return q;
  if (w.native) return q;
  return assemble(gen_round(q.x, w), gen_round(q.y, w));
}

// _wdiv (solvers.py:256-259); noinline: one shared copy (see fpm_cg.cuh)
template <int WK>
__device__ __noinline__ double2 wdiv(double2 num, double2 den, const FmtP& w) {
  return work_round_c<WK>(cdiv(num, den), w);
}

// axpy_fp (linalg.py:100-119) at the work format; returns assembled y + a*x
template <int WK>
__device__ __forceinline__ double2 axpy1(double2 a, double2 x, double2 y, const FmtP& w) {
  typedef Ar<WK> A;
  double2 t = A::mul(A::rnd(a, w), A::rnd(x, w), w);
  double2 s = A::add(A::rnd(y, w), t, w);
  return assemble(s.x, s.y);
}

__device__ __forceinline__ bool finite2(double2 v) { return isfinite(v.x) && isfinite(v.y); }

}  // namespace fpm
