// Kernels and C ABI of libfpmimo_b200.so (see include/fpmimo_b200.h).
//
//   fpm_detect_kernel  fused Gram/MF -> BJ setup -> (BJ-)CG -> slicer/counter
//   fpm_gram_kernel    Gram/MF to global A, b
//   fpm_bj_kernel      block-Jacobi Hermitian inverses from global A
//   fpm_cg_kernel      (BJ-)CG from global A, b, Minv
//   fpm_slice_kernel   slicer + error counters
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "../../include/fpmimo_b200.h"
#include "fpm_arith.cuh"
#include "fpm_cg.cuh"
#include "fpm_gram.cuh"
#include "fpm_ptx.cuh"

namespace fpm {

static std::atomic<long long> g_launches{0};
static long long* g_trace = nullptr;  // diagnostic phase timestamps (fpm_debug_set_trace)

constexpr int kMaxN = 128;
constexpr int kMaxL = 16;
constexpr int kMaxM = 4096;

struct Slicer {
  double th[7];
  int nth;  // 3 (16-QAM) or 7 (64-QAM)
  int bpa;  // bits per axis
};

// ---------------------------------------------------------------------------
// Hermitian-PD block inverse via Cholesky (fp64).  The reference inverts with
// LAPACK zgesv (solvers.py:250-251) after a Cholesky PD check
// (solvers.py:246-249) and symmetrizes (solvers.py:252); the bits of a
// LAPACK inverse are not portable, so parity for this piece is a tolerance
// (or Minv is injected).  B: Lk x Lk row-major (full Hermitian) -> inverse,
// in place; C: scratch Lk x Lk.
// ---------------------------------------------------------------------------
__device__ bool hpd_inverse(double2* B, double2* C, int Lk) {
  for (int j = 0; j < Lk; ++j) {
    double d = B[j * Lk + j].x;
    for (int k = 0; k < j; ++k) {
      double2 c = C[j * Lk + k];
      d = d - (c.x * c.x + c.y * c.y);
    }
    if (!(d > 0.0)) return false;
    double cjj = sqrt(d);
    C[j * Lk + j] = make_double2(cjj, 0.0);
    for (int i = j + 1; i < Lk; ++i) {
      double2 s = B[i * Lk + j];
      for (int k = 0; k < j; ++k) {
        double2 a = C[i * Lk + k], b = C[j * Lk + k];  // s -= a * conj(b)
        s.x -= a.x * b.x + a.y * b.y;
        s.y -= a.y * b.x - a.x * b.y;
      }
      C[i * Lk + j] = make_double2(s.x / cjj, s.y / cjj);
    }
  }
  // Linv (lower) into B
  for (int i = 0; i < Lk; ++i) {
    const double cii = C[i * Lk + i].x;
    for (int j = 0; j < i; ++j) {
      double2 s = make_double2(0.0, 0.0);
      for (int k = j; k < i; ++k) {
        double2 a = C[i * Lk + k], b = B[k * Lk + j];
        s.x += a.x * b.x - a.y * b.y;
        s.y += a.x * b.y + a.y * b.x;
      }
      B[i * Lk + j] = make_double2(-s.x / cii, -s.y / cii);
    }
    B[i * Lk + i] = make_double2(1.0 / cii, 0.0);
  }
  // Minv = Linv^H Linv (upper incl. diagonal) into C
  for (int i = 0; i < Lk; ++i)
    for (int j = i; j < Lk; ++j) {
      double2 s = make_double2(0.0, 0.0);
      for (int k = j; k < Lk; ++k) {
        double2 a = B[k * Lk + i], b = B[k * Lk + j];  // conj(a) * b
        s.x += a.x * b.x + a.y * b.y;
        s.y += a.x * b.y - a.y * b.x;
      }
      C[i * Lk + j] = s;
    }
  for (int i = 0; i < Lk; ++i)
    for (int j = i; j < Lk; ++j) {
      double2 v = C[i * Lk + j];
      if (i == j) {
        B[i * Lk + i] = make_double2(v.x, 0.0);
      } else {
        B[i * Lk + j] = v;
        B[j * Lk + i] = make_double2(v.x, -v.y);
      }
    }
  return true;
}

// Level index = #thresholds strictly below v (digitize right=True; NaN -> 0,
// detect.py:70-75), then the per-axis Gray label (detect.py:50).
__device__ __forceinline__ int level_index(double v, const Slicer& sl) {
  int idx = 0;
#pragma unroll
  for (int k = 0; k < 7; ++k)
    if (k < sl.nth && v > sl.th[k]) ++idx;
  return idx;
}

// Slices x[q] and compares with tx; returns (bit errors) and sets *sym_err.
__device__ __forceinline__ int slice_one(double2 x, const uint8_t* tx, uint8_t* rx, const Slicer& sl,
                                         int* sym_err) {
  int gi = level_index(x.x, sl), gq = level_index(x.y, sl);
  gi ^= gi >> 1;
  gq ^= gq >> 1;
  int errs = 0;
  for (int k = 0; k < sl.bpa; ++k) {
    uint8_t bi = (uint8_t)((gi >> (sl.bpa - 1 - k)) & 1);
    uint8_t bq = (uint8_t)((gq >> (sl.bpa - 1 - k)) & 1);
    if (rx) {
      rx[k] = bi;
      rx[sl.bpa + k] = bq;
    }
    if (tx) errs += (tx[k] != bi) + (tx[sl.bpa + k] != bq);
  }
  *sym_err = errs > 0;
  return errs;
}

__device__ __forceinline__ void block_add_counters(unsigned long long* cnt_smem, unsigned long long* cnt_g,
                                                   int tid, int nthreads) {
  __syncthreads();
  if (tid < FPM_NCOUNTERS && cnt_smem[tid]) atomicAdd(&cnt_g[tid], cnt_smem[tid]);
}

// ---------------------------------------------------------------------------
// Fused detector
// ---------------------------------------------------------------------------
struct DetectArgs {
  const double2* H;
  const double2* y;
  const uint8_t* tx;
  long T;
  double sigma2;
  int L, iters, bj, textbook;
  Prec pr;
  const double2* minv_in;
  double2* x;
  int* brk;
  int* div;
  uint8_t* rx;
  unsigned long long* counters;
  Slicer sl;
  GramGeom G;
  int ldA;
  // dynamic shared memory offsets (bytes)
  int off_ys, off_union, off_minv, off_scr, off_vec, off_pmv, off_tip, off_sc, off_fl;
  int smem_bytes;
  long long* trace;  // nullable: [0] start [1] gram done [2] bj done [3..9] cg phases it=1 [10] cg done [11] end
};

template <int WK, int MVK, int IPK>
struct EmitSmem {
  CgSmem<MVK, IPK>* S;
  const FmtP* fm;
  int bj;
  __device__ __forceinline__ void a(int g, int i, int j, double2 v) {
    const int N = S->N;
    S->At[(long)g * N * S->ldA + (long)j * S->ldA + i] = Ar<MVK>::rnd(v, *fm);
    if (bj) {
      const int L = S->L;
      const int kb = i / L;
      if (kb == j / L) {
        const int Lk = min(L, N - kb * L);
        S->minv[(long)g * N * L + kb * L * L + (i - kb * L) * Lk + (j - kb * L)] = v;
      }
    }
  }
  __device__ __forceinline__ void b(int g, int n, double2 v) { S->b[g * S->N + n] = v; }
};

template <int WK, int MVK, int IPK>
__global__ void __launch_bounds__(512, 1) fpm_detect_kernel(const DetectArgs args) {
  extern __shared__ __align__(128) unsigned char smem[];
  typedef typename Ar<MVK>::C MC;
  const int tid = threadIdx.x, nthreads = blockDim.x;
  const GramGeom& G = args.G;
  const long t0 = (long)blockIdx.x * G.R;
  const int Rv = (int)min((long)G.R, args.T - t0);
  const int N = G.N;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);  // S full, S empty, 1 y
  __shared__ unsigned long long cnt[FPM_NCOUNTERS];
  typedef typename Ar<IPK>::C IC;
  CgSmem<MVK, IPK> S;
  S.R = G.R;
  S.N = N;
  S.L = args.bj ? args.L : 1;
  S.ldA = args.ldA;
  S.At = reinterpret_cast<MC*>(smem + args.off_union);
  S.minv = reinterpret_cast<double2*>(smem + args.off_minv);
  double2* vec = reinterpret_cast<double2*>(smem + args.off_vec);
  const long RN = (long)G.R * N;
  S.b = vec;
  S.x = vec + RN;
  S.r = vec + 2 * RN;
  S.p = vec + 3 * RN;
  S.z = vec + 4 * RN;
  S.w = vec + 5 * RN;
  S.xn = vec + 6 * RN;
  S.rn = vec + 7 * RN;
  S.pmv = reinterpret_cast<MC*>(smem + args.off_pmv);
  S.tphi = reinterpret_cast<IC*>(smem + args.off_tip);
  S.trho = S.tphi + RN;
  S.tr1 = S.trho + RN;
  S.sc = reinterpret_cast<double2*>(smem + args.off_sc);
  S.fl = reinterpret_cast<int*>(smem + args.off_fl);

  if (tid == 0) {
    for (int s = 0; s < G.S; ++s) {
      mbar_init(&bars[s], 1);
      mbar_init(&bars[G.S + s], nthreads / 32);
    }
    mbar_init(&bars[2 * G.S], 1);
    fence_mbar_init();
  }
  if (tid < FPM_NCOUNTERS) cnt[tid] = 0ULL;
  for (int g = tid; g < G.R; g += nthreads) S.fl[g * 4] = g < Rv ? 1 : 0;
  long long* tr = (args.trace && blockIdx.x == 0) ? args.trace : nullptr;
  FPM_STAMP(tr, 0);
  __syncthreads();

  // 1) Gram + matched filter straight into shared memory
  EmitSmem<WK, MVK, IPK> em;
  em.S = &S;
  em.fm = &args.pr.mv;
  em.bj = args.bj && !args.minv_in;
  gram_run(args.H, args.y, t0, Rv, G, args.sigma2, reinterpret_cast<double2*>(smem + args.off_union),
           reinterpret_cast<double2*>(smem + args.off_ys), bars, nthreads, tid, em);
  FPM_STAMP(tr, 1);

  // 2) block-Jacobi inverses (on-chip fp64 Cholesky, or injected)
  if (args.bj) {
    const int L = args.L;
    const int nblk = (N + L - 1) / L;
    if (args.minv_in) {
      for (long q = tid; q < (long)Rv * N * L; q += nthreads) {
        const int g = (int)(q / ((long)N * L));
        const long e = q - (long)g * N * L;
        S.minv[q] = Ar<WK>::rnd(args.minv_in[(t0 + g) * (long)N * L + e], args.pr.work);
      }
    } else {
      double2* scr = reinterpret_cast<double2*>(smem + args.off_scr);
      for (int q = tid; q < Rv * nblk; q += nthreads) {
        const int g = q / nblk, kb = q - g * nblk;
        const int Lk = min(L, N - kb * L);
        double2* B = S.minv + (long)g * N * L + kb * L * L;
        if (!hpd_inverse(B, scr + (long)g * N * L + kb * L * L, Lk)) {
          atomicExch(&S.fl[g * 4], 0);
          atomicAdd(&cnt[FPM_CNT_NONPD], 1ULL);
        } else if (WK != FK_F64) {
          for (int e = 0; e < Lk * Lk; ++e) B[e] = Ar<WK>::rnd(B[e], args.pr.work);
        }
      }
    }
    __syncthreads();
  }

  FPM_STAMP(tr, 2);
  // 3) CG in shared memory
  cg_team<WK, MVK, IPK>(S, Rv, args.iters, args.bj != 0, args.textbook != 0, args.pr, nthreads, tid,
                        tr ? tr + 3 : nullptr);

  // 4) slicer + counters + write-back
  const int bps = 2 * args.sl.bpa;
  unsigned long long be = 0, se = 0;
  for (int q = tid; q < Rv * N; q += nthreads) {
    const int g = q / N, n = q - g * N;
    const long gq = (t0 + g) * (long)N + n;
    const double2 xv = S.x[q];
    args.x[gq] = xv;
    int sym;
    be += slice_one(xv, args.tx ? args.tx + gq * bps : nullptr, args.rx ? args.rx + gq * bps : nullptr,
                    args.sl, &sym);
    se += sym;
  }
  for (int off = 16; off; off >>= 1) {
    be += __shfl_xor_sync(0xffffffffu, be, off);
    se += __shfl_xor_sync(0xffffffffu, se, off);
  }
  if ((tid & 31) == 0) {
    if (be) atomicAdd(&cnt[FPM_CNT_BIT_ERRORS], be);
    if (se) atomicAdd(&cnt[FPM_CNT_SYMBOL_ERRORS], se);
  }
  for (int g = tid; g < Rv; g += nthreads) {
    const int bk = S.fl[g * 4 + 2], dv = S.fl[g * 4 + 3];
    args.brk[t0 + g] = bk;
    args.div[t0 + g] = dv;
    if (dv >= 0) atomicAdd(&cnt[FPM_CNT_DIVERGED], 1ULL);
    if (bk >= 0) atomicAdd(&cnt[FPM_CNT_BREAKDOWN], 1ULL);
  }
  if (tid == 0) atomicAdd(&cnt[FPM_CNT_TRIALS], (unsigned long long)Rv);
  block_add_counters(cnt, args.counters, tid, nthreads);
  FPM_STAMP(tr, 11);
}

// ---------------------------------------------------------------------------
// Standalone Gram
// ---------------------------------------------------------------------------
struct EmitGlobal {
  double2* Aout;
  double2* bout;
  long t0;
  int N;
  __device__ __forceinline__ void a(int g, int i, int j, double2 v) {
    Aout[((t0 + g) * (long)N + i) * N + j] = v;
  }
  __device__ __forceinline__ void b(int g, int n, double2 v) { bout[(t0 + g) * (long)N + n] = v; }
};

struct GramArgs {
  const double2* H;
  const double2* y;
  long T;
  double sigma2;
  double2* A;
  double2* b;
  GramGeom G;
  int off_ys, off_union;
};

__global__ void __launch_bounds__(512, 1) fpm_gram_kernel(const GramArgs args) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, nthreads = blockDim.x;
  const GramGeom& G = args.G;
  const long t0 = (long)blockIdx.x * G.R;
  const int Rv = (int)min((long)G.R, args.T - t0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  if (tid == 0) {
    for (int s = 0; s < G.S; ++s) {
      mbar_init(&bars[s], 1);
      mbar_init(&bars[G.S + s], nthreads / 32);
    }
    mbar_init(&bars[2 * G.S], 1);
    fence_mbar_init();
  }
  __syncthreads();
  EmitGlobal em;
  em.Aout = args.A;
  em.bout = args.b;
  em.t0 = t0;
  em.N = G.N;
  gram_run(args.H, args.y, t0, Rv, G, args.sigma2, reinterpret_cast<double2*>(smem + args.off_union),
           reinterpret_cast<double2*>(smem + args.off_ys), bars, nthreads, tid, em);
}

// ---------------------------------------------------------------------------
// Standalone block-Jacobi setup: one thread per (realization, block)
// ---------------------------------------------------------------------------
__global__ void fpm_bj_kernel(const double2* __restrict__ A, long T, int N, int L, double2* __restrict__ Minv,
                              int* bad_block, unsigned int* nonpd) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int nblk = (N + L - 1) / L;
  const long q = (long)blockIdx.x * blockDim.x + threadIdx.x;
  double2* B = reinterpret_cast<double2*>(smem) + (long)threadIdx.x * 2 * L * L;
  double2* C = B + L * L;
  if (q >= T * nblk) return;
  const long t = q / nblk;
  const int kb = (int)(q - t * nblk);
  const int s0 = kb * L, Lk = min(L, N - s0);
  for (int i = 0; i < Lk; ++i)
    for (int j = 0; j < Lk; ++j) B[i * Lk + j] = A[(t * N + s0 + i) * (long)N + s0 + j];
  bool ok = hpd_inverse(B, C, Lk);
  double2* out = Minv + t * (long)N * L + (long)kb * L * L;
  for (int e = 0; e < Lk * Lk; ++e) out[e] = B[e];
  if (!ok) {
    atomicAdd(nonpd, 1u);
    if (bad_block) atomicMin(&bad_block[t], s0);
  }
}

__global__ void fpm_bad_fix_kernel(int* bad_block, long T) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T && bad_block[t] == 0x7f7f7f7f) bad_block[t] = -1;
}

// ---------------------------------------------------------------------------
// Standalone CG from global A / b / Minv
// ---------------------------------------------------------------------------
struct CgArgs {
  const double2* A;
  const double2* b;
  const double2* minv;
  long T;
  int N, L, iters, bj, textbook, R, ldA;
  Prec pr;
  double2* x;
  int* brk;
  int* div;
  int off_minv, off_vec, off_pmv, off_tip, off_sc, off_fl;
};

template <int WK, int MVK, int IPK>
__global__ void __launch_bounds__(256) fpm_cg_kernel(const CgArgs args) {
  extern __shared__ __align__(128) unsigned char smem[];
  typedef typename Ar<MVK>::C MC;
  typedef typename Ar<IPK>::C IC;
  const int tid = threadIdx.x, nthreads = blockDim.x;
  const long t0 = (long)blockIdx.x * args.R;
  const int Rv = (int)min((long)args.R, args.T - t0);
  const int N = args.N;
  CgSmem<MVK, IPK> S;
  S.R = args.R;
  S.N = N;
  S.L = args.bj ? args.L : 1;
  S.ldA = args.ldA;
  S.At = reinterpret_cast<MC*>(smem);
  S.minv = reinterpret_cast<double2*>(smem + args.off_minv);
  double2* vec = reinterpret_cast<double2*>(smem + args.off_vec);
  const long RN = (long)args.R * N;
  S.b = vec;
  S.x = vec + RN;
  S.r = vec + 2 * RN;
  S.p = vec + 3 * RN;
  S.z = vec + 4 * RN;
  S.w = vec + 5 * RN;
  S.xn = vec + 6 * RN;
  S.rn = vec + 7 * RN;
  S.pmv = reinterpret_cast<MC*>(smem + args.off_pmv);
  S.tphi = reinterpret_cast<IC*>(smem + args.off_tip);
  S.trho = S.tphi + RN;
  S.tr1 = S.trho + RN;
  S.sc = reinterpret_cast<double2*>(smem + args.off_sc);
  S.fl = reinterpret_cast<int*>(smem + args.off_fl);

  // A (row-major, global) -> At (transposed, u_MV), coalesced along k
  const long NN = (long)N * N;
  for (long q = tid; q < (long)Rv * NN; q += nthreads) {
    const int g = (int)(q / NN);
    const long e = q - g * NN;
    const int i = (int)(e / N), k = (int)(e - (long)i * N);
    S.At[(long)g * N * S.ldA + (long)k * S.ldA + i] = Ar<MVK>::rnd(args.A[(t0 + g) * NN + e], args.pr.mv);
  }
  for (long q = tid; q < (long)Rv * N; q += nthreads) S.b[q] = args.b[t0 * N + q];
  if (args.bj)
    for (long q = tid; q < (long)Rv * N * args.L; q += nthreads)
      S.minv[q] = Ar<WK>::rnd(args.minv[t0 * (long)N * args.L + q], args.pr.work);
  for (int g = tid; g < args.R; g += nthreads) S.fl[g * 4] = g < Rv ? 1 : 0;
  __syncthreads();
  cg_team<WK, MVK, IPK>(S, Rv, args.iters, args.bj != 0, args.textbook != 0, args.pr, nthreads, tid);
  for (long q = tid; q < (long)Rv * N; q += nthreads) args.x[t0 * N + q] = S.x[q];
  for (int g = tid; g < Rv; g += nthreads) {
    args.brk[t0 + g] = S.fl[g * 4 + 2];
    args.div[t0 + g] = S.fl[g * 4 + 3];
  }
}

// ---------------------------------------------------------------------------
// Standalone slicer / counter
// ---------------------------------------------------------------------------
__global__ void fpm_slice_kernel(const double2* __restrict__ x, const uint8_t* __restrict__ tx, long TN,
                                 uint8_t* rx, unsigned long long* counters, Slicer sl) {
  __shared__ unsigned long long cnt[2];
  if (threadIdx.x < 2) cnt[threadIdx.x] = 0ULL;
  __syncthreads();
  const int bps = 2 * sl.bpa;
  unsigned long long be = 0, se = 0;
  for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < TN; q += (long)gridDim.x * blockDim.x) {
    int sym;
    be += slice_one(x[q], tx ? tx + q * bps : nullptr, rx ? rx + q * bps : nullptr, sl, &sym);
    se += sym;
  }
  for (int off = 16; off; off >>= 1) {
    be += __shfl_xor_sync(0xffffffffu, be, off);
    se += __shfl_xor_sync(0xffffffffu, se, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&cnt[0], be);
    atomicAdd(&cnt[1], se);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (cnt[0]) atomicAdd(&counters[FPM_CNT_BIT_ERRORS], cnt[0]);
    if (cnt[1]) atomicAdd(&counters[FPM_CNT_SYMBOL_ERRORS], cnt[1]);
  }
}

// ---------------------------------------------------------------------------
// FP64 issue-rate probe: independent non-fused DMUL/DADD chains (the only DP
// ops the bit-exact Gram may use).  Gives the denominator of the fp64
// roofline, which MEASURED_PEAKS.json does not carry.
// ---------------------------------------------------------------------------
__global__ void fpm_dp_probe_kernel(double* out, long iters) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + 1e-3 * (threadIdx.x + k);
  const double c1 = 0.999999999, c2 = 1e-9;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __dadd_rn(__dmul_rn(a[k], c1), c2);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // keep the work alive
}

// ===========================================================================
// Host side
// ===========================================================================

static int classify(const fpm_format& f) {
  if (f.subnormals) {
    if (f.sig_bits == 53 && f.exp_bits == 11) return FK_F64;
    if (f.sig_bits == 24 && f.exp_bits == 8) return FK_F32;
    if (f.sig_bits == 11 && f.exp_bits == 5) return FK_F16;
    if (f.sig_bits == 8 && f.exp_bits == 8) return FK_BF16;
  }
  return FK_GEN;
}

static bool valid_format(const fpm_format& f) {
  return f.sig_bits >= 2 && f.exp_bits >= 2 && f.sig_bits <= 53 && f.exp_bits <= 11;
}

static FmtP make_fmtp(const fpm_format& f) {
  FmtP p;
  const int bias = (1 << (f.exp_bits - 1)) - 1;
  p.sig = f.sig_bits;
  p.qmin = (1 - bias) - f.sig_bits + 1;
  p.sub = f.subnormals ? 1 : 0;
  p.native = (f.sig_bits == 53 && f.exp_bits == 11 && f.subnormals) ? 1 : 0;
  p.xmax = (2.0 - std::ldexp(1.0, 1 - f.sig_bits)) * std::ldexp(1.0, bias);
  p.xmin = std::ldexp(1.0, 1 - bias);
  return p;
}

static double unit_roundoff(const fpm_format& f) { return std::ldexp(1.0, -f.sig_bits); }

// Kernel instance selector: W in {F64, GEN}; MV == IP when native.
struct Kinds {
  int w, mv, ip;
};

static Kinds pick_kinds(const fpm_precision& p) {
  Kinds k;
  // test hook: run the integer-emulation path for every format (it must give
  // the same bits as the native-arithmetic kernels)
  const char* fg = std::getenv("FPM_FORCE_GENERIC");
  const bool force_gen = fg && fg[0] == '1';
  if (force_gen) return {FK_GEN, FK_GEN, FK_GEN};
  int w = classify(p.work), mv = classify(p.matvec), ip = classify(p.inner);
  if (w != FK_F64) return {FK_GEN, FK_GEN, FK_GEN};
  if (mv == ip && mv != FK_GEN) return {FK_F64, mv, mv};
  k = {FK_F64, FK_GEN, FK_GEN};
  return k;
}

static Slicer make_slicer(int qam) {
  Slicer s;
  std::memset(&s, 0, sizeof(s));
  if (qam == 64) {
    const double sc = 1.0 / std::sqrt(42.0);
    for (int k = 0; k < 7; ++k) s.th[k] = (2.0 * k - 6.0) * sc;
    s.nth = 7;
    s.bpa = 3;
  } else {
    const double sc = 1.0 / std::sqrt(10.0);  // detect.py:45, 51
    s.th[0] = -2.0 * sc;
    s.th[1] = 0.0 * sc;
    s.th[2] = 2.0 * sc;
    s.nth = 3;
    s.bpa = 2;
  }
  return s;
}

static int mv_bytes(int kind) {
  switch (kind) {
    case FK_F32: return 8;
    case FK_F16:
    case FK_BF16: return 4;
    default: return 16;
  }
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

static int max_smem_optin() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int s = 0;
    if (cudaDeviceGetAttribute(&s, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || s <= 0)
      s = 227 * 1024;
    v = s;
  }
  return v;
}

// Gram geometry for a given R: fills G and the union/ys sizes.
static void gram_geom(int R, int M, int N, GramGeom& G) {
  G.R = R;
  G.M = M;
  G.N = N;
  G.Np = (N + 7) / 8 * 8;
  G.nb = G.Np / 4;
  G.S = 3;
  const long row_bytes = (long)R * G.Np * 16;
  int mc = (int)std::max(1L, (long)(24 * 1024) / row_bytes);
  G.MC = std::min(mc, M);
}

static int gram_threads(const GramGeom& G) {
  int t = G.R * G.nb * G.nb / 2;
  return (t + 31) / 32 * 32;
}

// Plan the fused kernel for (M, N, L, kinds); returns false if it cannot fit.
static bool plan_detect(int M, int N, int L, int bj, int mvk, int ipk, DetectArgs& a, int& threads) {
  const int Np = (N + 7) / 8 * 8;
  int R = std::max(1, 256 / Np);
  const int limit = max_smem_optin();
  for (; R >= 1; R = (R > 1 ? R / 2 : 0)) {
    GramGeom G;
    gram_geom(R, M, N, G);
    threads = gram_threads(G);
    if (threads > 512) continue;
    const int ldA = N + 1;
    size_t off = 128;  // mbarriers (2S+1)
    a.off_ys = (int)off;
    off = align_up(off + (size_t)R * M * 16, 128);
    a.off_union = (int)off;
    size_t stage_b = (size_t)G.S * R * G.MC * G.Np * 16;
    size_t at_b = (size_t)R * N * ldA * mv_bytes(mvk);
    off = align_up(off + std::max(stage_b, at_b), 128);
    a.off_minv = (int)off;
    const int Lb = bj ? L : 1;
    off = align_up(off + (bj ? (size_t)R * N * Lb * 16 : 0), 128);
    a.off_scr = (int)off;
    off = align_up(off + (bj ? (size_t)R * N * Lb * 16 : 0), 128);
    a.off_vec = (int)off;
    off = align_up(off + (size_t)8 * R * N * 16, 128);
    a.off_pmv = (int)off;
    off = align_up(off + (size_t)R * N * mv_bytes(mvk), 128);
    a.off_tip = (int)off;
    off = align_up(off + (size_t)3 * R * N * mv_bytes(ipk), 128);
    a.off_sc = (int)off;
    off = align_up(off + (size_t)R * 8 * 16, 128);
    a.off_fl = (int)off;
    off = align_up(off + (size_t)R * 4 * 4, 128);
    if ((long)off + 1024 <= limit) {
      a.G = G;
      a.ldA = ldA;
      a.smem_bytes = (int)off;
      return true;
    }
    if (R == 1) break;
  }
  return false;
}

static bool plan_cg(int N, int L, int bj, int mvk, int ipk, CgArgs& a, int& smem) {
  const int limit = std::min(max_smem_optin(), 110 * 1024);  // aim for >= 2 CTAs / SM
  int R = std::max(1, 256 / N);
  for (; R >= 1; R = (R > 1 ? R / 2 : 0)) {
    const int ldA = N + 1;
    size_t off = 0;
    off = align_up(off + (size_t)R * N * ldA * mv_bytes(mvk), 128);
    a.off_minv = (int)off;
    off = align_up(off + (bj ? (size_t)R * N * L * 16 : 0), 128);
    a.off_vec = (int)off;
    off = align_up(off + (size_t)8 * R * N * 16, 128);
    a.off_pmv = (int)off;
    off = align_up(off + (size_t)R * N * mv_bytes(mvk), 128);
    a.off_tip = (int)off;
    off = align_up(off + (size_t)3 * R * N * mv_bytes(ipk), 128);
    a.off_sc = (int)off;
    off = align_up(off + (size_t)R * 8 * 16, 128);
    a.off_fl = (int)off;
    off = align_up(off + (size_t)R * 4 * 4, 128);
    if ((long)off <= limit || R == 1) {
      if ((long)off > max_smem_optin()) return false;
      a.R = R;
      a.ldA = ldA;
      smem = (int)off;
      return true;
    }
  }
  return false;
}

template <int WK, int MVK, int IPK>
static int launch_detect_t(const DetectArgs& a, int threads, cudaStream_t st) {
  auto k = fpm_detect_kernel<WK, MVK, IPK>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes) != cudaSuccess)
    return FPM_ECUDA;
  const long grid = (a.T + a.G.R - 1) / a.G.R;
  k<<<(unsigned)grid, threads, a.smem_bytes, st>>>(a);
  g_launches++;
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}

static int launch_detect(const Kinds& k, const DetectArgs& a, int threads, cudaStream_t st) {
  if (k.w == FK_GEN) return launch_detect_t<FK_GEN, FK_GEN, FK_GEN>(a, threads, st);
  switch (k.mv) {
    case FK_F64: return launch_detect_t<FK_F64, FK_F64, FK_F64>(a, threads, st);
    case FK_F32: return launch_detect_t<FK_F64, FK_F32, FK_F32>(a, threads, st);
    case FK_F16: return launch_detect_t<FK_F64, FK_F16, FK_F16>(a, threads, st);
    case FK_BF16: return launch_detect_t<FK_F64, FK_BF16, FK_BF16>(a, threads, st);
    default: return launch_detect_t<FK_F64, FK_GEN, FK_GEN>(a, threads, st);
  }
}

template <int WK, int MVK, int IPK>
static int launch_cg_t(const CgArgs& a, int smem, cudaStream_t st) {
  auto k = fpm_cg_kernel<WK, MVK, IPK>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return FPM_ECUDA;
  const long grid = (a.T + a.R - 1) / a.R;
  k<<<(unsigned)grid, 256, smem, st>>>(a);
  g_launches++;
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}

static int launch_cg(const Kinds& k, const CgArgs& a, int smem, cudaStream_t st) {
  if (k.w == FK_GEN) return launch_cg_t<FK_GEN, FK_GEN, FK_GEN>(a, smem, st);
  switch (k.mv) {
    case FK_F64: return launch_cg_t<FK_F64, FK_F64, FK_F64>(a, smem, st);
    case FK_F32: return launch_cg_t<FK_F64, FK_F32, FK_F32>(a, smem, st);
    case FK_F16: return launch_cg_t<FK_F64, FK_F16, FK_F16>(a, smem, st);
    case FK_BF16: return launch_cg_t<FK_F64, FK_BF16, FK_BF16>(a, smem, st);
    default: return launch_cg_t<FK_F64, FK_GEN, FK_GEN>(a, smem, st);
  }
}

static int check_prec(const fpm_precision* p) {
  if (!p) return FPM_EINVAL;
  if (!valid_format(p->work) || !valid_format(p->matvec) || !valid_format(p->inner)) return FPM_EINVAL;
  // solvers.py:68-74
  if (unit_roundoff(p->work) > unit_roundoff(p->matvec) || unit_roundoff(p->work) > unit_roundoff(p->inner))
    return FPM_EINVAL;
  return FPM_OK;
}

}  // namespace fpm

using namespace fpm;

extern "C" {

int fpm_version(void) { return 10000; /* 1.0.0 */ }

const char* fpm_strerror(int code) {
  switch (code) {
    case FPM_OK: return "ok";
    case FPM_EINVAL: return "invalid argument (contract violation)";
    case FPM_ENOTPD: return "non-PD diagonal block";
    case FPM_ECUDA: return "CUDA runtime error";
    case FPM_EUNSUPPORTED: return "configuration outside this build's limits";
    default: return "unknown error";
  }
}

int fpm_limits(int32_t* max_n, int32_t* max_l, int32_t* max_m) {
  if (max_n) *max_n = kMaxN;
  if (max_l) *max_l = kMaxL;
  if (max_m) *max_m = kMaxM;
  return FPM_OK;
}

int64_t fpm_launch_count(void) { return (int64_t)g_launches.load(); }

int fpm_debug_set_trace(int64_t* dev_buf) {
  g_trace = reinterpret_cast<long long*>(dev_buf);
  return FPM_OK;
}

int fpm_probe_fp64(int64_t iters, double* dp_ops_per_s) {
  if (iters < 1 || !dp_ops_per_s) return FPM_EINVAL;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  if (cudaMalloc(&d, sizeof(double)) != cudaSuccess) return FPM_ECUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int tpb = 512, blocks = sms * 4;
  fpm_dp_probe_kernel<<<blocks, tpb>>>(d, iters / 10 + 1);  // warm-up
  cudaEventRecord(e0);
  fpm_dp_probe_kernel<<<blocks, tpb>>>(d, iters);
  cudaEventRecord(e1);
  g_launches += 2;
  int rc = cudaEventSynchronize(e1) == cudaSuccess ? FPM_OK : FPM_ECUDA;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *dp_ops_per_s = (double)blocks * tpb * (double)iters * 16.0 / (ms * 1e-3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return rc;
}

int fpm_gram(const double* H, const double* y, int64_t T, int32_t M, int32_t N, double sigma2, double* A,
             double* b, void* stream) {
  if (T < 0 || M < 1 || N < 1 || !H || !y || !A || !b) return FPM_EINVAL;
  if (N > kMaxN || M > kMaxM) return FPM_EUNSUPPORTED;
  if (T == 0) return FPM_OK;
  GramArgs a;
  a.H = reinterpret_cast<const double2*>(H);
  a.y = reinterpret_cast<const double2*>(y);
  a.T = T;
  a.sigma2 = sigma2;
  a.A = reinterpret_cast<double2*>(A);
  a.b = reinterpret_cast<double2*>(b);
  const int Np = (N + 7) / 8 * 8;
  int R = std::max(1, 256 / Np);
  int threads = 0;
  size_t smem = 0;
  for (; R >= 1; R = R > 1 ? R / 2 : 0) {
    gram_geom(R, M, N, a.G);
    threads = gram_threads(a.G);
    a.off_ys = 128;
    a.off_union = (int)align_up(128 + (size_t)R * M * 16, 128);
    smem = a.off_union + (size_t)a.G.S * R * a.G.MC * a.G.Np * 16;
    if (threads <= 512 && (long)smem <= max_smem_optin()) break;
    if (R == 1) return FPM_EUNSUPPORTED;
  }
  if (cudaFuncSetAttribute(fpm_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return FPM_ECUDA;
  const long grid = (T + R - 1) / R;
  fpm_gram_kernel<<<(unsigned)grid, threads, smem, (cudaStream_t)stream>>>(a);
  g_launches++;
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}

int fpm_bj_setup(const double* A, int64_t T, int32_t N, int32_t L, int32_t allow_ragged, double* Minv,
                 int32_t* bad_block, void* stream) {
  if (T < 0 || N < 1 || L < 1 || L > N || !A || !Minv) return FPM_EINVAL;
  if (N % L && !allow_ragged) return FPM_EINVAL;  // solvers.py:240-241
  if (N > kMaxN || L > kMaxL) return FPM_EUNSUPPORTED;
  if (T == 0) return FPM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned int* d_nonpd = nullptr;
  if (cudaMallocAsync(&d_nonpd, sizeof(unsigned int), st) != cudaSuccess) return FPM_ECUDA;
  cudaMemsetAsync(d_nonpd, 0, sizeof(unsigned int), st);
  if (bad_block) {
    // fill with INT_MAX via memset pattern 0x7f
    cudaMemsetAsync(bad_block, 0x7f, sizeof(int32_t) * T, st);
  }
  const int nblk = (N + L - 1) / L;
  const int per = 2 * L * L * 16;
  int tpb = std::max(1, std::min(128, (48 * 1024) / per));
  const long work = T * nblk;
  const long grid = (work + tpb - 1) / tpb;
  fpm_bj_kernel<<<(unsigned)grid, tpb, (size_t)tpb * per, st>>>(reinterpret_cast<const double2*>(A), T, N, L,
                                                              reinterpret_cast<double2*>(Minv), bad_block,
                                                              d_nonpd);
  g_launches++;
  if (bad_block) {
    fpm_bad_fix_kernel<<<(unsigned)((T + 255) / 256), 256, 0, st>>>(bad_block, T);
    g_launches++;
  }
  unsigned int h_nonpd = 0;
  cudaMemcpyAsync(&h_nonpd, d_nonpd, sizeof(unsigned int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_nonpd, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return FPM_ECUDA;
  if (cudaGetLastError() != cudaSuccess) return FPM_ECUDA;
  return h_nonpd ? FPM_ENOTPD : FPM_OK;
}

int fpm_cg(const double* A, const double* b, const double* Minv, int64_t T, int32_t N, int32_t L, int32_t iters,
           const fpm_precision* prec, int32_t rho_update, double* x, int32_t* breakdown_at,
           int32_t* diverged_at, void* stream) {
  if (T < 0 || N < 1 || !A || !b || !x || !breakdown_at || !diverged_at) return FPM_EINVAL;
  if (iters < 1) return FPM_EINVAL;                                                   // solvers.py:282-283
  if (rho_update != FPM_RHO_AS_WRITTEN && rho_update != FPM_RHO_TEXTBOOK) return FPM_EINVAL;  // :280-281
  int rc = check_prec(prec);
  if (rc) return rc;
  const int bj = Minv != nullptr;
  if (bj && (L < 1 || L > N)) return FPM_EINVAL;
  if (N > kMaxN || (bj && L > kMaxL)) return FPM_EUNSUPPORTED;
  if (T == 0) return FPM_OK;
  Kinds k = pick_kinds(*prec);
  CgArgs a;
  std::memset(&a, 0, sizeof(a));
  a.A = reinterpret_cast<const double2*>(A);
  a.b = reinterpret_cast<const double2*>(b);
  a.minv = reinterpret_cast<const double2*>(Minv);
  a.T = T;
  a.N = N;
  a.L = bj ? L : 1;
  a.iters = iters;
  a.bj = bj;
  a.textbook = rho_update == FPM_RHO_TEXTBOOK;
  a.pr.work = make_fmtp(prec->work);
  a.pr.mv = make_fmtp(prec->matvec);
  a.pr.ip = make_fmtp(prec->inner);
  a.x = reinterpret_cast<double2*>(x);
  a.brk = breakdown_at;
  a.div = diverged_at;
  int smem = 0;
  if (!plan_cg(N, a.L, bj, k.mv, k.ip, a, smem)) return FPM_EUNSUPPORTED;
  return launch_cg(k, a, smem, (cudaStream_t)stream);
}

int fpm_slice_count(const double* x, const uint8_t* tx_bits, int64_t T, int32_t N, int32_t qam,
                    uint8_t* rx_bits, int64_t* counters, void* stream) {
  if (T < 0 || N < 1 || !x || !counters || (qam != 16 && qam != 64)) return FPM_EINVAL;
  if (T == 0) return FPM_OK;
  const long TN = T * (long)N;
  const int tpb = 256;
  long grid = std::min((TN + tpb - 1) / tpb, 148L * 8);
  fpm_slice_kernel<<<(unsigned)grid, tpb, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const double2*>(x), tx_bits, TN, rx_bits,
      reinterpret_cast<unsigned long long*>(counters), make_slicer(qam));
  g_launches++;
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}

static int detect_args(const double* H, const double* y, const uint8_t* tx_bits, int64_t T, int32_t M, int32_t N,
                       double sigma2, int32_t algorithm, int32_t L, int32_t iters, const fpm_precision* prec,
                       int32_t rho_update, int32_t qam, const double* Minv_in, double* x, int32_t* brk,
                       int32_t* div, uint8_t* rx, int64_t* counters, DetectArgs& a, Kinds& k, int& threads) {
  if (T < 0 || M < 1 || N < 1) return FPM_EINVAL;
  if (iters < 1) return FPM_EINVAL;
  if (rho_update != FPM_RHO_AS_WRITTEN && rho_update != FPM_RHO_TEXTBOOK) return FPM_EINVAL;
  if (qam != 16 && qam != 64) return FPM_EINVAL;
  if (algorithm != FPM_ALG_CG && algorithm != FPM_ALG_FP_CG && algorithm != FPM_ALG_FP_BJ_CG) return FPM_EINVAL;
  fpm_precision p64 = {{53, 11, 1}, {53, 11, 1}, {53, 11, 1}};
  const fpm_precision* pp = algorithm == FPM_ALG_CG ? &p64 : prec;  // detect.py:131-133
  int rc = check_prec(pp);
  if (rc) return rc;
  const int bj = algorithm == FPM_ALG_FP_BJ_CG;
  if (bj && (L < 1 || L > N || N % L)) return FPM_EINVAL;  // build_blocks_batch default: no ragged blocks
  if (N > kMaxN || M > kMaxM || (bj && L > kMaxL)) return FPM_EUNSUPPORTED;
  std::memset(&a, 0, sizeof(a));
  a.H = reinterpret_cast<const double2*>(H);
  a.y = reinterpret_cast<const double2*>(y);
  a.tx = tx_bits;
  a.T = T;
  a.sigma2 = sigma2;
  a.L = bj ? L : 1;
  a.iters = iters;
  a.bj = bj;
  a.textbook = rho_update == FPM_RHO_TEXTBOOK;
  a.pr.work = make_fmtp(pp->work);
  a.pr.mv = make_fmtp(pp->matvec);
  a.pr.ip = make_fmtp(pp->inner);
  a.minv_in = bj ? reinterpret_cast<const double2*>(Minv_in) : nullptr;
  a.x = reinterpret_cast<double2*>(x);
  a.brk = brk;
  a.div = div;
  a.rx = rx;
  a.counters = reinterpret_cast<unsigned long long*>(counters);
  a.sl = make_slicer(qam);
  a.trace = g_trace;
  k = pick_kinds(*pp);
  if (!plan_detect(M, N, a.L, bj, k.mv, k.ip, a, threads)) return FPM_EUNSUPPORTED;
  return FPM_OK;
}

int fpm_detect(const double* H, const double* y, const uint8_t* tx_bits, int64_t T, int32_t M, int32_t N,
               double sigma2, int32_t algorithm, int32_t L, int32_t iters, const fpm_precision* prec,
               int32_t rho_update, int32_t qam, const double* Minv_in, double* x, int32_t* breakdown_at,
               int32_t* diverged_at, uint8_t* rx_bits, int64_t* counters, void* stream) {
  if (!H || !y || !x || !breakdown_at || !diverged_at || !counters) return FPM_EINVAL;
  DetectArgs a;
  Kinds k;
  int threads = 0;
  int rc = detect_args(H, y, tx_bits, T, M, N, sigma2, algorithm, L, iters, prec, rho_update, qam, Minv_in, x,
                       breakdown_at, diverged_at, rx_bits, counters, a, k, threads);
  if (rc) return rc;
  if (T == 0) return FPM_OK;
  return launch_detect(k, a, threads, (cudaStream_t)stream);
}

int fpm_detect_host(const double* H, const double* y, const uint8_t* tx_bits, int64_t T, int32_t M, int32_t N,
                    double sigma2, int32_t algorithm, int32_t L, int32_t iters, const fpm_precision* prec,
                    int32_t rho_update, int32_t qam, const double* Minv_in, double* x, int32_t* breakdown_at,
                    int32_t* diverged_at, uint8_t* rx_bits, int64_t* counters, int64_t chunk) {
  if (!H || !y || !x || !breakdown_at || !diverged_at || !counters) return FPM_EINVAL;
  DetectArgs a;
  Kinds k;
  int threads = 0;
  int rc = detect_args(H, y, tx_bits, T, M, N, sigma2, algorithm, L, iters, prec, rho_update, qam, Minv_in, x,
                       breakdown_at, diverged_at, rx_bits, counters, a, k, threads);
  if (rc) return rc;
  if (T == 0) return FPM_OK;
  const int bps = qam == 64 ? 6 : 4;
  const int bj = algorithm == FPM_ALG_FP_BJ_CG;
  if (chunk <= 0) chunk = std::max<int64_t>(a.G.R, (int64_t)(512LL << 20) / ((int64_t)M * N * 16));
  chunk = std::max<int64_t>(1, std::min<int64_t>(chunk, T));
  const size_t hB = (size_t)chunk * M * N * 16, yB = (size_t)chunk * M * 16, tB = (size_t)chunk * bps * N;
  const size_t xB = (size_t)chunk * N * 16, fB = (size_t)chunk * 4, mB = (size_t)chunk * N * L * 16;
  cudaStream_t st[2];
  unsigned char* buf[2] = {nullptr, nullptr};
  int64_t* dcnt = nullptr;
  const size_t per = align_up(hB, 256) + align_up(yB, 256) + align_up(tB, 256) + align_up(tB, 256) +
                     align_up(xB, 256) + 2 * align_up(fB, 256) + (bj && Minv_in ? align_up(mB, 256) : 0);
  rc = FPM_OK;
  for (int s = 0; s < 2; ++s) {
    if (cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking) != cudaSuccess) return FPM_ECUDA;
    if (cudaMalloc(&buf[s], per) != cudaSuccess) rc = FPM_ECUDA;
  }
  if (!rc && cudaMalloc(&dcnt, 2 * FPM_NCOUNTERS * sizeof(int64_t)) != cudaSuccess) rc = FPM_ECUDA;
  if (!rc) cudaMemset(dcnt, 0, 2 * FPM_NCOUNTERS * sizeof(int64_t));
  for (int64_t c0 = 0, it = 0; !rc && c0 < T; c0 += chunk, ++it) {
    const int s = (int)(it & 1);
    const int64_t n = std::min<int64_t>(chunk, T - c0);
    unsigned char* p = buf[s];
    double* dH = (double*)p;
    p += align_up(hB, 256);
    double* dy = (double*)p;
    p += align_up(yB, 256);
    uint8_t* dtx = (uint8_t*)p;
    p += align_up(tB, 256);
    uint8_t* drx = (uint8_t*)p;
    p += align_up(tB, 256);
    double* dx = (double*)p;
    p += align_up(xB, 256);
    int32_t* dbk = (int32_t*)p;
    p += align_up(fB, 256);
    int32_t* ddv = (int32_t*)p;
    p += align_up(fB, 256);
    double* dm = (bj && Minv_in) ? (double*)p : nullptr;
    cudaMemcpyAsync(dH, H + c0 * (int64_t)M * N * 2, (size_t)n * M * N * 16, cudaMemcpyHostToDevice, st[s]);
    cudaMemcpyAsync(dy, y + c0 * (int64_t)M * 2, (size_t)n * M * 16, cudaMemcpyHostToDevice, st[s]);
    if (tx_bits)
      cudaMemcpyAsync(dtx, tx_bits + c0 * bps * N, (size_t)n * bps * N, cudaMemcpyHostToDevice, st[s]);
    if (dm) cudaMemcpyAsync(dm, Minv_in + c0 * (int64_t)N * L * 2, (size_t)n * N * L * 16, cudaMemcpyHostToDevice, st[s]);
    DetectArgs b = a;
    b.H = (const double2*)dH;
    b.y = (const double2*)dy;
    b.tx = tx_bits ? dtx : nullptr;
    b.T = n;
    b.minv_in = (const double2*)dm;
    b.x = (double2*)dx;
    b.brk = dbk;
    b.div = ddv;
    b.rx = rx_bits ? drx : nullptr;
    b.counters = reinterpret_cast<unsigned long long*>(dcnt + s * FPM_NCOUNTERS);
    rc = launch_detect(k, b, threads, st[s]);
    if (rc) break;
    cudaMemcpyAsync(x + c0 * (int64_t)N * 2, dx, (size_t)n * N * 16, cudaMemcpyDeviceToHost, st[s]);
    cudaMemcpyAsync(breakdown_at + c0, dbk, (size_t)n * 4, cudaMemcpyDeviceToHost, st[s]);
    cudaMemcpyAsync(diverged_at + c0, ddv, (size_t)n * 4, cudaMemcpyDeviceToHost, st[s]);
    if (rx_bits) cudaMemcpyAsync(rx_bits + c0 * bps * N, drx, (size_t)n * bps * N, cudaMemcpyDeviceToHost, st[s]);
  }
  int64_t hc[2 * FPM_NCOUNTERS] = {0};
  if (!rc) {
    for (int s = 0; s < 2; ++s)
      if (cudaStreamSynchronize(st[s]) != cudaSuccess) rc = FPM_ECUDA;
    if (!rc && cudaMemcpy(hc, dcnt, sizeof(hc), cudaMemcpyDeviceToHost) != cudaSuccess) rc = FPM_ECUDA;
    if (!rc)
      for (int i = 0; i < FPM_NCOUNTERS; ++i) counters[i] += hc[i] + hc[FPM_NCOUNTERS + i];
  }
  for (int s = 0; s < 2; ++s) {
    cudaStreamSynchronize(st[s]);
    if (buf[s]) cudaFree(buf[s]);
    cudaStreamDestroy(st[s]);
  }
  if (dcnt) cudaFree(dcnt);
  if (!rc && cudaGetLastError() != cudaSuccess) rc = FPM_ECUDA;
  return rc;
}

}  // extern "C"
