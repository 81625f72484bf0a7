// Fused detector kernel and standalone CG kernel templates.
//
//   fpm_detect_kernel<WK, K, NB, LB>: per CTA, R realizations:
//     Gram/MF (TMA-streamed H, bit-exact fp64) -> A in shared memory at u_MV
//     -> block-Jacobi inverses (fp64, on-chip or injected) -> (BJ-)CG in
//     shared memory -> QAM slicing + error counters -> x_hat, flags out.
//   A never touches HBM: per realization the kernel reads H and y once and
//   writes x_hat (+ optional bits).
//   fpm_cg_kernel<WK, K, LB>: the same CG from a caller-provided A, b, Minv
//   (run_batch boundary).
// WK: work kind (F64 or GEN); K: matvec/inner kind; NB: nb = N/4 fixed at
// compile time (0 = runtime); LB: block size fixed at compile time (0 =
// runtime or none).  Instantiated per kind in fpm_inst_<kind>.cu.
#pragma once
#include <cuda_runtime.h>

#include "../../include/fpmimo_b200.h"
#include "fpm_bj.cuh"
#include "fpm_cg.cuh"
#include "fpm_common.cuh"
#include "fpm_gram.cuh"
#include "fpm_ptx.cuh"

namespace fpm {

// Level index = #thresholds strictly below v (digitize right=True; NaN -> 0,
// detect.py:70-75), then the per-axis Gray label (detect.py:50).
__device__ __forceinline__ int level_index(double v, const Slicer& sl) {
  int idx = 0;
#pragma unroll
  for (int k = 0; k < 7; ++k)
    if (k < sl.nth && v > sl.th[k]) ++idx;
  return idx;
}

// Slices x and compares with tx; returns bit errors, sets *sym_err.
__device__ __forceinline__ int slice_one(double2 x, const uint8_t* tx, uint8_t* rx, const Slicer& sl,
                                         int* sym_err) {
  int gi = level_index(x.x, sl), gq = level_index(x.y, sl);
  gi ^= gi >> 1;
  gq ^= gq >> 1;
  int errs = 0;
#pragma unroll 1
  for (int k = 0; k < sl.bpa; ++k) {
    const uint8_t bi = (uint8_t)((gi >> (sl.bpa - 1 - k)) & 1);
    const uint8_t bq = (uint8_t)((gq >> (sl.bpa - 1 - k)) & 1);
    if (rx) {
      rx[k] = bi;
      rx[sl.bpa + k] = bq;
    }
    if (tx) errs += (tx[k] != bi) + (tx[sl.bpa + k] != bq);
  }
  *sym_err = errs > 0;
  return errs;
}

// Gram epilogue into shared memory: A at u_MV (transposed), b, and the fp64
// diagonal blocks (interleaved, for the block-Jacobi setup) when needed.
template <int K, int NB, int LB>
struct EmitSmem {
  CgSmem<K>* S;
  const FmtP* fm;
  int bj;        // build block inverses on chip
  double2* scr;  // diagonal blocks, entry e of block gb at scr[e*nbt + gb]
  int nblk, nbt;
  double sigma2;
  __device__ __forceinline__ void job(const GramJob& jb, const double2 (&acc)[16], int nb) {
    const int N = NB > 0 ? 4 * NB : S->N;
    const int ldA = NB > 0 ? lda_for(4 * NB, (int)sizeof(typename Ar<K>::C)) : S->ldA;
    const int L = LB > 0 ? LB : S->L;
    const int g = jb.g;
    typename Ar<K>::C* At = S->At + g * N * ldA;
    double2* sg = scr + g * nblk;
    const int nbt_ = nbt;
    const bool onchip = bj;
    const FmtP& f = *fm;
    gram_entries(
        jb, acc, nb, N, sigma2,
        [&](int i, int j, double2 vij, double2 vji) {
          At[i * ldA + j] = Ar<K>::rnd(vij, f);
          At[j * ldA + i] = Ar<K>::rnd(vji, f);
          if (onchip) {
            const int kb = i / L;
            if (kb == j / L) {
              const int il = i - kb * L, jl = j - kb * L;
              sg[(il * L + jl) * nbt_ + kb] = vij;
              sg[(jl * L + il) * nbt_ + kb] = vji;
            }
          }
        },
        [&](int i, double2 vii) {
          At[i * ldA + i] = Ar<K>::rnd(vii, f);
          if (onchip) {
            const int kb = i / L, il = i - kb * L;
            sg[(il * L + il) * nbt_ + kb] = vii;
          }
        });
  }
  __device__ __forceinline__ void b(int g, int n, int part, double v) {
    double* bp = reinterpret_cast<double*>(S->b + g * S->N + n);
    bp[part] = v;
  }
};

template <int WK, int K, int NB, int LB>
__global__ void __launch_bounds__(512, 1) fpm_detect_kernel(const DetectArgs args) {
  extern __shared__ __align__(128) unsigned char smem[];
  typedef typename Ar<K>::C C;
  typedef typename Ar<K>::P P;
  const int tid = threadIdx.x, nthreads = blockDim.x;
  const GramGeom& G = args.G;
  const long t0 = (long)blockIdx.x * G.R;
  const int Rv = (int)min((long)G.R, args.T - t0);
  const int N = NB > 0 ? 4 * NB : G.N;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);  // S full, S empty, 1 y
  __shared__ unsigned long long cnt[FPM_NCOUNTERS];
  CgSmem<K> S;
  S.R = G.R;
  S.N = N;
  S.L = args.bj ? (LB > 0 ? LB : args.L) : 1;
  S.ldA = NB > 0 ? lda_for(N, (int)sizeof(typename Ar<K>::C)) : args.ldA;
  S.At = reinterpret_cast<C*>(smem + args.off_union);
  S.minv = reinterpret_cast<double2*>(smem + args.off_minv);
  double2* vec = reinterpret_cast<double2*>(smem + args.off_vec);
  const int RN = G.R * N;
  S.b = vec;
  S.x = vec + RN;
  S.r = vec + 2 * RN;
  S.p = vec + 3 * RN;
  S.z = vec + 4 * RN;
  S.w = vec + 5 * RN;
  S.xn = vec + 6 * RN;
  S.rn = vec + 7 * RN;
  S.pmv = reinterpret_cast<P*>(smem + args.off_pmv);
  S.tphi = reinterpret_cast<C*>(smem + args.off_tip);
  S.trho = S.tphi + RN;
  S.tr1 = S.trho + RN;
  S.rip = S.tr1 + RN;
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
#pragma unroll 1
  for (int g = tid; g < G.R; g += nthreads) S.fl[g * 4] = g < Rv ? 1 : 0;
  long long* tr = (diag_trace(args.trace) && blockIdx.x == 0) ? diag_trace(args.trace) : nullptr;
  FPM_STAMP(tr, 0);
  __syncthreads();

  // 1) Gram + matched filter straight into shared memory
  const int L = S.L;
  const int nblk = args.bj ? (N + L - 1) / L : 1;
  EmitSmem<K, NB, LB> em;
  em.S = &S;
  em.fm = &args.pr.mv;
  em.bj = args.bj && !args.minv_in;
  em.scr = reinterpret_cast<double2*>(smem + args.off_scr);
  em.nblk = nblk;
  em.nbt = G.R * nblk;
  em.sigma2 = args.sigma2;
  gram_run<NB>(args.H, args.y, t0, Rv, G, reinterpret_cast<double2*>(smem + args.off_union),
               reinterpret_cast<double2*>(smem + args.off_ys), bars, nthreads, tid, em, tr ? tr + 16 : nullptr);
  FPM_STAMP(tr, 1);

  // 2) block-Jacobi inverses (on-chip fp64 Cholesky, or injected)
  if (args.bj) {
    if (args.minv_in) {  // row-major blocks in global -> column-major in shared
#pragma unroll 1
      for (int q = tid; q < Rv * N * L; q += nthreads) {
        const int g = q / (N * L);
        const int e = q - g * N * L;
        const int kb = e / (L * L), o = e - kb * L * L;
        const int Lk = min(L, N - kb * L);
        if (o >= Lk * Lk) continue;
        const int i = o / Lk, j = o - i * Lk;
        S.minv[g * N * L + kb * L * L + j * Lk + i] = Ar<WK>::rnd(args.minv_in[(t0 + g) * (long)N * L + e], args.pr.work);
      }
    } else {
      double2* scr = reinterpret_cast<double2*>(smem + args.off_scr);
      double2* scr2 = reinterpret_cast<double2*>(smem + args.off_scr2);
      const int nbt = em.nbt;
#pragma unroll 1
      for (int q = tid; q < Rv * nblk; q += nthreads) {
        const int g = q / nblk, kb = q - g * nblk;
        const int Lk = min(L, N - kb * L);
        double2* out = S.minv + g * N * L + kb * L * L;
        const bool ok = (LB > 0) ? hpd_inverse<LB>(scr + q, nbt, scr2 + q, nbt, out, Lk)
                                 : hpd_inverse<0>(scr + q, nbt, scr2 + q, nbt, out, Lk);
        if (!ok) {
          atomicExch(&S.fl[g * 4], 0);
          atomicAdd(&cnt[FPM_CNT_NONPD], 1ULL);
        } else if (WK != FK_F64) {
          for (int e = 0; e < Lk * Lk; ++e) out[e] = Ar<WK>::rnd(out[e], args.pr.work);
        }
      }
    }
    __syncthreads();
  }
  FPM_STAMP(tr, 2);

  // 3) CG in shared memory
  {
    CtaBar bar;
    cg_group<WK, K, LB, (NB > 0 ? 4 * NB : 0)>(S, Rv, args.iters, args.bj != 0, args.textbook != 0, args.pr, nthreads, tid, bar,
                        tr ? tr + 3 : nullptr);
  }
  FPM_STAMP(tr, 10);

  // 4) slicer + counters + write-back
  const int bps = 2 * args.sl.bpa;
  unsigned long long be = 0, se = 0;
#pragma unroll 1
  for (int q = tid; q < Rv * N; q += nthreads) {
    const long gq = t0 * N + q;
    const double2 xv = S.x[q];
    args.x[gq] = xv;
    int sym;
    be += slice_one(xv, args.tx ? args.tx + gq * bps : nullptr, args.rx ? args.rx + gq * bps : nullptr,
                    args.sl, &sym);
    se += sym;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    be += __shfl_xor_sync(0xffffffffu, be, off);
    se += __shfl_xor_sync(0xffffffffu, se, off);
  }
  if ((tid & 31) == 0) {
    if (be) atomicAdd(&cnt[FPM_CNT_BIT_ERRORS], be);
    if (se) atomicAdd(&cnt[FPM_CNT_SYMBOL_ERRORS], se);
  }
#pragma unroll 1
  for (int g = tid; g < Rv; g += nthreads) {
    const int bk = S.fl[g * 4 + 2], dv = S.fl[g * 4 + 3];
    args.brk[t0 + g] = bk;
    args.div[t0 + g] = dv;
    if (dv >= 0) atomicAdd(&cnt[FPM_CNT_DIVERGED], 1ULL);
    if (bk >= 0) atomicAdd(&cnt[FPM_CNT_BREAKDOWN], 1ULL);
  }
  if (tid == 0) atomicAdd(&cnt[FPM_CNT_TRIALS], (unsigned long long)Rv);
  __syncthreads();
  if (tid < FPM_NCOUNTERS && cnt[tid]) atomicAdd(&args.counters[tid], cnt[tid]);
  FPM_STAMP(tr, 15);
}

#ifndef FPM_CG_LOADS
#define FPM_CG_LOADS 8
#endif

template <int WK, int K, int LB, int NC>
__global__ void __launch_bounds__(256) fpm_cg_kernel(const CgArgs args) {
  extern __shared__ __align__(128) unsigned char smem[];
  typedef typename Ar<K>::C C;
  typedef typename Ar<K>::P P;
  const int tid = threadIdx.x, nthreads = blockDim.x;
  const long t0 = (long)blockIdx.x * args.R;
  const int Rv = (int)min((long)args.R, args.T - t0);
  const int N = NC > 0 ? NC : args.N;
  CgSmem<K> S;
  S.R = args.R;
  S.N = N;
  S.L = args.bj ? args.L : 1;
  S.ldA = args.a_glob ? N : args.ldA;
  S.At = args.a_glob ? const_cast<C*>(reinterpret_cast<const C*>(args.a_glob)) + t0 * (long)N * N
                     : reinterpret_cast<C*>(smem);
  S.minv = reinterpret_cast<double2*>(smem + args.off_minv);
  double2* vec = reinterpret_cast<double2*>(smem + args.off_vec);
  const int RN = args.R * N;
  S.b = vec;
  S.x = vec + RN;
  S.r = vec + 2 * RN;
  S.p = vec + 3 * RN;
  S.z = vec + 4 * RN;
  S.w = vec + 5 * RN;
  S.xn = vec + 6 * RN;
  S.rn = vec + 7 * RN;
  S.pmv = reinterpret_cast<P*>(smem + args.off_pmv);
  S.tphi = reinterpret_cast<C*>(smem + args.off_tip);
  S.trho = S.tphi + RN;
  S.tr1 = S.trho + RN;
  S.rip = S.tr1 + RN;
  S.sc = reinterpret_cast<double2*>(smem + args.off_sc);
  S.fl = reinterpret_cast<int*>(smem + args.off_fl);

  // A (row-major, global) -> At (row-major, pitch ldA, u_MV), coalesced;
  // 8 streaming loads in flight per thread (the copy is HBM-latency bound
  // with one outstanding load per thread)
  const int NN = N * N;
  if (!args.a_glob) {
    constexpr int U = FPM_CG_LOADS;
    const double2* Ag = args.A + t0 * (long)NN;
    const int tot = Rv * NN;
#pragma unroll 1
    for (int q0 = tid; q0 < tot; q0 += nthreads * U) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + u * nthreads;
        if (q < tot) v[u] = __ldcs(Ag + q);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + u * nthreads;
        if (q < tot) {
          const int g = q / NN;
          const int e = q - g * NN;
          const int i = e / N, k = e - i * N;
          S.At[(g * N + i) * S.ldA + k] = Ar<K>::rnd(v[u], args.pr.mv);
        }
      }
    }
  }
#pragma unroll 1
  for (int q = tid; q < Rv * N; q += nthreads) S.b[q] = args.b[t0 * N + q];
  if (args.bj) {  // row-major blocks in global -> column-major in shared
    const int L = args.L;
#pragma unroll 1
    for (int q = tid; q < Rv * N * L; q += nthreads) {
      const int g = q / (N * L);
      const int e = q - g * N * L;
      const int kb = e / (L * L), o = e - kb * L * L;
      const int Lk = min(L, N - kb * L);
      if (o >= Lk * Lk) continue;
      const int i = o / Lk, j = o - i * Lk;
      S.minv[g * N * L + kb * L * L + j * Lk + i] = Ar<WK>::rnd(args.minv[t0 * (long)N * L + q], args.pr.work);
    }
  }
#pragma unroll 1
  for (int g = tid; g < args.R; g += nthreads) S.fl[g * 4] = g < Rv ? 1 : 0;
  CgHist hh = args.h;  // run_batch histories (fpm_cg_ex)
  hh.t0 = t0;
  if (hh.on) S.h = &hh;
  __syncthreads();
  {
    CtaBar bar;
    long long* tr = (diag_trace(args.trace) && blockIdx.x == 0) ? diag_trace(args.trace) : nullptr;
    if (tr && tid == 0) tr[60] = clock64();
    cg_group<WK, K, LB, NC>(S, Rv, args.iters, args.bj != 0, args.textbook != 0, args.pr, nthreads, tid, bar, tr);
  }
#pragma unroll 1
  for (int q = tid; q < Rv * N; q += nthreads) args.x[t0 * N + q] = S.x[q];
#pragma unroll 1
  for (int g = tid; g < Rv; g += nthreads) {
    args.brk[t0 + g] = S.fl[g * 4 + 2];
    args.div[t0 + g] = S.fl[g * 4 + 3];
  }
}

template <int WK, int K, int NB, int LB>
int launch_detect_t(const DetectArgs& a, int threads, cudaStream_t st) {
  auto k = fpm_detect_kernel<WK, K, NB, LB>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes) != cudaSuccess)
    return FPM_ECUDA;
  const long grid = (a.T + a.G.R - 1) / a.G.R;
  k<<<(unsigned)grid, threads, a.smem_bytes, st>>>(a);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}

template <int WK, int K, int LB, int NC>
int launch_cg_nc(const CgArgs& a, int smem, cudaStream_t st) {
  auto k = fpm_cg_kernel<WK, K, LB, NC>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return FPM_ECUDA;
  const long grid = (a.T + a.R - 1) / a.R;
  k<<<(unsigned)grid, a.threads > 0 ? a.threads : 256, smem, st>>>(a);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}

// N = 64 (c2/c3/c5 shapes) gets the compile-time-N (fully unrolled) sums
template <int WK, int K, int LB>
int launch_cg_t(const CgArgs& a, int smem, cudaStream_t st) {
  if (a.N == 64) return launch_cg_nc<WK, K, LB, 64>(a, smem, st);
  return launch_cg_nc<WK, K, LB, 0>(a, smem, st);
}

}  // namespace fpm
