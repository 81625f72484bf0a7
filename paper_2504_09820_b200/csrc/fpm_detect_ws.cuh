// Warp-specialised persistent detector kernel (the fast path).
//
//   threads [0, gt)        "Gram" warps: accumulate the bit-exact Gram/MF of
//                          realization group j+1 from the TMA ring ...
//   threads [gt, gt+32)    producer warp: keeps the H / y TMA ring full
//   threads [gt+32, ...)   ... while the "CG" warps solve group j: block
//                          inverses, (BJ-)CG, slicing, counters, write-back.
//
// The hand-off is a double-buffered shared-memory slot (A at u_MV, b, fp64
// diagonal blocks; a single slot when two do not fit, e.g. fp64 matvec)
// guarded by two mbarrier pairs (slot full / slot empty), so
// the latency-bound CG of one group never stalls the FP64 pipe: the Gram
// warps only wait for a slot when the CG side is more than one group behind.
// The H ring runs continuously across groups (the producer prefetches the
// next group's first chunks and its y vector while the current group ends).
// Each CTA owns groups blockIdx.x, blockIdx.x + gridDim.x, ...  Named
// hardware barriers: 1 = Gram group, 2 = CG group.
#pragma once
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "fpm_detect.cuh"
#include "fpm_detect_sw.cuh"
#include "fpm_gram32.cuh"

namespace fpm {

#ifndef FPM_WIDE_NC_MAX_RS  // unrolled wide sums only when the CG side keeps >= 256 - this registers
#define FPM_WIDE_NC_MAX_RS 0
#endif
#ifndef FPM_G32_UNROLL  // binary32 Gram row loop unroll (two: slower with the clamped prefetch, faster without)
#define FPM_G32_UNROLL 4  // measured with the unclamped prefetch: 1: 0.740, 2: 0.761, 3: 0.770, 4: 0.773 of the packed binary32 ceiling
#endif
#ifndef FPM_CG_SPLIT  // c5 at fp64 matvec: CG group = warp group 3 at its own register budget (kCgOwn below)
#define FPM_CG_SPLIT 0
#endif
#ifndef FPM_CG_SPLIT_GRAM_REGS
#define FPM_CG_SPLIT_GRAM_REGS 176
#endif
#ifndef FPM_PIPE_UNROLL_N  // 0: per instance (kRowUnroll below)
#define FPM_PIPE_UNROLL_N 0
#endif

#ifndef FPM_PRODUCER_LANES  // threads of the producer warp issuing bulk copies (1 or 32)
#define FPM_PRODUCER_LANES 32
#endif
constexpr int kProducerLanes = FPM_PRODUCER_LANES;
#ifndef FPM_PRODUCER_SLEEP_NS  // back-off of the producer / CG-side waits (0: spin)
#define FPM_PRODUCER_SLEEP_NS 300  // measured: evens out the producer warp's SM sub-partition (+0.7 %)
#endif
#ifndef FPM_CG_SLEEP_NS
#define FPM_CG_SLEEP_NS 0
#endif
#ifndef FPM_WAIT_HINT_NS  // > 0: producer / CG-side waits suspend in hardware (try_wait hint) instead of polling
#define FPM_WAIT_HINT_NS 0
#endif
#define FPM_PWAIT(b, p)                                                                                       \
  (FPM_WAIT_HINT_NS ? mbar_wait_suspend((b), (p), FPM_WAIT_HINT_NS)                                          \
   : FPM_PRODUCER_SLEEP_NS ? mbar_wait_sleep((b), (p), FPM_PRODUCER_SLEEP_NS) : mbar_wait((b), (p)))
#ifndef FPM_G32_SLEEP_NS  // converter warp's wait for a landed stage (0: spin)
#define FPM_G32_SLEEP_NS 300
#endif
#define FPM_G32WAIT(b, p) (FPM_G32_SLEEP_NS ? mbar_wait_sleep((b), (p), FPM_G32_SLEEP_NS) : mbar_wait((b), (p)))
#ifndef FPM_GSLOT_SLEEP_NS  // Gram warps' wait for the hand-off slot (0: spin)
#define FPM_GSLOT_SLEEP_NS 0
#endif
#define FPM_GSWAIT(b, p) (FPM_GSLOT_SLEEP_NS ? mbar_wait_sleep((b), (p), FPM_GSLOT_SLEEP_NS) : mbar_wait((b), (p)))
#ifndef FPM_SW_WG3_REGS  // SW: registers of the producer's warp group
#define FPM_SW_WG3_REGS 24
#endif
#ifndef FPM_G32_ROW_CLAMP  // binary32 Gram row loop: clamp the prefetched row index (1) or read one row past (0)
#define FPM_G32_ROW_CLAMP 0  // measured c4 FP32 Gram: 0.716 -> 0.740, with the loop unrolled by two 0.760
#endif
#ifndef FPM_ROW_CLAMP  // -1: per instance (kRowClamp below); 0 / 1: force
#define FPM_ROW_CLAMP -1
#endif
#ifndef FPM_GFULL_SLEEP_NS  // Gram warps' wait for a landed stage (0: spin)
#define FPM_GFULL_SLEEP_NS 0
#endif
#define FPM_GFWAIT(b, p) (FPM_GFULL_SLEEP_NS ? mbar_wait_sleep((b), (p), FPM_GFULL_SLEEP_NS) : mbar_wait((b), (p)))
#define FPM_CWAIT(b, p)                                                                                       \
  (FPM_WAIT_HINT_NS ? mbar_wait_suspend((b), (p), FPM_WAIT_HINT_NS)                                          \
   : FPM_CG_SLEEP_NS ? mbar_wait_sleep((b), (p), FPM_CG_SLEEP_NS) : mbar_wait((b), (p)))

struct WsLayout {  // byte offsets inside one hand-off slot
  int at, b, d, bytes;
};

// role order (planner's choice, FPM_WS_ORDER knob overrides: 0 = Gram warps first, 1 = CG first)
inline int env_order(int planned) {
  const char* v = knob("FPM_WS_ORDER");
  return v ? (std::atoi(v) != 0) : planned;
}

// double2 elements of one stage: R x MC x Np of H, then R x MC of y padded
// to whole 128-byte units (every stage and its y block start 128-byte
// aligned: tensor-map TMA destinations)
__host__ __device__ __forceinline__ int ws_stage_elems(const GramGeom& G) {
  return G.R * G.MC * G.Np + (G.R * G.MC + 7) / 8 * 8;
}

// Stage c of a group: antenna rows m0 .. m0+rows of H for every realization
// of the group (one bulk copy each, rows contiguous in global memory) and the
// same rows of y (one bulk copy each), behind the R x MC x Np H block; the
// whole warp issues, lane 0 posts the stage's bytes first.
__device__ __forceinline__ void ws_issue(const double2* H, const double2* y, long t0, int Rv, const GramGeom& G,
                                         int chunk, double2* stage_buf, uint64_t* bar, int lane, int nlanes) {
  const int m0 = chunk * G.MC;
  const int rows = min(G.MC, G.M - m0);
  const uint32_t rowb = (uint32_t)G.N * 16u;
  if (lane == 0) mbar_expect_tx(bar, (uint32_t)Rv * (uint32_t)rows * (rowb + 16u));
  if (nlanes > 1) __syncwarp();
  double2* ybuf = stage_buf + (long)G.R * G.MC * G.Np;
  for (int g = lane; g < Rv; g += nlanes) {
    const double2* src = H + ((t0 + g) * (long)G.M + m0) * (long)G.N;
    double2* dst = stage_buf + (long)g * G.MC * G.Np;
    if (G.N == G.Np) {
      bulk_g2s(dst, src, rows * rowb, bar);
    } else {
      for (int r = 0; r < rows; ++r) bulk_g2s(dst + r * G.Np, src + (long)r * G.N, rowb, bar);
    }
    bulk_g2s(ybuf + g * G.MC, y + (t0 + g) * (long)G.M + m0, (uint32_t)rows * 16u, bar);
  }
}

// extra matched-filter chains of a Gram thread (kCPT > 1): operands of row
// mm loaded before the row's tile products, added after them (exact split
// re / im chains: re += fl(fl(hr yr) + fl(hi yi)), im += fl(fl(hr yi) + fl(hi (-yr))))
template <int X>
__device__ __forceinline__ void xchain_load(const double2* sb, const double2* ys, int m0, int mm, int Np,
                                            const int (&hoff)[X], const int (&yoff)[X], double2 (&h)[X],
                                            double2 (&y)[X]) {
#pragma unroll
  for (int k = 0; k < X; ++k) {
    h[k] = sb[hoff[k] + mm * Np];
    y[k] = ys[yoff[k] + m0 + mm];  // ys: the stage's y block (m0 = 0)
  }
}
template <int X>
__device__ __forceinline__ void xchain_add(double (&c)[X], const double2 (&h)[X], const double2 (&y)[X],
                                           const int (&part)[X]) {
#pragma unroll
  for (int k = 0; k < X; ++k) {
    const double y1 = part[k] ? y[k].y : y[k].x;
    const double y2 = part[k] ? __longlong_as_double(__double_as_longlong(y[k].x) ^ 0x8000000000000000ULL) : y[k].y;
    c[k] = __dadd_rn(c[k], __dadd_rn(__dmul_rn(h[k].x, y1), __dmul_rn(h[k].y, y2)));
  }
}

// pairs (0,1), (2,3) exchanged when s (register selects; the loads were pair-swapped)
__device__ __forceinline__ void swap_pairs(double2 (&h)[4], int s) {
  if (s) {
    const double2 t0 = h[0], t2 = h[2];
    h[0] = h[1];
    h[1] = t0;
    h[2] = h[3];
    h[3] = t2;
  }
}

// ---- FP32-Gram extension (G32): rows of a stage converted in place to binary32 ----
// operands of one row of a binary32 Gram job (circulant: hi[4] hj[4]; half:
// hx[4] hy[2] hz[4])
template <bool HALF>
__device__ __forceinline__ void g32_load(const GramJob& jb, const float2* row, int nb, float2 (&o)[10]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) o[u] = row[jb.a + nb * u];
  if constexpr (!HALF) {
#pragma unroll
    for (int v = 0; v < 4; ++v) o[4 + v] = row[jb.c + nb * v];
  } else {
#pragma unroll
    for (int w = 0; w < 2; ++w) o[4 + w] = row[jb.y + nb * (jb.yo + w)];
#pragma unroll
    for (int v = 0; v < 4; ++v) o[6 + v] = row[jb.c + nb * v];
  }
}
// the products of one row (gram32_row's arithmetic, operands from registers)
template <bool HALF>
__device__ __forceinline__ void g32_mac(const float2 (&o)[10], const Cj32& cj, f2x (&acc)[16]) {
  if constexpr (!HALF) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) cj.mac(acc[u * 4 + v], o[u], o[4 + v]);
  } else {
    int p = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = u + 1; v < 4; ++v) cj.mac(acc[p++], o[u], o[v]);
#pragma unroll
    for (int w = 0; w < 2; ++w)
#pragma unroll
      for (int v = 0; v < 4; ++v) cj.mac(acc[6 + w * 4 + v], o[4 + w], o[6 + v]);
    const f2x q0 = mul2(pk2(o[0].x, o[1].x), pk2(o[0].x, o[1].x));
    const f2x q1 = mul2(pk2(o[0].y, o[1].y), pk2(o[0].y, o[1].y));
    const f2x q2 = mul2(pk2(o[2].x, o[3].x), pk2(o[2].x, o[3].x));
    const f2x q3 = mul2(pk2(o[2].y, o[3].y), pk2(o[2].y, o[3].y));
    acc[14] = fma2(fma2(q1, cj.one, q0), cj.one, acc[14]);
    acc[15] = fma2(fma2(q3, cj.one, q2), cj.one, acc[15]);
  }
}
// N = 128 in binary32 (G32): the thread's two jobs (t and t + 256) in ONE
// pass over the antenna rows (binary32 accumulators take half the registers,
// so H streams once): job 1's operands load while job 0's products run and
// vice versa; the thread's split matched-filter chain runs alongside in
// binary32: re += fl(fl(hr yr) + fl(hi yi)), im += fl(fl(hr yi) + fl(hi (-yr)))
// (gram_mf_fp32's b)
template <bool HALF1>
__device__ __forceinline__ void g32_rows2(const GramJob& j0, const GramJob& j1, const float2* r0, const float2* r1,
                                          int Np, int nb, int rows, const Cj32& cj, f2x (&acc0)[16],
                                          f2x (&acc1)[16], const float2* hcp, const float2* ycp, int part, float& ca) {
  float2 o0[10], o1[10];
  g32_load<false>(j0, r0, nb, o0);
  float2 hc = hcp[0], yc = ycp[0];
FPM_UNROLL_(FPM_G32_UNROLL)
  for (int mm = 0; mm < rows; ++mm) {
    const int mn = FPM_G32_ROW_CLAMP ? ((mm + 1 < rows) ? mm + 1 : mm) : mm + 1;  // (see kRowClamp)
    g32_load<HALF1>(j1, r1 + mm * Np, nb, o1);
    const float2 nh = hcp[mn * Np], ny = ycp[mn];
    g32_mac<false>(o0, cj, acc0);
    const float y1 = part ? yc.y : yc.x, y2 = part ? -yc.x : yc.y;
    ca = __fadd_rn(ca, __fadd_rn(__fmul_rn(hc.x, y1), __fmul_rn(hc.y, y2)));
    g32_load<false>(j0, r0 + mn * Np, nb, o0);
    g32_mac<HALF1>(o1, cj, acc1);
    hc = nh;
    yc = ny;
  }
}

// producer side: convert stage s (H rows then y rows, binary64 from TMA) to
// binary32 in place (float2 k over the first half of double2 k's bytes).  A
// warp step handles 128 consecutive elements: its stores overwrite the bytes
// of elements < k0/2 + 64, read by this or an earlier step, so the loads of a
// step complete (__syncwarp) before its stores.
__device__ __forceinline__ void g32_convert(double2* buf, int n, int lane) {
  float2* out = reinterpret_cast<float2*>(buf);
#pragma unroll 1
  for (int k0 = 0; k0 < n; k0 += 128) {
    double2 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = k0 + j * 32 + lane;
      v[j] = k < n ? buf[k] : make_double2(0.0, 0.0);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = k0 + j * 32 + lane;
      if (k < n) out[k] = make_float2(__double2float_rn(v[j].x), __double2float_rn(v[j].y));
    }
    __syncwarp();
  }
}

#ifdef FPM_CHECKED
__device__ __forceinline__ long stage_elems_of(const GramGeom& G, int Np) { return ws_stage_elems(G); }
__device__ __forceinline__ int nsl_of(const DetectArgs& a) { return a.ws_nslot; }
#endif

// RS > 0: register split (setmaxnreg) for a 512-thread block: the GWG Gram
// warp groups (gt = 128 * GWG) run with RS registers per thread, the other
// 4 - GWG (producer + CG + idle warps) with the rest of the register file.
template <int WK, int K, int NB, int LB, int RS, int GWG = 2, int G32 = 0, int TA = 0, int SW = 0>
__global__ void __launch_bounds__(512, 1) fpm_detect_ws_kernel(const __grid_constant__ DetectArgs args, const WsLayout sl) {
  // SW: the CG side is four independent solver warps (fpm_detect_sw.cuh), one
  // realization each, instead of a lockstep CG group: thread layout
  // [Gram 0..255 | solver warps 256..383 | producer warp 384..415 | idle],
  // registers RS / kSwRegs / 24 per thread by warp group
  static_assert(!SW || (WK == FK_F64 && (K == FK_F16 || K == FK_BF16) && RS > 0 && GWG == 2 && !G32 && !TA &&
                        ((NB == 16 && LB == 4) || (NB == 8 && LB == 0))),
                "solver warps: fp64 work, 32-bit native u_MV == u_IP, N = 64 with L = 4 or N = 32 plain");
  constexpr int kSwRegs = SW ? ((65536 - RS * 256 - FPM_SW_WG3_REGS * 128) / 128) / 8 * 8 : 0;
  // TA: the fp64 matrix of the hand-off lives in TENSOR MEMORY (two 256-column
  // slots, row q of a group in lane q % 128), staged through a small
  // shared-memory area in rounds -- the 128 KB of shared memory an fp64 A
  // slot took go to the H ring, and two slots decouple the Gram and the CG
  static_assert(!TA || (K == FK_F64 && (NB == 16 || NB == 4)), "A in tensor memory: fp64 matvec, N = 16 / 64");
  // G32: binary32 Gram (FP32-Gram extension, BASELINE c4); only N = 128 (one
  // realization per group, two Gram passes) is instantiated
  static_assert(!G32 || NB == 32, "binary32 Gram: N = 128 only");
  constexpr int kOtherRegs = RS > 0 ? ((512 - RS * GWG) / (4 - GWG)) / 8 * 8 : 0;
  // FPM_CG_SPLIT (c5 at fp64 matvec): the CG group = warp group 3 (128 threads)
  // with its own budget, the producer + idle warps of warp group 2 at the
  // minimum, so that the Gram warps keep FPM_WS_GRAM_REGS registers
  constexpr bool kCgOwn = FPM_CG_SPLIT && K == FK_F64 && NB == 16 && LB == 4 && RS > 0 && GWG == 2 && !G32 && !TA && !SW;
  constexpr int kCgOwnRegs = kCgOwn ? ((65536 - RS * 256 - FPM_SW_WG3_REGS * 128) / 128) / 8 * 8 : 0;
  extern __shared__ __align__(128) unsigned char smem[];
  typedef typename Ar<K>::C C;
  typedef typename Ar<K>::P P;
  const int tid = threadIdx.x;
  const GramGeom& G = args.G;
  const int R = G.R;
  const int N = NB > 0 ? 4 * NB : G.N;
  const int Np = NB > 0 ? 4 * NB : G.Np;
  const int nb = NB > 0 ? NB : G.nb;
  const int gt = args.ws_gt, ct = args.ws_ct;
  const long ngroups = (args.T + R - 1) / R;
  const int my_groups = blockIdx.x < ngroups ? (int)((ngroups - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
  const int nch = (G.M + G.MC - 1) / G.MC;
  const int L = args.bj ? (LB > 0 ? LB : args.L) : 1;
  // compile-time N for the CG sums, except for 16-byte (fp64 / generic)
  // matvec terms under the register split: their unrolled sums do not fit the
  // CG warps' 256 - RS registers, the loop versions do
  constexpr int kCgNC = (NB > 0 && (RS == 0 || RS <= FPM_WIDE_NC_MAX_RS || sizeof(typename Ar<K>::C) != 16 ||
                                    K == FK_F64)) ? 4 * NB : 0;
  const int nblk = args.bj ? (N + L - 1) / L : 1;
  const int ldA = NB > 0 ? lda_for(N, (int)sizeof(C)) : args.ldA;

  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + G.S;
  uint64_t* sfull = full + 2 * G.S + 2;  // [2]
  uint64_t* sempty = sfull + 2;      // [2]
  uint64_t* conv = sempty + 2;       // [S] G32: stage converted to binary32 (producer)
  const int nsl = args.ws_nslot;     // hand-off slots (2, or 1 when two do not fit)
  double2* stages = reinterpret_cast<double2*>(smem + args.off_union);
  unsigned char* slots = smem + args.off_slot;
  __shared__ unsigned long long cnt[FPM_NCOUNTERS];
  __shared__ uint32_t tm_slot;  // TA: tensor-memory base address (tcgen05.alloc)
  // diagnostic timeline of CTA 0, groups 0..7: [j*8 + 0] gram loop start,
  // 1 gram loop end, 2 slot acquired, 3 hand-off done, 4 cg start, 5 cg end
  long long* tr = (diag_trace(args.trace) && blockIdx.x == 0) ? diag_trace(args.trace) : nullptr;

#ifdef FPM_CHECKED
  if (tid == 0) {  // the planner's shared-memory layout lies inside the launch's dynamic allocation
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    const long ends[] = {(long)(2 * G.S + 8) * 8 - args.off_union + 256,  // barriers <= 256 B
                         (long)args.off_union + (long)G.S * stage_elems_of(G, Np) * 16,
                         (long)args.off_ys, (long)args.off_slot + (long)nsl_of(args) * sl.bytes,
                         (long)args.off_bsm + 2L * R * N * 8, (long)args.smem_bytes};
    const long starts[] = {256, args.off_ys, args.off_slot, args.off_bsm, args.off_minv, (long)dyn};
    for (int k = 0; k < 6; ++k)
      if (ends[k] > starts[k]) {
        printf("FPM_CHECKED: shared-memory region %d ends at %ld > %ld (dyn %u)\n", k, ends[k], starts[k], dyn);
        __trap();
      }
    if (gt + 32 + ct > (int)blockDim.x || (gt & 31) || (ct & 31)) __trap();
  }
#endif
  if (tid == 0) {
    for (int s = 0; s < G.S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], gt / 32);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&sfull[k], gt / 32);
      mbar_init(&sempty[k], SW ? R : 1);  // SW: one arrival per realization's solver warp
    }
    if constexpr (G32)
      for (int s = 0; s < G.S; ++s) mbar_init(&conv[s], 1);
    fence_mbar_init();
  }
  if (tid < FPM_NCOUNTERS) cnt[tid] = 0ULL;
  if constexpr (TA) {
    if (tid < 32) tmx_alloc(&tm_slot, 512);
    tmx_fence_before();
  }
  __syncthreads();
  uint32_t tm_base = 0;
  if constexpr (TA) {
    tmx_fence_after();
    tm_base = tm_slot;
  }

  const int stage_elems = ws_stage_elems(G);  // H rows, then the rows' y entries
  // N = 128: the 512 Gram jobs of a realization run as two passes of 256
  // over all antenna rows (H streams twice; the FP64 work is unchanged); the
  // hand-off of pass 0's entries goes out before pass 1 starts
  constexpr int kNpass = (NB == 32 && !G32) ? 2 : (NB > 0 ? 1 : 0);  // 0: run time (G32: both jobs in one pass)
  // the pipelined row loops unrolled by two where the Gram warps have the
  // registers (176 at nb = 16 / 32): c5 fp16 0.755 -> 0.779, c3 0.831 -> 0.864,
  // c4 0.808 -> 0.856 of FP64; at 136 registers (fp64 matvec) and at nb = 4 / 8
  // it measured slower (c5 fp64 0.634 -> 0.621, c1 0.452 -> 0.424, c2 -0.6 %)
  constexpr int kRowUnroll = FPM_PIPE_UNROLL_N > 0 ? FPM_PIPE_UNROLL_N : ((NB == 16 || NB == 32) && RS >= 176 ? 2 : 1);
  // The row loops prefetch row mm + 1 while row mm's products run.  Unclamped
  // (kRowClamp = false), the prefetch after a stage's last row reads one row
  // past the realization's block -- the next block, the stage's y rows or the
  // start of the next shared-memory region: always inside the launch's
  // allocation, never used -- and the operand addresses become pointer bumps
  // with immediate offsets instead of a clamped index multiply: 21-24 fewer
  // integer instructions per two rows (322 -> 301 / 330 -> 306).  Measured:
  // c5 fp16 0.783 -> 0.791, c3 0.862 -> 0.873, c4 0.877 -> 0.881 where the loops
  // are unrolled by two; c5 fp64 0.637 -> 0.631, c2 0.728 -> 0.723, c1 0.461 ->
  // 0.459 elsewhere (kept clamped there).
  constexpr bool kRowClamp = FPM_ROW_CLAMP >= 0 ? (FPM_ROW_CLAMP != 0) : (kRowUnroll < 2);
  const int npass = kNpass ? kNpass : args.ws_npass;
  const long total = (long)my_groups * npass * nch;
  // role layout: ws_order 0 = [Gram | producer | CG], 1 = [CG | producer |
  // Gram].  CG-first gives the latency-bound CG warps the lower warp ids,
  // which the warp schedulers favour when several warps are ready, so the
  // throughput-bound Gram warps fill the issue slots the CG chains leave.
  const int cbase = SW ? gt : kCgOwn ? 384 : args.ws_order ? 0 : gt + 32;
  const int pbase = SW ? gt + 128 : args.ws_order ? ct : gt;
  const int gbase = SW ? 0 : args.ws_order ? ct + 32 : 0;
  if (tid >= gbase && tid < gbase + gt) {
    if constexpr (RS > 0) reg_alloc<RS>();
    const int tid = threadIdx.x - gbase;  // Gram-local thread id
    // =========================== Gram warps ===========================
    NamedBar gbar{1, gt};
    const GramJob job0 = gram_job(tid, R, nb);
    // matched-filter chain accumulators live in shared memory between chunks
    // (one binary64 per chain), so no chain state occupies registers across
    // the tile loop
    double* bsm = reinterpret_cast<double*>(smem + args.off_bsm);
    // Compile-time nb in {4, 8, 16}: the layout has 2*R*N = (16/nb) * gt
    // chains, so each thread carries kCPT = 16/nb chains inside the tile loop
    // (their latency hidden by the tile math).  Chain 0 is software-pipelined
    // with the tile operands; the extra chains (N = 32: one, N = 16: three)
    // load their operands at the top of each row and add after its products.
    // (extra chains only with the register split: at 128 registers they spill)
    // N = 32 (nb = 8; R * N == 256 == gt): one "paired" chain per thread
    // instead of two split ones -- chain (g, n) accumulates b.re and b.im
    // from one H load and one (warp-broadcast) y load per row:
    //   re += fl(fl(hr yr) + fl(hi yi)),  im += fl(fl(hr yi) - fl(hi yr))
    // (bit-identical to the split chains: fl(hi (-yr)) = -fl(hi yr)); the
    // split form needs 2.4x the shared-memory wavefronts per row
    // N = 16 (nb = 4): two paired chains per thread, (g, n) and (g, n + 8),
    // sharing the y load (the four split chains took 24 wavefronts per
    // warp-row beside the tile's 32: shared memory near its bandwidth)
    constexpr bool kPair = (NB == 8 || NB == 4) && RS > 0;
    constexpr int kPPT = NB == 4 ? 2 : 1;  // paired chains per thread
    constexpr int kCPT = kPair ? 1 : (NB == 16 || NB == 32 || ((NB == 4 || NB == 8) && RS > 0)) ? (NB == 32 ? 1 : 16 / NB) : 0;
    constexpr bool kChainInLoop = kCPT > 0;
    constexpr int kXC = kCPT > 1 ? kCPT - 1 : 1;  // extra chains (array size >= 1)
    const int cq_g = kPair ? tid / (N / kPPT) : tid / (2 * N), cq_e = kPair ? tid - cq_g * (N / kPPT) : tid - cq_g * 2 * N;
    const int cq_part = kPair ? 0 : cq_e / N, cq_n = cq_e - cq_part * N;
    const int cq_hoff = cq_g * G.MC * Np + cq_n, cq_yoff = cq_g * G.MC;  // y: the stage's y block
    int xq_hoff[kXC], xq_yoff[kXC], xq_part[kXC];
#pragma unroll
    for (int k = 0; k < kXC; ++k) {
      const int q = tid + (k + 1) * gt;  // < 2*R*N: in-bounds operands even for idle chains
      const int g = q / (2 * N), e = q - g * 2 * N;
      xq_part[k] = e / N;
      xq_hoff[k] = g * G.MC * Np + (e - xq_part[k] * N);
      xq_yoff[k] = g * G.MC;
    }

    // ring position of the next stage this warp consumes: stage index and
    // phase parity advance with every stage (no 64-bit division per stage)
    int rs = 0;
    uint32_t rph = 0;
#pragma unroll 1
    for (int j = 0; j < my_groups; ++j) {
      const long t0 = ((long)blockIdx.x + (long)j * gridDim.x) * R;
      const int Rv = (int)min((long)R, args.T - t0);
      const int slot = nsl == 2 ? (j & 1) : 0;  // hand-off slot and its use count
      const int use = nsl == 2 ? (j >> 1) : j;
      const int nchain = 2 * Rv * N;
      const bool chain_ok = kChainInLoop && tid < (kPair ? Rv * N / kPPT : nchain);
      double ca = 0.0, cb = 0.0;  // cb: imaginary part of a paired chain
      double ca2 = 0.0, cb2 = 0.0;  // kPPT = 2: the second paired chain (entry n + N/2)
      double cx[kXC];
#pragma unroll
      for (int k = 0; k < kXC; ++k) cx[k] = 0.0;
      if (!kChainInLoop) {
#pragma unroll 1
        for (int q = tid; q < nchain; q += gt) bsm[q] = 0.0;
      }
      double ca_keep = 0.0, cb_keep = 0.0, cx_keep[kXC];
      float ca32 = 0.f, ca32_keep = 0.f;  // G32: the split chain in binary32  // chains of pass 0 (later passes recompute and discard them)
#pragma unroll
      for (int k = 0; k < kXC; ++k) cx_keep[k] = 0.0;
#pragma unroll 1
      for (int pass = 0; pass < (kNpass ? kNpass : npass); ++pass) {
      const GramJob job = kNpass == 1 ? job0 : gram_job(tid + pass * gt, R, nb);
      const int joff = job.g * G.MC * Np;
      const bool active = job.g >= 0 && job.g < Rv;
      // nb = 4 (c1: 8 jobs per realization, two realizations per quarter-warp,
      // realization blocks 0 mod 128 bytes apart): odd realizations load their
      // operand pairs swapped (u ^ 1), so the two realizations' LDS.128 of one
      // instruction fall in different bank halves (2-way conflicts otherwise);
      // the triangle operands are swapped back in registers, the rest is
      // undone in the hand-off's index map
      constexpr bool kPerm = NB == 4;
      const int psw = kPerm ? (job.g & 1) : 0;
      const int pu[4] = {nb * (0 ^ psw), nb * (1 ^ psw), nb * (2 ^ psw), nb * (3 ^ psw)};
      double2 acc[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = make_double2(0.0, 0.0);
      f2x acc32[16], acc32b[16];  // G32: binary32 pairs of the thread's jobs t and t + 256
#pragma unroll
      for (int k = 0; k < 16; ++k) acc32[k] = acc32b[k] = 0ull;
      const GramJob job1 = G32 ? gram_job(tid + gt, R, nb) : job;
      // serial mode (debug bit 8): the Gram of group j starts only once the CG
      // has released the slot of group j - nsl, i.e. no Gram / CG overlap --
      // faster when both compete for the FP64 pipe (fp64 matvec)
      if ((diag_bits(args.debug) & 8) && j >= nsl && !args.gram_A) mbar_wait(&sempty[slot], (uint32_t)((use - 1) & 1));
      if (tr && tid == 0 && j < 8) tr[j * 8 + 0] = clock64();

#pragma unroll 1
      for (int c = 0; c < nch; ++c) {
        const int s = rs, gc = (j * npass + pass) * nch + c;  // gc: diagnostics only
        FPM_GFWAIT(G32 ? &conv[s] : &full[s], rph);
        if (++rs == G.S) {
          rs = 0;
          rph ^= 1u;
        }
        diag_jitter(args.debug, 2, gc);
        const double2* sb = stages + s * stage_elems;
        const double2* sy = sb + R * G.MC * Np;  // y rows m0 .. m0 + rows of every realization of the group
        const int m0 = c * G.MC;
        const int rows = min(G.MC, G.M - m0);
        const double2* pa = sb + joff + job.a;
        const double2* pc = sb + joff + job.c;
        if constexpr (G32) {
          const float2* sbf = reinterpret_cast<const float2*>(sb);
          const float2* syf = sbf + 2 * (R * G.MC * Np);  // the stage's y rows (converted)
          const Cj32 cj{args.g32_one, args.g32_pm};
          const float2* r1 = sbf + job1.g * G.MC * Np;
          if (active && !job1.half)
            g32_rows2<false>(job, job1, sbf + joff, r1, Np, nb, rows, cj, acc32, acc32b, sbf + cq_hoff, syf + cq_yoff,
                             cq_part, ca32);
          else if (active)
            g32_rows2<true>(job, job1, sbf + joff, r1, Np, nb, rows, cj, acc32, acc32b, sbf + cq_hoff, syf + cq_yoff,
                            cq_part, ca32);
        } else if (diag_bits(args.debug) & 4) {
          // diagnostic: Gram math skipped (CG measured without FP64 contention)
        } else if (active && !job.half) {
          // software-pipelined: row mm+1's operands (tile and chain) are in
          // flight while row mm's products run.  The chain runs branch-free
          // (its operands are in-bounds stale data for an idle chain, and the
          // result is only stored when chain_ok); part 1 reads (yi, yr) and
          // flips the sign of yr exactly (sign-bit xor = IEEE negation).
          const double* yrow = reinterpret_cast<const double*>(sy + cq_yoff);
          const double* y1p = yrow + cq_part;
          const double* y2p = yrow + (1 - cq_part);
          const unsigned long long yneg = cq_part ? 0x8000000000000000ULL : 0ULL;
          const double2* hcp = sb + cq_hoff;
          double2 hi[4], hj[4], hc = make_double2(0.0, 0.0);
          double y1 = 0.0, y2 = 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u) hi[u] = pa[pu[u]];
#pragma unroll
          for (int v = 0; v < 4; ++v) hj[v] = pc[pu[v]];
          double2 hc2 = make_double2(0.0, 0.0);
          if (kChainInLoop) {
            hc = hcp[0];
            y1 = y1p[0];
            y2 = y2p[0];
            if constexpr (kPPT == 2) hc2 = hcp[N / 2];
          }
#pragma unroll kRowUnroll
          for (int mm = 0; mm < rows; ++mm) {
            const int mn = kRowClamp ? ((mm + 1 < rows) ? mm + 1 : mm) : mm + 1;
            double2 ni[4], nj[4], nhc = hc;
            double ny1 = y1, ny2 = y2;
#pragma unroll
            for (int u = 0; u < 4; ++u) ni[u] = pa[mn * Np + pu[u]];
#pragma unroll
            for (int v = 0; v < 4; ++v) nj[v] = pc[mn * Np + pu[v]];
            double2 nhc2 = hc2;
            if (kChainInLoop) {
              nhc = hcp[mn * Np];
              ny1 = y1p[2 * mn];
              ny2 = y2p[2 * mn];
              if constexpr (kPPT == 2) nhc2 = hcp[mn * Np + N / 2];
            }
            double2 xh[kXC], xy[kXC];
            if constexpr (kCPT > 1) xchain_load<kXC>(sb, sy, 0, mm, Np, xq_hoff, xq_yoff, xh, xy);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int v = 0; v < 4; ++v) cmac_conj(acc[u * 4 + v], hi[u], hj[v]);
            if (kChainInLoop) {
              const double y2s = __longlong_as_double(__double_as_longlong(y2) ^ yneg);
              ca = __dadd_rn(ca, __dadd_rn(__dmul_rn(hc.x, y1), __dmul_rn(hc.y, y2s)));
              if constexpr (kPair) cb = __dadd_rn(cb, __dsub_rn(__dmul_rn(hc.x, y2), __dmul_rn(hc.y, y1)));
              if constexpr (kPPT == 2) {
                ca2 = __dadd_rn(ca2, __dadd_rn(__dmul_rn(hc2.x, y1), __dmul_rn(hc2.y, y2)));
                cb2 = __dadd_rn(cb2, __dsub_rn(__dmul_rn(hc2.x, y2), __dmul_rn(hc2.y, y1)));
              }
            }
            if constexpr (kCPT > 1) xchain_add<kXC>(cx, xh, xy, xq_part);
#pragma unroll
            for (int u = 0; u < 4; ++u) hi[u] = ni[u];
#pragma unroll
            for (int v = 0; v < 4; ++v) hj[v] = nj[v];
            hc = nhc;
            hc2 = nhc2;
            y1 = ny1;
            y2 = ny2;
          }
        } else if (active) {
          // half-pair job, software-pipelined like the circulant loop above
          const double2* py = sb + joff + job.y + nb * job.yo;
          const double* yrow = reinterpret_cast<const double*>(sy + cq_yoff);
          const double* y1p = yrow + cq_part;
          const double* y2p = yrow + (1 - cq_part);
          const unsigned long long yneg = cq_part ? 0x8000000000000000ULL : 0ULL;
          const double2* hcp = sb + cq_hoff;
          double2 hx[4], hy[2], hz[4], hc = make_double2(0.0, 0.0);
          double y1 = 0.0, y2 = 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u) hx[u] = pa[pu[u]];
          if (kPerm) swap_pairs(hx, psw);
#pragma unroll
          for (int w = 0; w < 2; ++w) hy[w] = py[nb * (w ^ psw)];
#pragma unroll
          for (int v = 0; v < 4; ++v) hz[v] = pc[pu[v]];
          double2 hc2 = make_double2(0.0, 0.0);
          if (kChainInLoop) {
            hc = hcp[0];
            y1 = y1p[0];
            y2 = y2p[0];
            if constexpr (kPPT == 2) hc2 = hcp[N / 2];
          }
#pragma unroll kRowUnroll
          for (int mm = 0; mm < rows; ++mm) {
            const int mn = kRowClamp ? ((mm + 1 < rows) ? mm + 1 : mm) : mm + 1;
            double2 nx[4], ny[2], nz[4], nhc = hc;
            double ny1 = y1, ny2 = y2;
#pragma unroll
            for (int u = 0; u < 4; ++u) nx[u] = pa[mn * Np + pu[u]];
            if (kPerm) swap_pairs(nx, psw);
#pragma unroll
            for (int w = 0; w < 2; ++w) ny[w] = py[mn * Np + nb * (w ^ psw)];
#pragma unroll
            for (int v = 0; v < 4; ++v) nz[v] = pc[mn * Np + pu[v]];
            double2 nhc2 = hc2;
            if (kChainInLoop) {
              nhc = hcp[mn * Np];
              ny1 = y1p[2 * mn];
              ny2 = y2p[2 * mn];
              if constexpr (kPPT == 2) nhc2 = hcp[mn * Np + N / 2];
            }
            double2 xh[kXC], xy[kXC];
            if constexpr (kCPT > 1) xchain_load<kXC>(sb, sy, 0, mm, Np, xq_hoff, xq_yoff, xh, xy);
            int p = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int v = u + 1; v < 4; ++v) cmac_conj(acc[p++], hx[u], hx[v]);
            acc[14].x = __dadd_rn(acc[14].x, sqmag(hx[0]));
            acc[14].y = __dadd_rn(acc[14].y, sqmag(hx[1]));
            acc[15].x = __dadd_rn(acc[15].x, sqmag(hx[2]));
            acc[15].y = __dadd_rn(acc[15].y, sqmag(hx[3]));
#pragma unroll
            for (int w = 0; w < 2; ++w)
#pragma unroll
              for (int v = 0; v < 4; ++v) cmac_conj(acc[6 + w * 4 + v], hy[w], hz[v]);
            if (kChainInLoop) {
              const double y2s = __longlong_as_double(__double_as_longlong(y2) ^ yneg);
              ca = __dadd_rn(ca, __dadd_rn(__dmul_rn(hc.x, y1), __dmul_rn(hc.y, y2s)));
              if constexpr (kPair) cb = __dadd_rn(cb, __dsub_rn(__dmul_rn(hc.x, y2), __dmul_rn(hc.y, y1)));
              if constexpr (kPPT == 2) {
                ca2 = __dadd_rn(ca2, __dadd_rn(__dmul_rn(hc2.x, y1), __dmul_rn(hc2.y, y2)));
                cb2 = __dadd_rn(cb2, __dsub_rn(__dmul_rn(hc2.x, y2), __dmul_rn(hc2.y, y1)));
              }
            }
            if constexpr (kCPT > 1) xchain_add<kXC>(cx, xh, xy, xq_part);
#pragma unroll
            for (int u = 0; u < 4; ++u) hx[u] = nx[u];
#pragma unroll
            for (int w = 0; w < 2; ++w) hy[w] = ny[w];
#pragma unroll
            for (int v = 0; v < 4; ++v) hz[v] = nz[v];
            hc = nhc;
            hc2 = nhc2;
            y1 = ny1;
            y2 = ny2;
          }
        } else if (kChainInLoop) {  // idle job slot (partial group): its chains only
#pragma unroll 1
          for (int mm = 0; mm < rows; ++mm) {
            const double2 h = sb[cq_hoff + mm * Np];
            const double2 yv = sy[cq_yoff + mm];
            const double y1 = cq_part ? yv.y : yv.x, y2 = cq_part ? -yv.x : yv.y;
            ca = __dadd_rn(ca, __dadd_rn(__dmul_rn(h.x, y1), __dmul_rn(h.y, y2)));
            if constexpr (kPair) cb = __dadd_rn(cb, __dsub_rn(__dmul_rn(h.x, yv.y), __dmul_rn(h.y, yv.x)));
            if constexpr (kPPT == 2) {
              const double2 h2 = sb[cq_hoff + mm * Np + N / 2];
              ca2 = __dadd_rn(ca2, __dadd_rn(__dmul_rn(h2.x, yv.x), __dmul_rn(h2.y, yv.y)));
              cb2 = __dadd_rn(cb2, __dsub_rn(__dmul_rn(h2.x, yv.y), __dmul_rn(h2.y, yv.x)));
            }
            if constexpr (kCPT > 1) {
              double2 xh[kXC], xy[kXC];
              xchain_load<kXC>(sb, sy, 0, mm, Np, xq_hoff, xq_yoff, xh, xy);
              xchain_add<kXC>(cx, xh, xy, xq_part);
            }
          }
        }
        // matched-filter chains (split re / im, exact): chain q -> slot g,
        // entry n, part (0 re / 1 im); accumulators round-trip through smem
        if (!kChainInLoop && pass == 0 && !(diag_bits(args.debug) & 2)) {
#pragma unroll 1
          for (int q = tid; q < nchain; q += gt) {
            const int g = q / (2 * N), e = q - g * 2 * N;
            const int part = e / N, n = e - part * N;
            const double2* hcol = sb + g * G.MC * Np + n;
            const double2* yy = sy + g * G.MC;
            double a = bsm[q];
#pragma unroll 1
            for (int mm = 0; mm < rows; ++mm) {
              const double2 h = hcol[mm * Np];
              const double2 yv = yy[mm];
              const double y1 = part ? yv.y : yv.x, y2 = part ? -yv.x : yv.y;
              a = __dadd_rn(a, __dadd_rn(__dmul_rn(h.x, y1), __dmul_rn(h.y, y2)));
            }
            bsm[q] = a;
          }
        }
        diag_jitter(args.debug, 3, gc);
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[s]);
      }

      if (kNpass != 1 && pass == 0) {
        ca_keep = ca;
        cb_keep = cb;
        ca32_keep = ca32;
#pragma unroll
        for (int k = 0; k < kXC; ++k) cx_keep[k] = cx[k];
      }
      if (!G32 && args.gram_A) {
        // Gram-only mode (fpm_gram): final / mirror entries straight to HBM
        // in binary64, no hand-off to the CG side
        if (active) {
          double2* Agl = args.gram_A + (t0 + job.g) * (long)N * N;
          gram_entries(
              job, acc, nb, N, args.sigma2,
              [&](int i, int jx, double2 vij, double2 vji) {
                Agl[(long)i * N + jx] = vij;
                Agl[(long)jx * N + i] = vji;
              },
              [&](int i, double2 vii) { Agl[(long)i * N + i] = vii; }, psw);
        }
        if (pass + 1 < npass) continue;
        if (kNpass != 1) {
          ca = ca_keep;
          cb = cb_keep;
#pragma unroll
          for (int k = 0; k < kXC; ++k) cx[k] = cx_keep[k];
        }
        if (kPair) {
          if (chain_ok) args.gram_b[(t0 + cq_g) * N + cq_n] = make_double2(ca, cb);
          if (kPPT == 2 && chain_ok) args.gram_b[(t0 + cq_g) * N + cq_n + N / 2] = make_double2(ca2, cb2);
        } else if (kChainInLoop) {
          if (chain_ok) reinterpret_cast<double*>(args.gram_b + (t0 + cq_g) * N + cq_n)[cq_part] = ca;
#pragma unroll
          for (int k = 0; k < kCPT - 1; ++k) {
            const int q = tid + (k + 1) * gt;
            if (q < nchain) {
              const int g = q / (2 * N), e = q - g * 2 * N;
              reinterpret_cast<double*>(args.gram_b + (t0 + g) * N + (e - xq_part[k] * N))[xq_part[k]] = cx[k];
            }
          }
        } else {
#pragma unroll 1
          for (int q = tid; q < nchain; q += gt) {
            const int g = q / (2 * N), e = q - g * 2 * N;
            const int part = e / N;
            reinterpret_cast<double*>(args.gram_b + (t0 + g) * N + (e - part * N))[part] = bsm[q];
          }
        }
        gbar.sync();
        continue;
      }
      // ---- hand-off: wait until the CG side has released this slot ----
      if (pass == 0) {
        if (tr && tid == 0 && j < 8) tr[j * 8 + 1] = clock64();
        if (tr && (tid & 31) == 0 && j == 2) tr[72 + tid / 32] = clock64();
        diag_jitter(args.debug, 4, j);
        if (j >= nsl) FPM_GSWAIT(&sempty[slot], (uint32_t)((use - 1) & 1));
        if (tr && tid == 0 && j < 8) tr[j * 8 + 2] = clock64();
      }
      unsigned char* sp = slots + slot * sl.bytes;
      C* At = reinterpret_cast<C*>(sp + sl.at);
      double2* bS = reinterpret_cast<double2*>(sp + sl.b);
      double2* dS = reinterpret_cast<double2*>(sp + sl.d);
      const int nbt = R * nblk;
      const bool onchip = args.bj && !args.minv_in;
      if constexpr (TA) {
        // fp64 A -> tensor memory slot `slot`, in rounds of RR rows through the
        // staging area (pitch N + 1: conflict-free row reads); the Gram warps
        // of a lane quarter move that quarter's rows (tcgen05.st 32x32b)
        const int RR = args.ws_rr, RNt = R * N, pitch = N + 1;
        double2* stg = reinterpret_cast<double2*>(smem + args.off_stg);
        const int wg = tid >> 5, lane = tid & 31;
        const int Q = (gbase / 32 + wg) & 3;
        const int nwq = gt / 128, kq = wg >> 2;  // Gram warps per lane quarter, this warp's rank
        const uint32_t tslot = tm_base + (uint32_t)(slot * 256);
        double2* dg = dS + job.g * nblk;
        tmx_fence_after();  // the CG's reads of this slot (released through sempty) came first
        long long tw = 0, tmv = 0, tc0 = 0;  // diagnostic: time in entry writes / moves (thread 0)
#pragma unroll 1
        for (int r0 = 0; r0 < RNt; r0 += RR) {
          if (tr && tid == 0 && j < 8) tc0 = clock64();
          if (active) {
            const int qg = job.g * N - r0;
            gram_entries(
                job, acc, nb, N, args.sigma2,
                [&](int i, int jx, double2 vij, double2 vji) {
                  if ((unsigned)(qg + i) < (unsigned)RR) stg[(qg + i) * pitch + jx] = vij;
                  if ((unsigned)(qg + jx) < (unsigned)RR) stg[(qg + jx) * pitch + i] = vji;
                  if (onchip && r0 == 0) {
                    const int kb = i / L;
                    if (kb == jx / L) {
                      const int il = i - kb * L, jl = jx - kb * L;
                      dg[(il * L + jl) * nbt + kb] = vij;
                      dg[(jl * L + il) * nbt + kb] = vji;
                    }
                  }
                },
                [&](int i, double2 vii) {
                  if ((unsigned)(qg + i) < (unsigned)RR) stg[(qg + i) * pitch + i] = vii;
                  if (onchip && r0 == 0) {
                    const int kb = i / L, il = i - kb * L;
                    dg[(il * L + il) * nbt + kb] = vii;
                  }
                },
                psw);
          }
          gbar.sync();
          if (tr && tid == 0 && j < 8) {
            const long long t1 = clock64();
            tw += t1 - tc0;
            tc0 = t1;
          }
#pragma unroll 1
          for (int qb = r0; qb < r0 + RR; qb += 32) {
            if (((qb >> 5) & 3) != Q) continue;  // warp-uniform
            const int srow = qb - r0 + lane, RB = qb >> 7, per = N / nwq;
            const uint32_t ta = tslot + ((uint32_t)(Q * 32) << 16) + (uint32_t)(RB * 4 * N);
#pragma unroll 2
            for (int e = kq * per; e < (kq + 1) * per; e += 4) {
              uint32_t v[16];
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                const double2 a = stg[srow * pitch + e + jj];
                v[4 * jj] = __double2loint(a.x);
                v[4 * jj + 1] = __double2hiint(a.x);
                v[4 * jj + 2] = __double2loint(a.y);
                v[4 * jj + 3] = __double2hiint(a.y);
              }
              tmx_st16(ta + (uint32_t)(4 * e), v);
            }
          }
          gbar.sync();  // the staging area is free for the next round
          if (tr && tid == 0 && j < 8) tmv += clock64() - tc0;
        }
        tmx_wait_st();
        tmx_fence_before();
        if (tr && tid == 0 && j < 8) {
          tr[j * 8 + 6] = tw;
          tr[j * 8 + 7] = tmv;
        }
      } else if (active) {
        C* Ag = At + job.g * N * (SW ? N : ldA);  // SW: unpadded, swizzled (CgwLayout::at)
        double2* dg = dS + job.g * nblk;
        auto aidx = [&](int i, int jx) -> int {
          if constexpr (SW) return CgwLayout<K, 4 * NB, 0>::at(i, jx);
          else return i * ldA + jx;
        };
        // (onchip implies block-Jacobi: the block size is the compile-time LB
        // when there is one, so the index divisions are shifts; not for 16-byte
        // entries, whose 136-register Gram warps spill the unrolled form:
        // c5 fp64 0.632 -> 0.595)
        const int Ld = (LB > 0 && sizeof(C) < 16) ? LB : L;
        auto put = [&](int i, int jx, double2 vij, double2 vji) {
          Ag[aidx(i, jx)] = Ar<K>::rnd(vij, args.pr.mv);
          Ag[aidx(jx, i)] = Ar<K>::rnd(vji, args.pr.mv);
          if (onchip) {
            const int kb = i / Ld;
            if (kb == jx / Ld) {
              const int il = i - kb * Ld, jl = jx - kb * Ld;
              dg[(il * Ld + jl) * nbt + kb] = vij;
              dg[(jl * Ld + il) * nbt + kb] = vji;
            }
          }
        };
        auto put_diag = [&](int i, double2 vii) {
          Ag[aidx(i, i)] = Ar<K>::rnd(vii, args.pr.mv);
          if (onchip) {
            const int kb = i / Ld, il = i - kb * Ld;
            dg[(il * Ld + il) * nbt + kb] = vii;
          }
        };
        if constexpr (G32) {
          gram32_entries(job, acc32, nb, N, __double2float_rn(args.sigma2), put, put_diag);
          gram32_entries(job1, acc32b, nb, N, __double2float_rn(args.sigma2), put, put_diag);
        } else {
          gram_entries(job, acc, nb, N, args.sigma2, put, put_diag, psw);
        }
      }
      if (pass + 1 < npass) continue;
      } // pass loop (the last pass falls through with its slot pointers)
      unsigned char* sp = slots + slot * sl.bytes;
      double2* bS = reinterpret_cast<double2*>(sp + sl.b);
      if (kNpass != 1) {
        ca = ca_keep;
        cb = cb_keep;
        ca32 = ca32_keep;
#pragma unroll
        for (int k = 0; k < kXC; ++k) cx[k] = cx_keep[k];
      }
      if constexpr (G32) ca = (double)ca32;  // exact widening
      if (kPair) {
        if (chain_ok) bS[cq_g * N + cq_n] = make_double2(ca, cb);
        if (kPPT == 2 && chain_ok) bS[cq_g * N + cq_n + N / 2] = make_double2(ca2, cb2);
      } else if (kChainInLoop) {
        if (chain_ok) reinterpret_cast<double*>(bS + cq_g * N + cq_n)[cq_part] = ca;
#pragma unroll
        for (int k = 0; k < kCPT - 1; ++k) {
          const int q = tid + (k + 1) * gt;
          if (q < nchain) {
            const int g = q / (2 * N), e = q - g * 2 * N;
            reinterpret_cast<double*>(bS + g * N + (e - xq_part[k] * N))[xq_part[k]] = cx[k];
          }
        }
      } else {
#pragma unroll 1
        for (int q = tid; q < nchain; q += gt) {
          const int g = q / (2 * N), e = q - g * 2 * N;
          const int part = e / N;
          reinterpret_cast<double*>(bS + g * N + (e - part * N))[part] = bsm[q];
        }
      }
      // every Gram warp publishes its own part of the slot (sfull counts the
      // Gram warps): a warp that is done goes straight on to the next group
      // instead of waiting for the slowest one at a group barrier
      __syncwarp();
      diag_jitter(args.debug, 5, j);
      if ((tid & 31) == 0) mbar_arrive(&sfull[slot]);
      if (tr && tid == 0 && j < 8) tr[j * 8 + 3] = clock64();
    }
  } else if (SW && tid >= cbase && tid < cbase + 128) {
    // warp group 2: the solver warps, on their own register budget (the role's
    // code must be dominated by this reallocation alone: ptxas budgets a join
    // of differently sized branches at the smaller count)
    if constexpr (kSwRegs > 128) reg_alloc<kSwRegs>();
    else if constexpr (SW && kSwRegs < 128) reg_dealloc<kSwRegs>();
    if (!args.gram_A) {
    // ========================== solver warps ==========================
    // realization ticket q = j * R + g (group j, entry g) belongs to solver
    // warp q % 4, which takes its tickets in order (the planner only picks
    // layouts in which a warp sees EVERY use of the slots it consumes -- R a
    // multiple of 4, or R = 2 on two slots -- so its phase-parity waits never
    // skip a phase): wait for the group's slot,
    // block inverses (lanes 0 .. N/L-1, one block each), the (BJ-)CG, release
    // the slot (sempty counts the R realizations), slicer / counters / write-back
    if constexpr (SW) {
      constexpr int NC = 4 * NB, RPL = NC / 32, LBm = LB > 0 ? LB : 1, NBLK = LB > 0 ? NC / LB : 1;
      const int w = (tid - cbase) >> 5, l = tid & 31;
      unsigned char* scr = smem + args.off_vec + w * SwScratch<K, NC, LB>::bytes;
      const int bps = 2 * args.sl.bpa;
      unsigned long long be = 0, se = 0;
      const long nq = (long)my_groups * R;
#pragma unroll 1
      for (long q = w; q < nq; q += 4) {
        const int j = (int)(q / R), g = (int)(q - (long)j * R);
        const long t0 = ((long)blockIdx.x + (long)j * gridDim.x) * R;
        const int Rv = (int)min((long)R, args.T - t0);
        const int slot = nsl == 2 ? (j & 1) : 0;
        const int use = nsl == 2 ? (j >> 1) : j;
        unsigned char* sp = slots + slot * sl.bytes;
        FPM_CWAIT(&sfull[slot], (uint32_t)(use & 1));
        diag_jitter(args.debug, 6, j);
        if (tr && g == 0 && l == 0 && j < 8) tr[j * 8 + 4] = clock64();
        if (g >= Rv) {  // entry past T in the last group: nothing to solve
          __syncwarp();
          if (l == 0) mbar_arrive(&sempty[slot]);
          continue;
        }
        const long t = t0 + g;
        const C* Ag = reinterpret_cast<const C*>(sp + sl.at) + g * NC * NC;
        const double2* bv = reinterpret_cast<const double2*>(sp + sl.b) + g * NC;
        double2 m[RPL][LBm];
        bool live = true;
        if constexpr (LB > 0) {
          if (args.minv_in) {
#pragma unroll
            for (int jr = 0; jr < RPL; ++jr)
#pragma unroll
              for (int k = 0; k < LB; ++k) m[jr][k] = args.minv_in[(t * NC + l + 32 * jr) * LB + k];
          } else {
            const double2* dS = reinterpret_cast<const double2*>(sp + sl.d);
            double2* fac = reinterpret_cast<double2*>(scr);            // Cholesky factors, interleaved over blocks
            double2* inv = fac + NC * LB;                               // inverses, column-major per block
            bool ok = true;
            if (l < NBLK) ok = hpd_inverse<LB>(dS + g * NBLK + l, R * NBLK, fac + l, NBLK, inv + l * LB * LB, LB);
            const unsigned bad = __ballot_sync(0xffffffffu, !ok);
            if (bad) {
              live = false;
              if (l == 0) atomicAdd(&cnt[FPM_CNT_NONPD], (unsigned long long)__popc(bad));
            }
            __syncwarp();
#pragma unroll
            for (int jr = 0; jr < RPL; ++jr) {
              const int i = l + 32 * jr, kb = i / LB, il = i - kb * LB;
#pragma unroll
              for (int k = 0; k < LB; ++k) m[jr][k] = inv[kb * LB * LB + k * LB + il];  // row il of the block
            }
            __syncwarp();  // the scratch is the CG's from here on
          }
        } else {
#pragma unroll
          for (int jr = 0; jr < RPL; ++jr) m[jr][0] = make_double2(0.0, 0.0);
        }
        double2 xs[RPL];
#pragma unroll
        for (int jr = 0; jr < RPL; ++jr) xs[jr] = make_double2(0.0, 0.0);
        int bk = -1, dv = -1;
        if (live) sw_solve<K, NC, LB>(Ag, bv, m, scr, args.iters, args.textbook != 0, args.pr, l, xs, bk, dv);
        // slot no longer needed by this realization (A, b, diagonal blocks consumed)
        __syncwarp();
        diag_jitter(args.debug, 7, j);
        if (l == 0) mbar_arrive(&sempty[slot]);
        if (tr && g == 0 && l == 0 && j < 8) tr[j * 8 + 5] = clock64();
#pragma unroll
        for (int jr = 0; jr < RPL; ++jr) {
          const long gq = t * NC + l + 32 * jr;
          args.x[gq] = xs[jr];
          int sym;
          be += slice_one(xs[jr], args.tx ? args.tx + gq * bps : nullptr, args.rx ? args.rx + gq * bps : nullptr,
                          args.sl, &sym);
          se += sym;
        }
        if (l == 0) {
          args.brk[t] = bk;
          args.div[t] = dv;
          if (dv >= 0) atomicAdd(&cnt[FPM_CNT_DIVERGED], 1ULL);
          if (bk >= 0) atomicAdd(&cnt[FPM_CNT_BREAKDOWN], 1ULL);
          atomicAdd(&cnt[FPM_CNT_TRIALS], 1ULL);
        }
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        be += __shfl_xor_sync(0xffffffffu, be, off);
        se += __shfl_xor_sync(0xffffffffu, se, off);
      }
      if (l == 0) {
        if (be) atomicAdd(&cnt[FPM_CNT_BIT_ERRORS], be);
        if (se) atomicAdd(&cnt[FPM_CNT_SYMBOL_ERRORS], se);
      }
    }
    }
  } else if (kCgOwn && tid >= cbase && tid < cbase + ct && !args.gram_A) {
    // FPM_CG_SPLIT: the CG group is warp group 3 at its own register budget
    // (its own top-level branch: ptxas budgets code after a join of differently
    // sized setmaxnreg branches at the smaller count)
    if constexpr (kCgOwnRegs > 128) reg_alloc<kCgOwnRegs>();
    else if constexpr (kCgOwnRegs < 128) reg_dealloc<kCgOwnRegs>();
#include "fpm_detect_ws_cgrole.cuh"
  } else {
    // the producer warp and the CG warp groups hand registers to the Gram warps
    // (SW: warp group 3 = the producer warp and three idle warps; FPM_CG_SPLIT:
    // warp group 2 = the same)
    if constexpr (SW) reg_dealloc<FPM_SW_WG3_REGS>();
    else if constexpr (kCgOwn) reg_dealloc<FPM_SW_WG3_REGS>();
    else if constexpr (RS > 0) reg_dealloc<kOtherRegs>();
    if (tid >= pbase && tid < pbase + 32) {
    // ========================= producer warp ==========================
    // the whole warp issues (many realizations per group at small N: one bulk
    // copy per realization and stage, spread over the lanes); lane 0 posts the
    // expected bytes, every lane waits on the ring barriers
    const int pl = tid - pbase;
    const int pn = kProducerLanes;
    if (pl < pn) {
      // issue chunk c of group jj into stage s
      auto issue = [&](int jj, int c, int s) {
        const long t0 = ((long)blockIdx.x + (long)jj * gridDim.x) * R;
        const int Rv = (int)min((long)R, args.T - t0);
        if (args.use_tma) {
          // one tensor-map TMA per operand and stage: the whole group's rows
          // m0 .. m0+MC of H and of y (realizations past T / rows past M are
          // zero-filled and never read)
          if (pl == 0) {
            double2* sbuf = stages + s * stage_elems;
            mbar_expect_tx(&full[s], (uint32_t)R * (uint32_t)G.MC * ((uint32_t)G.N * 16u + 16u));
            tma_load_3d(sbuf, &args.tmH, 0, c * G.MC, (int)t0, &full[s]);
            tma_load_3d(sbuf + R * G.MC * G.Np, &args.tmY, 0, c * G.MC, (int)t0, &full[s]);
          }
        } else {
          ws_issue(args.H, args.y, t0, Rv, G, c, stages + s * stage_elems, &full[s], pl, pn);
        }
      };
      fence_proxy_async();
      // ring position: stage index, parity of the stage's previous use, and
      // the (group, pass, chunk) counters advance together
      int ps = 0, pc = 0, pp = 0, pj = 0;
      uint32_t pph = 1;  // parity of use (gc / S) - 1
#pragma unroll 1
      for (long gc = 0; gc < total; ++gc) {
        if (gc >= G.S) FPM_PWAIT(&empty[ps], pph);
        diag_jitter(args.debug, 1, (int)gc);
        issue(pj, pc, ps);
        if (++ps == G.S) {
          ps = 0;
          pph ^= 1u;
        }
        if (++pc == nch) {
          pc = 0;
          if (++pp == npass) {
            pp = 0;
            ++pj;
          }
        }
      }
    }
    } else if (G32 && tid >= gt + 32 + ct && tid < gt + 64 + ct) {
    // ===================== converter warp (G32 only) ======================
    // the warp past the CG group: each landed stage (binary64 from TMA) is
    // converted in place to binary32 for the Gram warps (conv[s]), in ring order
    const int lane = tid & 31;
    int cs = 0;
    uint32_t cph = 0;
#pragma unroll 1
    for (long gc = 0; gc < total; ++gc) {
      const int s = cs;
      FPM_G32WAIT(&full[s], cph);
      if (++cs == G.S) {
        cs = 0;
        cph ^= 1u;
      }
      double2* sbuf = stages + s * stage_elems;
      g32_convert(sbuf, R * G.MC * Np, lane);
      g32_convert(sbuf + R * G.MC * Np, R * G.MC, lane);
      fence_proxy_async();  // these generic-proxy writes precede the next TMA into the stage
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[s]);
    }
    } else if (!kCgOwn && !SW && tid >= cbase && tid < cbase + ct && !args.gram_A) {
#include "fpm_detect_ws_cgrole.cuh"
    }
  }
  if constexpr (TA) tmx_fence_before();
  __syncthreads();
  if (tid < FPM_NCOUNTERS && cnt[tid]) atomicAdd(&args.counters[tid], cnt[tid]);
  if constexpr (TA) {
    if (tid < 32) {
      tmx_fence_after();
      tmx_dealloc(tm_base, 512);
    }
  }
}

#ifndef FPM_WS_GRAM_REGS_WIDE  // 16-byte matvec terms (fp64 / generic): the CG side needs more
#define FPM_WS_GRAM_REGS_WIDE 136  // measured: c5 fp64 3.57 M (176) -> 3.95 M det/s
#endif
#ifndef FPM_WS_GRAM_REGS
#define FPM_WS_GRAM_REGS 176
#endif
#ifndef FPM_WS_GRAM_REGS_1WG  // one Gram warp group (c1: N = 16, R = 16): 216 + 3 x 96
#define FPM_WS_GRAM_REGS_1WG 216  // measured c1: 184 0.315, 200 0.354, 216 0.363, 232 0.358 of FP64
#endif
#ifndef FPM_WS_GRAM_REGS_NB8  // N = 32: two matched-filter chains per Gram thread
#define FPM_WS_GRAM_REGS_NB8 184  // measured c2: 176 0.610, 184 0.618, 192 0.581 of FP64
#endif

template <int WK, int K, int NB, int LB>
int launch_detect_ws_t(const DetectArgs& a, const WsLayout& sl, int grid, cudaStream_t st) {
  DetectArgs b = a;
  b.ws_order = env_order(a.ws_order);
  const int threads = a.ws_gt + 32 + a.ws_ct;
  if constexpr (K == FK_F64 && (NB == 16 || NB == 4)) {
    if (a.ws_tmem) {  // fp64 A in tensor memory: two Gram warp groups, Gram-first order
      if (a.ws_gt != 256 || a.ws_ncg != 1 || a.ws_nslot != 2 || threads > 512) return FPM_EUNSUPPORTED;
      if (threads < 512) b.ws_order = 0;
      auto k = fpm_detect_ws_kernel<WK, K, NB, LB, FPM_WS_GRAM_REGS_WIDE, 2, 0, 1>;
      if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes) != cudaSuccess)
        return FPM_ECUDA;
      k<<<(unsigned)grid, 512, a.smem_bytes, st>>>(b, sl);
      count_launch();
      return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
    }
  }
  if (a.ws_tmem) return FPM_EUNSUPPORTED;
  if constexpr (NB == 32 && K != FK_F64 && K != FK_GEN) {
    if (a.gram32) {  // binary32 Gram (FP32-Gram extension): N = 128, two passes of 256 Gram threads
      if (a.ws_gt != 256 || a.ws_ncg != 1 || threads > 480) return FPM_EUNSUPPORTED;  // + the converter warp
      b.ws_order = 0;
      auto k = fpm_detect_ws_kernel<WK, K, NB, LB, FPM_WS_GRAM_REGS, 2, 1>;
      if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes) != cudaSuccess)
        return FPM_ECUDA;
      k<<<(unsigned)grid, 512, a.smem_bytes, st>>>(b, sl);
      count_launch();
      return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
    }
  }
  if (a.gram32) return FPM_EUNSUPPORTED;
  if constexpr (WK == FK_F64 && (K == FK_F16 || K == FK_BF16) && ((NB == 16 && LB == 4) || (NB == 8 && LB == 0))) {
    if (a.ws_sw) {  // solver warps on the CG side (fpm_detect_sw.cuh)
      if (a.ws_gt != 256 || a.ws_ct != 128) return FPM_EUNSUPPORTED;
      constexpr int kRS = NB == 8 ? FPM_WS_GRAM_REGS_NB8 : FPM_WS_GRAM_REGS;
      auto k = fpm_detect_ws_kernel<WK, K, NB, LB, kRS, 2, 0, 0, 1>;
      if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes) != cudaSuccess)
        return FPM_ECUDA;
      k<<<(unsigned)grid, 512, a.smem_bytes, st>>>(b, sl);
      count_launch();
      return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
    }
  }
  if (a.ws_sw) return FPM_EUNSUPPORTED;
  if constexpr (NB > 0) {
    // 256 Gram threads (N = 64: R = 2, N = 32: R = 8, N = 16: R = 32) = two
    // warp groups of a 512-thread block -> register split between the Gram
    // and the other warp groups
    if (a.ws_gt == 256 && threads <= 512 && !knob("FPM_WS_NOSPLIT")) {
      // a narrower CG group leaves idle warps in the upper warp groups (they
      // still take part in the register hand-over); CG-first order needs the
      // CG group to fill warp groups 0-1 so the Gram starts at warp group 2
      if (threads < 512) b.ws_order = 0;
      constexpr bool kSplit = FPM_CG_SPLIT && K == FK_F64 && NB == 16 && LB == 4;
      // the split instance's budgets add up only for a 128-thread CG group in warp group 3
      if (kSplit && (a.ws_ct != 128 || a.ws_ncg != 1)) return FPM_EUNSUPPORTED;
      constexpr int kRS = kSplit                             ? FPM_CG_SPLIT_GRAM_REGS
                          : sizeof(typename Ar<K>::C) >= 16 ? FPM_WS_GRAM_REGS_WIDE
                          : NB == 8                        ? FPM_WS_GRAM_REGS_NB8
                                                           : FPM_WS_GRAM_REGS;
      auto k = fpm_detect_ws_kernel<WK, K, NB, LB, kRS>;
      if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes) != cudaSuccess)
        return FPM_ECUDA;
      k<<<(unsigned)grid, 512, a.smem_bytes, st>>>(b, sl);
      count_launch();
      return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
    }
    // one Gram warp group (gt = 128) as the last warp group of a 512-thread
    // CG-first block (ct = 352): it takes 216 registers, the CG / producer
    // groups 96 (the 128-register default spills the pipelined tile loop)
    if constexpr (NB == 4) {
      if (a.ws_gt == 128 && threads == 512 && b.ws_order == 1 && !knob("FPM_WS_NOSPLIT")) {
        auto k = fpm_detect_ws_kernel<WK, K, NB, LB, FPM_WS_GRAM_REGS_1WG, 1>;
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes) != cudaSuccess)
          return FPM_ECUDA;
        k<<<(unsigned)grid, 512, a.smem_bytes, st>>>(b, sl);
        count_launch();
        return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
      }
    }
  }
  auto k = fpm_detect_ws_kernel<WK, K, NB, LB, 0>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes) != cudaSuccess)
    return FPM_ECUDA;
  k<<<(unsigned)grid, threads, a.smem_bytes, st>>>(b, sl);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? FPM_OK : FPM_ECUDA;
}

}  // namespace fpm
