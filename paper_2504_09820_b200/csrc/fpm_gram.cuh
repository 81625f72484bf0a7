// Gram / matched filter, bit-exact with the reference's einsum
// (detect.py:215-218):  A = H^H H (+symmetrize) + sigma^2 I,  b = H^H y.
//
// Arithmetic contract (verified against the reference, tests/golden):
//   per output entry, acc = +0; for m = 0..M-1 in order:
//     acc.re += fl(fl(hr_i*hr_j) + fl(hi_i*hi_j))
//     acc.im += fl(fl(hr_i*hi_j) - fl(hi_i*hr_j))
//   no FMA (DMMA/DFMA would change the bits), no reordering of m.
//   final(i,j) = (G.re + (i==j ? sigma^2 : 0.0), G.im + 0.0),
//   final(j,i) = (G.re + 0.0, 0.0 - G.im)   [what 0.5(A+A^H) + s2 I yields].
//
// Work decomposition (B200): the index set 0..Np-1 (Np = N rounded up to a
// multiple of 8, nb = Np/4) is split into nb residue classes
// S_a = {a, a+nb, a+2nb, a+3nb}.  One thread owns one 4x4 block S_a x S_c of
// the Gram (16 complex accumulators in registers):
//   * "circulant" jobs  c = (a+d) mod nb, d = 1..nb/2-1
//   * "half-pair" jobs  one diagonal triangle + half of a cross block
//     (see gram_job)
// Both job kinds cost 128 DP ops per antenna row, every unordered pair {i,j}
// is produced exactly once, and lanes of an 8-thread LDS.128 phase touch
// consecutive residues, so the shared-memory reads are conflict-free.  The
// inner loop sustains 98% of the measured non-fused FP64 rate on its own
// (tools/gram_variants.cu).
//
// The matched-filter chains b_n ride in the same row loop (their latency
// hides under the tile math).  Rows of H stream global -> shared through
// cp.async.bulk (TMA 1-D) into an S-stage full/empty mbarrier ring; no tensor
// cores: tcgen05 has no f64 kind and DMMA fuses the multiply-add.
#pragma once
#include "fpm_arith.cuh"
#include "fpm_ptx.cuh"

#ifndef FPM_ROW_UNROLL_N
#define FPM_ROW_UNROLL_N 1
#endif
#define FPM_PRAGMA_(x) _Pragma(#x)
#define FPM_UNROLL_(n) FPM_PRAGMA_(unroll n)
#define FPM_ROW_UNROLL FPM_UNROLL_(FPM_ROW_UNROLL_N)

namespace fpm {

struct GramJob {
  int g;     // realization slot within the CTA, -1 = idle
  int half;  // 0 = circulant 4x4 block S_a x S_c; 1 = half of a diagonal pair
  int a, c;  // circulant: residues of the row / column sets.  half: X = S_a, Z = S_c
  int y, yo; // half: Y = (S_y[yo], S_y[yo+1])
};

// Jobs of one realization: nb*(nb/2-1) circulant blocks (a, (a+d) mod nb),
// d = 1..nb/2-1, then nb "half-pair" jobs covering, for each pair
// (k, k+nb/2), the two diagonal triangles and the cross block S_k x S_{k+nb/2}:
//   side 0: tri(S_k)        + rows S_k[0..1] x S_{k+nb/2}
//   side 1: tri(S_{k+nb/2}) + rows S_k[2..3] x S_{k+nb/2}
// Both job kinds are 128 DP ops per row with one instruction stream each; all
// circulant jobs of the CTA come first, so with R*nb*(nb/2-1) % 32 == 0 every
// warp is uniform (R=2 for N=64, R=1 for N=128, R=4 for N=32, R=8 for N=16).
__device__ __forceinline__ GramJob gram_job(int t, int R, int nb) {
  GramJob j;
  const int hp = nb >> 1;
  const int Cc = nb * (hp - 1);
  j.y = 0;
  j.yo = 0;
  if (t < R * Cc) {
    j.g = t / Cc;
    const int q = t - j.g * Cc;
    j.half = 0;
    const int d = 1 + q / nb;
    j.a = q % nb;
    j.c = (j.a + d) % nb;
  } else if (t < R * (Cc + nb)) {
    const int u = t - R * Cc;
    j.g = u / nb;
    const int rem = u - j.g * nb;
    const int side = rem / hp, k = rem - side * hp;
    j.half = 1;
    j.a = side ? k + hp : k;  // X (triangle set)
    j.c = k + hp;             // Z (cross columns)
    j.y = k;                  // Y rows from S_k
    j.yo = side ? 2 : 0;
  } else {
    j.g = -1;
    j.half = 0;
    j.a = j.c = 0;
  }
  return j;
}

__device__ __forceinline__ void cmac_conj(double2& acc, double2 hi, double2 hj) {
  double pr = __dadd_rn(__dmul_rn(hi.x, hj.x), __dmul_rn(hi.y, hj.y));
  double pi = __dsub_rn(__dmul_rn(hi.x, hj.y), __dmul_rn(hi.y, hj.x));
  acc.x = __dadd_rn(acc.x, pr);
  acc.y = __dadd_rn(acc.y, pi);
}

__device__ __forceinline__ double sqmag(double2 h) {
  return __dadd_rn(__dmul_rn(h.x, h.x), __dmul_rn(h.y, h.y));
}

// final reference bits of an accumulated Gram entry and of its mirror
__device__ __forceinline__ double2 gram_final(double2 G) {
  return make_double2(__dadd_rn(G.x, 0.0), __dadd_rn(G.y, 0.0));
}
__device__ __forceinline__ double2 gram_mirror(double2 G) {
  return make_double2(__dadd_rn(G.x, 0.0), __dsub_rn(0.0, G.y));
}

struct GramGeom {
  int R;    // realization slots per CTA
  int M, N, Np, nb;
  int MC;   // antenna rows per stage
  int S;    // stages
};

// Issue the bulk copies of chunk `c` (rows c*MC ..) for every valid slot.
// lane / nlanes: the copies of one stage are issued by nlanes threads of one
// warp (the realizations' row blocks are separate bulk copies); lane 0 posts
// the stage's expected bytes first.  nlanes > 1 must be a whole warp.
__device__ __forceinline__ void gram_issue(const double2* H, long t0, int Rv, const GramGeom& G,
                                           int chunk, double2* stage_buf, uint64_t* bar, int lane = 0,
                                           int nlanes = 1) {
  const int m0 = chunk * G.MC;
  const int rows = min(G.MC, G.M - m0);
  const uint32_t rowb = (uint32_t)G.N * 16u;
  if (lane == 0) mbar_expect_tx(bar, (uint32_t)Rv * (uint32_t)rows * rowb);
  if (nlanes > 1) __syncwarp();
  for (int g = lane; g < Rv; g += nlanes) {
    const double2* src = H + ((t0 + g) * (long)G.M + m0) * (long)G.N;
    double2* dst = stage_buf + (long)g * G.MC * G.Np;
    if (G.N == G.Np) {
      bulk_g2s(dst, src, rows * rowb, bar);
    } else {
      for (int r = 0; r < rows; ++r) bulk_g2s(dst + r * G.Np, src + (long)r * G.N, rowb, bar);
    }
  }
}

// Runs the whole Gram + matched filter for the CTA's realizations
// [t0, t0+Rv), then (after a __syncthreads) hands every thread's finished
// job to emit.job(job, acc) and every matched-filter entry to emit.b(g, n, v);
// returns after a final __syncthreads.  NB > 0 fixes nb at compile time.
// bars: full[0..S-1], empty[S..2S-1], y-barrier [2S]; full/y count 1,
// empty count = warps per CTA.  Thread 0 is the (lagging) producer: before
// consuming chunk c it refills the stage chunk c-1 used once every warp has
// released it, so warps are never forced into lockstep.
template <int NB, class Emit>
__device__ void gram_run(const double2* __restrict__ H, const double2* __restrict__ y, long t0, int Rv,
                         const GramGeom& G, double2* stages, double2* ys, uint64_t* bars, int nthreads, int tid,
                         Emit& emit, long long* tr = nullptr) {
  uint64_t* full = bars;
  uint64_t* empty = bars + G.S;
  uint64_t* ybar = bars + 2 * G.S;
  const int nb = NB > 0 ? NB : G.nb;
  const int Np = NB > 0 ? 4 * NB : G.Np;
  const int nchunks = (G.M + G.MC - 1) / G.MC;
  const int stage_elems = G.R * G.MC * Np;
  if (tid == 0) {
    fence_proxy_async();  // stage memory may have been written by generic stores before
    mbar_expect_tx(ybar, (uint32_t)Rv * (uint32_t)G.M * 16u);
    for (int g = 0; g < Rv; ++g) bulk_g2s(ys + (long)g * G.M, y + (t0 + g) * (long)G.M, G.M * 16u, ybar);
    for (int c = 0; c < G.S && c < nchunks; ++c) gram_issue(H, t0, Rv, G, c, stages + c * stage_elems, &full[c]);
  }
  const GramJob job = gram_job(tid, G.R, nb);
  const bool active = job.g >= 0 && job.g < Rv;

  double2 acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = make_double2(0.0, 0.0);

  // Matched-filter chains, split into independent real / imaginary
  // accumulators (b.re and b.im are separate sequential sums in the
  // reference, so the split is exact): chain q in [0, 2*Rv*N) -> realization
  // g, entry n, part (0 re / 1 im).  With R*2N == threads (the planned
  // geometry) every thread carries exactly one chain, branch-free:
  //   re += fl(fl(hr*yr) + fl(hi*yi)),  im += fl(fl(hr*yi) + fl(hi*(-yr)))
  const int nch = 2 * Rv * G.N;
  const int nbc = nch > tid ? min(4, (nch - tid + nthreads - 1) / nthreads) : 0;
  double bacc[4];
  int boff[4], yoff[4], bim[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    bacc[k] = 0.0;
    const int q = min(tid + k * nthreads, nch - 1);
    const int g = q / (2 * G.N), e = q - g * 2 * G.N;
    const int part = e / G.N, n = e - part * G.N;
    boff[k] = g * G.MC * Np + n;
    yoff[k] = g * G.M;
    bim[k] = part;
  }

  mbar_wait(ybar, 0);
  const int joff = job.g * G.MC * Np;
  long long t_empty = 0, t_full = 0;
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % G.S;
    if (tid == 0 && c >= 1 && c - 1 + G.S < nchunks) {
      const int ps = (c - 1) % G.S;
      const long long w0 = tr ? clock64() : 0;
      mbar_wait(&empty[ps], (uint32_t)(((c - 1) / G.S) & 1));
      if (tr) t_empty += clock64() - w0;
      gram_issue(H, t0, Rv, G, c - 1 + G.S, stages + ps * stage_elems, &full[ps]);
    }
    const long long f0 = tr ? clock64() : 0;
    mbar_wait(&full[s], (uint32_t)((c / G.S) & 1));
    if (tr) t_full += clock64() - f0;
    const double2* sb = stages + s * stage_elems;
    const int m0 = c * G.MC;
    const int rows = min(G.MC, G.M - m0);
    const double2* pa = sb + joff + job.a;
    const double2* pc = sb + joff + job.c;
    if (active && !job.half) {
FPM_ROW_UNROLL
      for (int mm = 0; mm < rows; ++mm) {
        double2 hi[4], hj[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) hi[u] = pa[mm * Np + nb * u];
#pragma unroll
        for (int v = 0; v < 4; ++v) hj[v] = pc[mm * Np + nb * v];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) cmac_conj(acc[u * 4 + v], hi[u], hj[v]);
      }
    } else if (active) {
      const double2* py = sb + joff + job.y + nb * job.yo;
FPM_ROW_UNROLL
      for (int mm = 0; mm < rows; ++mm) {
        double2 hx[4], hy[2], hz[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) hx[u] = pa[mm * Np + nb * u];
#pragma unroll
        for (int w = 0; w < 2; ++w) hy[w] = py[mm * Np + nb * w];
#pragma unroll
        for (int v = 0; v < 4; ++v) hz[v] = pc[mm * Np + nb * v];
        int p = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = u + 1; v < 4; ++v) cmac_conj(acc[p++], hx[u], hx[v]);
#pragma unroll
        for (int w = 0; w < 2; ++w)
#pragma unroll
          for (int v = 0; v < 4; ++v) cmac_conj(acc[6 + w * 4 + v], hy[w], hz[v]);
        acc[14].x = __dadd_rn(acc[14].x, sqmag(hx[0]));
        acc[14].y = __dadd_rn(acc[14].y, sqmag(hx[1]));
        acc[15].x = __dadd_rn(acc[15].x, sqmag(hx[2]));
        acc[15].y = __dadd_rn(acc[15].y, sqmag(hx[3]));
      }
    }
    // matched-filter chains (separate pass over the stage: keeps the tile
    // loop branch-free; the chains' latency overlaps other warps' tiles)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < nbc) {
        const double2* hcol = sb + boff[k];
        const double2* yy = ys + yoff[k] + m0;
        const bool im = bim[k];
        double a = bacc[k];
#pragma unroll 2
        for (int mm = 0; mm < rows; ++mm) {
          const double2 h = hcol[mm * Np];
          const double2 yv = yy[mm];
          const double y1 = im ? yv.y : yv.x, y2 = im ? -yv.x : yv.y;
          a = __dadd_rn(a, __dadd_rn(__dmul_rn(h.x, y1), __dmul_rn(h.y, y2)));
        }
        bacc[k] = a;
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
  }
  if (tr && (tid & 31) == 0) {
    tr[8 + tid / 32] = clock64();      // per-warp main-loop finish
    if (tid == 0) { tr[5] = t_empty; tr[6] = t_full; }
    if (tid == 32) tr[7] = t_full;
  }
  __syncthreads();  // every warp is past the last stage before the epilogue reuses it
  if (tr && tid == 0) {
    __shared__ int _fpm_g_dummy;
    tr[0] = (long long)clock64() + (*(volatile int*)&_fpm_g_dummy == 0x7fffffff);
  }

  if (active) emit.job(job, acc, nb);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < nbc) {
      const int q = tid + k * nthreads;
      const int g = q / (2 * G.N), e = q - g * 2 * G.N;
      const int part = e / G.N;
      emit.b(g, e - part * G.N, part, bacc[k]);
    }
  }
  __syncthreads();
}

// Iterate the final entries of a finished job: f(i, j, value_ij, mirror_ji)
// for i != j (both orientations' bits), d(i, value_ii) for diagonal entries.
template <class F, class D>
__device__ __forceinline__ void gram_entries(const GramJob& job, const double2 (&acc)[16], int nb, int N,
                                             double sigma2, F&& f, D&& d, int sp = 0) {
  // sp = 1: the job's circulant rows / columns and its cross-block rows and
  // columns were accumulated in pair-swapped order (u ^ 1; see the
  // warp-specialised kernel's bank-conflict note at nb = 4)
  if (!job.half) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = job.a + nb * (u ^ sp), j = job.c + nb * (v ^ sp);
        if (i < N && j < N) f(i, j, gram_final(acc[u * 4 + v]), gram_mirror(acc[u * 4 + v]));
      }
  } else {
    int p = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = u + 1; v < 4; ++v) {
        const int i = job.a + nb * u, j = job.a + nb * v;
        if (i < N && j < N) f(i, j, gram_final(acc[p]), gram_mirror(acc[p]));
        ++p;
      }
#pragma unroll
    for (int w = 0; w < 2; ++w)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = job.y + nb * (job.yo + (w ^ sp)), j = job.c + nb * (v ^ sp);
        if (i < N && j < N) f(i, j, gram_final(acc[6 + w * 4 + v]), gram_mirror(acc[6 + w * 4 + v]));
      }
    const double dg[4] = {acc[14].x, acc[14].y, acc[15].x, acc[15].y};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = job.a + nb * u;
      if (i < N) d(i, make_double2(__dadd_rn(dg[u], sigma2), 0.0));
    }
  }
}

}  // namespace fpm
