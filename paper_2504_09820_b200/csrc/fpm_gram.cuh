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
//   * "circulant" jobs  c = (a+d) mod nb, d = 1..nb/2-1, and (a, a+nb/2)
//   * "diagonal" jobs   the two triangles S_k x S_k and S_{k+nb/2} x S_{k+nb/2}
// Both job kinds cost 128 DP ops per antenna row and load the same 8
// operands (S_a, S_c), every unordered pair {i,j} is produced exactly once,
// and lanes of an 8-thread LDS.128 phase touch consecutive residues, so the
// shared-memory reads are conflict-free.  R realizations per CTA make the
// diagonal jobs fill whole warps (R = 256/Np).
//
// Rows of H stream global -> shared through cp.async.bulk (TMA 1-D) into an
// S-stage ring; one DP op stream per thread, no tensor cores (tcgen05 has no
// f64 kind and DMMA fuses the multiply-add, so neither is bit-exact here).
#pragma once
#include "fpm_arith.cuh"
#include "fpm_ptx.cuh"

namespace fpm {

struct GramJob {
  int g;     // realization slot within the CTA, -1 = idle
  int diag;  // 0 = circulant 4x4 block, 1 = pair of diagonal triangles
  int a, c;  // residue classes
};

__device__ __forceinline__ GramJob gram_job(int t, int R, int nb) {
  GramJob j;
  const int half = nb >> 1;
  const int ncirc0 = nb * (half - 1);
  const int Cn = ncirc0 + half;
  if (t < R * Cn) {
    j.g = t / Cn;
    int q = t - j.g * Cn;
    j.diag = 0;
    if (q < ncirc0) {
      int d = 1 + q / nb;
      j.a = q % nb;
      j.c = (j.a + d) % nb;
    } else {
      j.a = q - ncirc0;
      j.c = j.a + half;
    }
  } else if (t < R * (Cn + half)) {
    int u = t - R * Cn;
    j.g = u / half;
    j.diag = 1;
    j.a = u - j.g * half;
    j.c = j.a + half;
  } else {
    j.g = -1;
    j.diag = 0;
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

struct GramGeom {
  int R;    // realization slots per CTA
  int M, N, Np, nb;
  int MC;   // antenna rows per stage
  int S;    // stages
};

// Issue the bulk copies of chunk `c` (rows c*MC ..) for every valid slot.
__device__ __forceinline__ void gram_issue(const double2* H, long t0, int Rv, const GramGeom& G,
                                           int chunk, double2* stage_buf, uint64_t* bar) {
  const int m0 = chunk * G.MC;
  const int rows = min(G.MC, G.M - m0);
  const uint32_t rowb = (uint32_t)G.N * 16u;
  mbar_expect_tx(bar, (uint32_t)Rv * (uint32_t)rows * rowb);
  for (int g = 0; g < Rv; ++g) {
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
// [t0, t0+Rv).  On return (after a __syncthreads), `emit` has received every
// final A entry (both triangles) and every b entry.
//   emit.a(g, i, j, value)   value already in its final (reference) bits
//   emit.b(g, n, value)
// bars: full[0..S-1], empty[S..2S-1], y-barrier [2S]; full/y count 1,
// empty count = warps per CTA.  Thread 0 is the (lagging) producer: before
// consuming chunk c it refills the stage chunk c-1 used once every warp has
// released it, so warps are never forced into lockstep.
template <class Emit>
__device__ void gram_run(const double2* __restrict__ H, const double2* __restrict__ y, long t0, int Rv,
                         const GramGeom& G, double sigma2, double2* stages, double2* ys, uint64_t* bars,
                         int nthreads, int tid, Emit& emit) {
  uint64_t* full = bars;
  uint64_t* empty = bars + G.S;
  uint64_t* ybar = bars + 2 * G.S;
  const int nchunks = (G.M + G.MC - 1) / G.MC;
  const long stage_elems = (long)G.R * G.MC * G.Np;
  if (tid == 0) {
    fence_proxy_async();  // stage memory may have been written by generic stores before
    mbar_expect_tx(ybar, (uint32_t)Rv * (uint32_t)G.M * 16u);
    for (int g = 0; g < Rv; ++g) bulk_g2s(ys + (long)g * G.M, y + (t0 + g) * (long)G.M, G.M * 16u, ybar);
    for (int c = 0; c < G.S && c < nchunks; ++c) gram_issue(H, t0, Rv, G, c, stages + c * stage_elems, &full[c]);
  }
  const GramJob job = gram_job(tid, G.R, G.nb);
  const bool active = job.g >= 0 && job.g < Rv;

  double2 acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = make_double2(0.0, 0.0);

  // matched-filter chains: pairs (g, n) strided over the CTA
  const int npairs = Rv * G.N;
  double2 bacc[4];
  int bg[4], bn[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    bacc[k] = make_double2(0.0, 0.0);
    int q = tid + k * nthreads;
    bg[k] = q < npairs ? q / G.N : -1;
    bn[k] = q < npairs ? q % G.N : 0;
  }

  mbar_wait(ybar, 0);
  const int nb = G.nb;
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % G.S;
    if (tid == 0 && c >= 1 && c - 1 + G.S < nchunks) {
      const int ps = (c - 1) % G.S;
      mbar_wait(&empty[ps], (uint32_t)(((c - 1) / G.S) & 1));
      gram_issue(H, t0, Rv, G, c - 1 + G.S, stages + ps * stage_elems, &full[ps]);
    }
    mbar_wait(&full[s], (uint32_t)((c / G.S) & 1));
    const double2* sb = stages + s * stage_elems;
    const int m0 = c * G.MC;
    const int rows = min(G.MC, G.M - m0);
    if (active) {
      const double2* base = sb + (long)job.g * G.MC * G.Np;
      if (!job.diag) {
        for (int mm = 0; mm < rows; ++mm) {
          const double2* row = base + mm * G.Np;
          double2 hi[4], hj[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) hi[u] = row[job.a + nb * u];
#pragma unroll
          for (int v = 0; v < 4; ++v) hj[v] = row[job.c + nb * v];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) cmac_conj(acc[u * 4 + v], hi[u], hj[v]);
        }
      } else {
        for (int mm = 0; mm < rows; ++mm) {
          const double2* row = base + mm * G.Np;
          double2 ha[4], hc[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) ha[u] = row[job.a + nb * u];
#pragma unroll
          for (int v = 0; v < 4; ++v) hc[v] = row[job.c + nb * v];
          int p = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = u + 1; v < 4; ++v) {
              cmac_conj(acc[p], ha[u], ha[v]);
              cmac_conj(acc[6 + p], hc[u], hc[v]);
              ++p;
            }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            acc[12 + u].x = __dadd_rn(acc[12 + u].x, sqmag(ha[u]));
            acc[12 + u].y = __dadd_rn(acc[12 + u].y, sqmag(hc[u]));
          }
        }
      }
    }
    // matched filter b = sum_m conj(h_m,n) y_m
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (bg[k] >= 0) {
        const double2* col = sb + (long)bg[k] * G.MC * G.Np + bn[k];
        const double2* yy = ys + (long)bg[k] * G.M + m0;
        for (int mm = 0; mm < rows; ++mm) {
          double2 h = col[mm * G.Np];
          double2 yv = yy[mm];
          bacc[k].x = __dadd_rn(bacc[k].x, __dadd_rn(__dmul_rn(h.x, yv.x), __dmul_rn(h.y, yv.y)));
          bacc[k].y = __dadd_rn(bacc[k].y, __dsub_rn(__dmul_rn(h.x, yv.y), __dmul_rn(h.y, yv.x)));
        }
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
  }
  __syncthreads();  // every warp is past the last stage before the epilogue reuses it

  // ---- epilogue: final reference bits for both triangles ----
  if (active) {
    const int g = job.g;
    if (!job.diag) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          int i = job.a + nb * u, j = job.c + nb * v;
          if (i < G.N && j < G.N) {
            double2 Gv = acc[u * 4 + v];
            emit.a(g, i, j, make_double2(__dadd_rn(Gv.x, 0.0), __dadd_rn(Gv.y, 0.0)));
            emit.a(g, j, i, make_double2(__dadd_rn(Gv.x, 0.0), __dsub_rn(0.0, Gv.y)));
          }
        }
    } else {
      int p = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = u + 1; v < 4; ++v) {
#pragma unroll
          for (int side = 0; side < 2; ++side) {
            int r0 = side ? job.c : job.a;
            int i = r0 + nb * u, j = r0 + nb * v;
            if (i < G.N && j < G.N) {
              double2 Gv = acc[side * 6 + p];
              emit.a(g, i, j, make_double2(__dadd_rn(Gv.x, 0.0), __dadd_rn(Gv.y, 0.0)));
              emit.a(g, j, i, make_double2(__dadd_rn(Gv.x, 0.0), __dsub_rn(0.0, Gv.y)));
            }
          }
          ++p;
        }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int i0 = job.a + nb * u, i1 = job.c + nb * u;
        if (i0 < G.N) emit.a(g, i0, i0, make_double2(__dadd_rn(acc[12 + u].x, sigma2), 0.0));
        if (i1 < G.N) emit.a(g, i1, i1, make_double2(__dadd_rn(acc[12 + u].y, sigma2), 0.0));
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (bg[k] >= 0) emit.b(bg[k], bn[k], bacc[k]);
  __syncthreads();
}

}  // namespace fpm
