// The CG warps' role of fpm_detect_ws_kernel (textually included at its call
// sites in fpm_detect_ws.cuh: the role is a top-level branch of its own when
// the CG warp group runs at its own register budget, FPM_CG_SPLIT).
// NOT a standalone header: uses the kernel's locals.
    // ============================ CG warps ============================
    // ws_ncg CG groups; group cgi owns hand-off slot cgi, i.e. realization
    // groups j = cgi, cgi + ncg, ... (two latency-bound solves in flight)
    const int ncg = args.ws_ncg;
    const int cgi = (ncg == 2 && tid - cbase >= args.ws_ct0) ? 1 : 0;
    const int lt = tid - cbase - (cgi ? args.ws_ct0 : 0);
    const int ctg = ncg == 2 ? (cgi ? ct - args.ws_ct0 : args.ws_ct0) : ct;
    unsigned char* cgs = smem + cgi * args.cg_stride;  // this group's CG state
    NamedBar cbar{2 + cgi, ctg};
    CgSmem<K> S;
    S.R = R;
    S.N = N;
    S.L = L;
    S.ldA = ldA;
    S.minv = reinterpret_cast<double2*>(cgs + args.off_minv);
    S.dbg = diag_bits(args.debug);
    double2* vec = reinterpret_cast<double2*>(cgs + args.off_vec);
    const int RN = R * N;
    // z only with block-Jacobi, the rho0 terms only for BJ as_written: they
    // come last so the planner can leave them out (ws_cg_layout)
    S.x = vec;
    S.r = vec + RN;
    S.p = vec + 2 * RN;
    S.w = vec + 3 * RN;
    S.xn = vec + 4 * RN;
    S.rn = vec + 5 * RN;
    S.z = vec + 6 * RN;
    S.pmv = reinterpret_cast<P*>(cgs + args.off_pmv);
    S.tphi = reinterpret_cast<C*>(cgs + args.off_tip);
    S.tr1 = S.tphi + RN;
    S.rip = S.tr1 + RN;
    S.trho = S.rip + RN;
    S.sc = reinterpret_cast<double2*>(cgs + args.off_sc);
    S.fl = reinterpret_cast<int*>(cgs + args.off_fl);
    double2* scr2 = reinterpret_cast<double2*>(cgs + args.off_scr2);
    const int bps = 2 * args.sl.bpa;
    unsigned long long be = 0, se = 0;
#pragma unroll 1
    for (int j = cgi; j < my_groups; j += ncg) {
      const long t0 = ((long)blockIdx.x + (long)j * gridDim.x) * R;
      const int Rv = (int)min((long)R, args.T - t0);
      const int slot = nsl == 2 ? (j & 1) : 0;
      const int use = nsl == 2 ? (j >> 1) : j;
      unsigned char* sp = slots + slot * sl.bytes;
      S.At = reinterpret_cast<C*>(sp + sl.at);
      S.b = reinterpret_cast<double2*>(sp + sl.b);
      double2* dS = reinterpret_cast<double2*>(sp + sl.d);
      FPM_CWAIT(&sfull[slot], (uint32_t)(use & 1));
      if constexpr (TA) tmx_fence_after();
      diag_jitter(args.debug, 6, j);
      if (tr && lt == 0 && j < 8) tr[j * 8 + 4] = clock64();
#pragma unroll 1
      for (int g = lt; g < R; g += ctg) S.fl[g * 4] = g < Rv ? 1 : 0;
      cbar.sync();
      // block-Jacobi inverses (on-chip fp64 Cholesky, or injected)
      if (args.bj) {
        if (args.minv_in) {
#pragma unroll 1
          for (int q = lt; q < Rv * N * L; q += ctg) {
            const int g = q / (N * L);
            const int e = q - g * N * L;
            const int kb = e / (L * L), o = e - kb * L * L;
            const int Lk = min(L, N - kb * L);
            if (o >= Lk * Lk) continue;
            const int i = o / Lk, jj = o - i * Lk;
            S.minv[g * N * L + kb * L * L + jj * Lk + i] =
                Ar<WK>::rnd(args.minv_in[(t0 + g) * (long)N * L + e], args.pr.work);
          }
        } else {
          const int nbt = R * nblk;
#pragma unroll 1
          for (int q = lt; q < Rv * nblk; q += ctg) {
            const int g = q / nblk, kb = q - g * nblk;
            const int Lk = min(L, N - kb * L);
            double2* out = S.minv + g * N * L + kb * L * L;
            const bool ok = (diag_bits(args.debug) & 32) ? true : (LB > 0) ? hpd_inverse<LB>(dS + q, nbt, scr2 + q, nbt, out, Lk)
                                     : hpd_inverse<0>(dS + q, nbt, scr2 + q, nbt, out, Lk);
            if (!ok) {
              atomicExch(&S.fl[g * 4], 0);
              atomicAdd(&cnt[FPM_CNT_NONPD], 1ULL);
            } else if (WK != FK_F64) {
              for (int e = 0; e < Lk * Lk; ++e) out[e] = Ar<WK>::rnd(out[e], args.pr.work);
            }
          }
        }
        cbar.sync();
      }
      long long* tc = (tr && j == 2 && args.iters <= 8) ? tr + 96 : nullptr;  // CG phase stamps, group 2
      if (tc && lt == 0) {
        __shared__ int _fpm_dummy_ws;
        tc[60] = (long long)clock64() + (*(volatile int*)&_fpm_dummy_ws == 0x7fffffff);
      }
      if (!(diag_bits(args.debug) & 1))
        cg_group<WK, K, LB, kCgNC, TA != 0>(S, Rv, args.iters, args.bj != 0, args.textbook != 0, args.pr, ctg, lt, cbar,
                                            tc, TmRows{tm_base + (uint32_t)(slot * 256), cbase / 32, ctg / 32});
      // slot no longer needed (A, b, diagonal blocks consumed)
      diag_jitter(args.debug, 7, j);
      if (lt == 0) mbar_arrive(&sempty[slot]);
      if (tr && lt == 0 && j < 8) tr[j * 8 + 5] = clock64();
      // slicer + counters + write-back
#pragma unroll 1
      for (int q = lt; q < Rv * N; q += ctg) {
        const long gq = t0 * N + q;
        const double2 xv = S.x[q];
        args.x[gq] = xv;
        int sym;
        be += slice_one(xv, args.tx ? args.tx + gq * bps : nullptr, args.rx ? args.rx + gq * bps : nullptr,
                        args.sl, &sym);
        se += sym;
      }
#pragma unroll 1
      for (int g = lt; g < Rv; g += ctg) {
        const int bk = S.fl[g * 4 + 2], dv = S.fl[g * 4 + 3];
        args.brk[t0 + g] = bk;
        args.div[t0 + g] = dv;
        if (dv >= 0) atomicAdd(&cnt[FPM_CNT_DIVERGED], 1ULL);
        if (bk >= 0) atomicAdd(&cnt[FPM_CNT_BREAKDOWN], 1ULL);
      }
      if (lt == 0) atomicAdd(&cnt[FPM_CNT_TRIALS], (unsigned long long)Rv);
      cbar.sync();  // x / flags read before the next group overwrites them
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      be += __shfl_xor_sync(0xffffffffu, be, off);
      se += __shfl_xor_sync(0xffffffffu, se, off);
    }
    if ((lt & 31) == 0) {
      if (be) atomicAdd(&cnt[FPM_CNT_BIT_ERRORS], be);
      if (se) atomicAdd(&cnt[FPM_CNT_SYMBOL_ERRORS], se);
    }
