// Host/device shared argument blocks and the per-kind launcher interface.
// Each format kind's kernels live in their own translation unit
// (fpm_inst_<kind>.cu, compiled in parallel); fpm_host.cu plans and dispatches.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fpmimo_b200.h"
#include "fpm_arith.cuh"
#include "fpm_cg.cuh"
#include "fpm_gram.cuh"

namespace fpm {

struct Slicer {
  double th[7];
  int nth;  // 3 (16-QAM) or 7 (64-QAM)
  int bpa;  // bits per axis
};

// 128-byte opaque TMA descriptor (CUtensorMap layout; encoded on the host by
// cuTensorMapEncodeTiled, fpm_host.cu)
struct alignas(64) TmaDesc {
  unsigned long long w[16];
};

struct DetectArgs {
  // tensor maps of the WS kernel's stages (use_tma): H as (2N doubles, M, T)
  // with box (2N, MC, R), y as (2 doubles, M, T) with box (2, MC, R)
  TmaDesc tmH, tmY;
  int use_tma;
  const double2* H;
  const double2* y;
  const uint8_t* tx;
  long T;
  double sigma2;
  int L, iters, bj, textbook;
  int tl;  // CG team lanes per realization
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
  int off_ys, off_union, off_minv, off_scr, off_scr2, off_vec, off_pmv, off_tip, off_sc, off_fl;
  int smem_bytes;
  long long* trace;  // nullable: phase clock stamps of CTA 0 (diagnostic)
  // warp-specialised persistent kernel: Gram / CG thread counts, slots base
  int ws_gt, ws_ct, off_slot, off_bsm;
  int ws_order;  // 0: [Gram | producer | CG] threads, 1: [CG | producer | Gram]
  int ws_ncg, ws_ct0;  // CG groups (1 or 2) and the thread count of group 0
  int cg_stride;       // bytes between the two CG groups' state regions
  int ws_nslot;        // hand-off slots (2 double-buffered, 1 when two do not fit)
  int ws_npass;        // Gram passes per group (2 at N = 128: 512 jobs on 256 Gram threads)
  int ws_tmem;         // fp64 A of the hand-off in tensor memory (two TMEM slots), staged through off_stg
  int ws_rr, off_stg;  // rows per staging round, staging offset (pitch N + 1 double2)
  int ws_sw;           // CG side = four solver warps, one realization each (fpm_detect_sw.cuh); scratch at off_vec
  int debug;  // diagnostic bits (FPM_DEBUG): 1 = WS kernel skips the CG side
  int composed;  // no fused plan fits: fpm_gram -> fpm_bj_setup -> fpm_cg -> slicer
  int gram32;    // FPM_FLAG_GRAM_FP32: binary32 Gram (extension): fused WS kernel at N = 128, else composed
  unsigned long long g32_one, g32_pm;  // (1, 1), (1, -1) binary32 pairs, opaque run-time values (fpm_gram32.cuh)
  double2* gram_A;  // non-null: Gram-only mode of the WS kernel (fpm_gram): A, b to HBM
  double2* gram_b;
};

struct WsLayout;  // fpm_detect_ws.cuh

struct CgArgs {
  const double2* A;
  const double2* b;
  const double2* minv;
  long T;
  int N, L, iters, bj, textbook, R, ldA;
  int tl;  // CG team lanes per realization
  Prec pr;
  double2* x;
  int* brk;
  int* div;
  int off_minv, off_vec, off_pmv, off_tip, off_sc, off_fl;
  CgHist h;
  long long* trace;  // nullable: phase clock stamps of CTA 0 (diagnostic)
  // non-null: A already on the u_MV grid in global memory ((T, N, N), pitch
  // N, C layout) -- the matrix does not fit shared memory (16-byte matvec
  // terms at large N); rows are read through L2 every sweep
  const void* a_glob;
  int threads;  // block size (0: 256)
};

// Launchers (return FPM_* codes).  nb / lb: compile-time specialisation
// requested by the planner (0 = generic); a launcher falls back to its generic
// instance when it has no matching specialisation.
#define FPM_DECLARE_KIND(name)                                                                 \
  int launch_detect_##name(const DetectArgs& a, int threads, int nb, int lb, cudaStream_t st); \
  int launch_detect_ws_##name(const DetectArgs& a, const WsLayout& sl, int grid, int nb, int lb, \
                              cudaStream_t st);                                                \
  int launch_cg_##name(const CgArgs& a, int smem, int lb, cudaStream_t st);
FPM_DECLARE_KIND(f64)
FPM_DECLARE_KIND(f32)
FPM_DECLARE_KIND(f16)
FPM_DECLARE_KIND(bf16)
FPM_DECLARE_KIND(gen)    // W = fp64, MV/IP generic emulation
FPM_DECLARE_KIND(gen_w)  // everything generic (W != fp64)
#undef FPM_DECLARE_KIND

void count_launch();

// FPM_* planner knob from the load-time snapshot (fpm_host.cu), nullptr if unset
const char* knob(const char* name);

// warp-per-realization CG (fpm_cgw.cuh, one unit per kind: fpm_cgw_<kind>.cu);
// FPM_EUNSUPPORTED when it has no instance for the configuration
int launch_cgw_f64(const CgArgs& a, cudaStream_t st);
int launch_cgw_f32(const CgArgs& a, cudaStream_t st);
int launch_cgw_f16(const CgArgs& a, cudaStream_t st);
int launch_cgw_bf16(const CgArgs& a, cudaStream_t st);
inline int launch_cgw(int mv_kind, const CgArgs& a, cudaStream_t st) {
  switch (mv_kind) {
    case FK_F64: return launch_cgw_f64(a, st);
    case FK_F32: return launch_cgw_f32(a, st);
    case FK_F16: return launch_cgw_f16(a, st);
    case FK_BF16: return launch_cgw_bf16(a, st);
    default: return FPM_EUNSUPPORTED;
  }
}

// FP32-Gram extension (fpm_gram32.cu)
int launch_gram32(const double2* H, const double2* y, long T, int M, int N, double sigma2, double2* A, double2* b,
                  cudaStream_t st);

// A -> A rounded to a generic matvec format, C layout (global-A CG mode)
int launch_round_mv_gen(const double2* A, double2* out, long n, FmtP f, cudaStream_t st);

// LMMSE direct comparator (fpm_lmmse.cu): one CTA per realization
int launch_lmmse(const double2* A, const double2* b, long T, int N, double2* x, int* nonpd,
                 unsigned long long* nonpd64, cudaStream_t st);

}  // namespace fpm
