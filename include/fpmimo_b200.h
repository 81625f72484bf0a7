/*
 * fpmimo_b200 -- C ABI of the B200-native batched FP-CG / FP-BJ-CG detector.
 *
 * Drop-in boundary for the reference package `fpmimo` (pure Python/NumPy, no
 * FFI of its own).  Each entry point replaces the reference interface cited
 * beside it (paths relative to /root/reference/pkg/src/fpmimo/):
 *
 *   fpm_gram        <- Gram / matched filter inline in simulate_trials,
 *                      detect.py:215-218 (A = H^H H sym + s2 I, b = H^H y)
 *   fpm_bj_setup    <- build_blocks_batch, solvers.py:232-253
 *   fpm_cg          <- run_batch, solvers.py:262-393 (x, breakdown_at,
 *                      diverged_at)
 *   fpm_cg_ex       <- run_batch with the BatchResult histories,
 *                      solvers.py:188-204, 306-319, 371-393
 *   fpm_herm_norm2  <- np.linalg.norm(A, 2) of the convergence study,
 *                      experiments.py:246-256
 *   fpm_residual_gaps <- run_batch's record_gaps diagnostic,
 *                      solvers.py:289-294, 375-377
 *   fpm_lmmse       <- _solve_direct_batch, linalg.py:223-231 (the
 *                      detector "lmmse", detect.py:230-231)
 *   fpm_gen_trials  <- the draws of simulate_trials, detect.py:189-214,
 *                      channel.py:138-161, 206-219, rng.py:19-39
 *                      (distribution level, keyed per-trial streams)
 *   fpm_simulate    <- simulate_trials, detect.py:189-214 (whole link model:
 *                      colouring, QAM payload, y = H s + n; one kernel)
 *   fpm_gram32      <- EXTENSION: binary32 Gram (BASELINE config c4)
 *   fpm_slice_count <- demodulate_16qam + error sum, detect.py:78-84, :260-262
 *   fpm_detect      <- _detect_batch, detect.py:223-237, fused with the Gram
 *                      of simulate_trials and the slicer/counter of
 *                      run_ber_sweep (one kernel, A never leaves the SM)
 *   fpm_detect_host <- the same call on HOST buffers (chunked H2D / compute /
 *                      D2H pipeline on two streams)
 *
 * Conventions
 *   - complex128 arrays are interleaved (re, im) doubles, C-contiguous,
 *     exactly NumPy's layout: H (T, M, N), y (T, M), A (T, N, N), b/x (T, N).
 *     Device complex128 arrays must be 16-byte aligned (NumPy / torch
 *     allocations are); the device entry points return FPM_EINVAL otherwise
 *     (fpm_detect_host copies host arrays and accepts any alignment).
 *   - Block-Jacobi inverses ("Minv") are packed per realization with a fixed
 *     stride of N*L complex entries: block k (size Lk = min(L, N - kL)) is the
 *     row-major Lk x Lk matrix starting at entry k*L*L.
 *   - All pointers except in fpm_detect_host are DEVICE pointers owned by the
 *     caller; inputs are never modified (solvers.py:297-298).  `stream` is a
 *     cudaStream_t (NULL = legacy default stream).  Calls are asynchronous on
 *     `stream`, carry no global mutable state and are re-entrant.  (The
 *     only process-wide objects: an atomic launch counter, the FPM_* planner
 *     knobs read once when the library loads, and fpm_detect_host's per-device
 *     staging pool, created once.)
 *   - Return: FPM_OK, or an error code; precondition failures (the reference's
 *     ContractViolation, errors.py:4-9) are FPM_EINVAL / FPM_ENOTPD.
 *     Numerical failures are flags, not errors (solvers.py:302-303).
 *   - counters (int64[FPM_NCOUNTERS]) are ACCUMULATED into (zero them first).
 */
#ifndef FPMIMO_B200_H
#define FPMIMO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* FloatFormat (formats.py:51-98): significand bits incl. hidden bit,
 * exponent bits, subnormals.  binary16 = {11,5,1}, bfloat16 = {8,8,1},
 * binary32 = {24,8,1}, binary64 = {53,11,1}. */
typedef struct fpm_format {
  int32_t sig_bits;
  int32_t exp_bits;
  int32_t subnormals;
} fpm_format;

/* PrecisionConfig (solvers.py:56-85): work must be at least as fine as the
 * other two. */
typedef struct fpm_precision {
  fpm_format work;
  fpm_format matvec;
  fpm_format inner;
} fpm_precision;

enum {
  FPM_OK = 0,
  FPM_EINVAL = 1,      /* bad argument (ContractViolation) */
  FPM_ENOTPD = 2,      /* non-PD diagonal block (solvers.py:246-249) */
  FPM_ECUDA = 3,       /* CUDA runtime error */
  FPM_EUNSUPPORTED = 4 /* configuration outside this build's limits */
};

enum { FPM_RHO_AS_WRITTEN = 0, FPM_RHO_TEXTBOOK = 1 };

/* DetectorSpec.algorithm (detect.py:115); "cg" computes at fp64 throughout;
 * "lmmse" is the direct Cholesky comparator (detect.py:230-231) */
enum { FPM_ALG_LMMSE = 0, FPM_ALG_CG = 1, FPM_ALG_FP_CG = 2, FPM_ALG_FP_BJ_CG = 3 };

/* OR-ed into `algorithm`: FP32 Gram / matched filter (EXTENSION for
 * BASELINE config c4; the reference has no such knob): H, y rounded once to
 * binary32, every Gram / MF op in binary32, widened to the fp64 carriers. */
enum { FPM_FLAG_GRAM_FP32 = 0x100 };

enum {
  FPM_CNT_BIT_ERRORS = 0,
  FPM_CNT_SYMBOL_ERRORS = 1, /* extension: the reference counts bits only */
  FPM_CNT_DIVERGED = 2,
  FPM_CNT_BREAKDOWN = 3,
  FPM_CNT_TRIALS = 4,
  FPM_CNT_NONPD = 5,
  FPM_NCOUNTERS = 8
};

int fpm_version(void);
const char* fpm_strerror(int code);

/* Largest N / L / M this build accepts (N <= 128, L <= 16, M <= 4096). */
int fpm_limits(int32_t* max_n, int32_t* max_l, int32_t* max_m);

int fpm_gram(const double* H, const double* y, int64_t T, int32_t M, int32_t N, double sigma2,
             double* A, double* b, void* stream);

/* FP32-Gram extension of fpm_gram (see FPM_FLAG_GRAM_FP32); same layouts. */
int fpm_gram32(const double* H, const double* y, int64_t T, int32_t M, int32_t N, double sigma2, double* A,
               double* b, void* stream);

/* bad_block: optional int32[T], set to the first non-PD block start or -1.
 * Returns FPM_ENOTPD if any block of any realization is not PD. */
int fpm_bj_setup(const double* A, int64_t T, int32_t N, int32_t L, int32_t allow_ragged, double* Minv,
                 int32_t* bad_block, void* stream);

/* Minv == NULL -> plain FP-CG, else FP-BJ-CG with block size L.  Minv is
 * (T, N*L) complex128: block k row-major at k*L*L (solvers.py:207-229
 * _BatchBlocks.mats packed).  Kernel: one warp per realization
 * (fpm_cgw_kernel) for fp64 work, native u_MV == u_IP, N in {32, 64} and L in
 * {1, 2, 4, 8}; the CTA-lockstep fpm_cg_kernel otherwise.  Same bits either
 * way. */
int fpm_cg(const double* A, const double* b, const double* Minv, int64_t T, int32_t N, int32_t L,
           int32_t iters, const fpm_precision* prec, int32_t rho_update, double* x, int32_t* breakdown_at,
           int32_t* diverged_at, void* stream);

/* Optional run_batch outputs (BatchResult, solvers.py:188-204; recorded at
 * solvers.py:306-319, 371-386).  Every pointer may be NULL.  Layouts are the
 * reference's, complex values as interleaved binary64 (re, im):
 *   residual_norms, iterate_norms  (iters+1, T)  norm2 of r_i / x_i (linalg.py:122-134)
 *   alphas, betas                  (iters, T)    complex; 0 where the reference records 0
 *   converged_at                   (T,)          first i with ||r_i|| <= rtol*max(||b||, 1e-300), else -1
 *   iterates, residual_vectors     (iters+1, T, N) complex (record_iterates / record_residual_vectors)
 * b_norm is residual_norms[0].  Norms are within a few ulps of NumPy's (its
 * hypot / pairwise sum), everything else is bit-identical. */
typedef struct fpm_cg_history {
  double* residual_norms;
  double* iterate_norms;
  double* alphas;
  double* betas;
  int32_t* converged_at;
  double rtol;
  double* iterates;
  double* residual_vectors;
} fpm_cg_history;

/* fpm_cg plus the BatchResult histories (run_batch, solvers.py:262-393). */
int fpm_cg_ex(const double* A, const double* b, const double* Minv, int64_t T, int32_t N, int32_t L,
              int32_t iters, const fpm_precision* prec, int32_t rho_update, double* x, int32_t* breakdown_at,
              int32_t* diverged_at, const fpm_cg_history* hist, void* stream);

/* Spectral norm ||A_t||_2 = max |lambda| of Hermitian matrices (the a_norm of
 * the convergence study: np.linalg.norm(A, 2), experiments.py:246-256;
 * solvers.py:289-294).  A (T,N,N) complex128 on the device (read as stored:
 * pass exactly Hermitian matrices), norms (T,) float64.  N <= 128.  Lanczos +
 * Sturm-count multisection in binary64; agrees with LAPACK to ~1e-12 relative
 * on the Gram matrices of the study. */
int fpm_herm_norm2(const double* A, int64_t T, int32_t N, double* norms, void* stream);

/* True-residual gaps of the recorded sweeps (run_batch with record_gaps,
 * solvers.py:289-294, 375-377): gaps[i, t] = ||b_t - A_t x_{i,t} - r_{i,t}||_2 /
 * scale[t] for i = 1 .. iters (row 0 is left untouched: the caller zeroes it),
 * from fpm_cg_ex's iterates / residual_vectors ((iters+1, T, N) complex128).
 * A (T,N,N), b (T,N) complex128; scale (T,), gaps (iters+1, T) float64; all on
 * the device.  N <= 128.  Binary64; agrees with the reference's BLAS matvec to
 * rounding. */
int fpm_residual_gaps(const double* A, const double* b, const double* iterates, const double* residual_vectors,
                      const double* scale, int64_t T, int32_t N, int32_t iters, double* gaps, void* stream);

/* LMMSE direct solve x = A^-1 b by fp64 Cholesky (linalg.py:223-231
 * _solve_direct_batch: scipy cho_factor / cho_solve).  A (T,N,N), b (T,N)
 * complex128 on the device.  nonpd: optional device int32 counter of
 * realizations whose A is not positive definite (their x is NaN; the
 * reference raises LinAlgError).  LAPACK bits are not reproduced: x agrees
 * to ~1e-13 normwise. */
int fpm_lmmse(const double* A, const double* b, int64_t T, int32_t N, double* x, int32_t* nonpd, void* stream);

/* Input generation (detect.py:189-214 simulate_trials; channel.py:138-161;
 * rng.py:19-39): per-trial counter-based Philox4x32-10 streams keyed by
 * (seed, context, point, trial) -- trial t's draws are independent of the
 * batch, chunking and device.  Writes, for trials trial0 .. trial0+T-1:
 *   W     (T, M, N) complex  i.i.d. CN(0, 1/M) core (colour with sqrt(R_r) W sqrt(R_t))
 *   bits  (T, nbits) uint8   uniform {0, 1} payload (nbits = 4N for 16-QAM)
 *   noise (T, M)    complex  unit complex normals (scale by sqrt(sigma^2 / 2))
 *   csi   (T, M, N) complex  unit complex normals for perturb_csi, or NULL
 * Distribution-level parity: NumPy's Philox / libm stream is not
 * reproduced.  context < 2^12, point < 2^16 as in rng.py. */
int fpm_gen_trials(uint64_t seed, int32_t context, int32_t point, int64_t trial0, int64_t T, int32_t M, int32_t N,
                   int32_t nbits, double* W, uint8_t* bits, double* noise, double* csi, void* stream);

/* The whole link model of simulate_trials (detect.py:189-214) in one kernel,
 * from the same draws as fpm_gen_trials: H = F_r W F_t^T with F the AR(1)
 * (Cholesky) factor of the exponential correlation zeta^|i-j| (channel.py:
 * 101-125; same distribution as the reference's symmetric square roots,
 * restarting per user block when block_diag_users with n_ue users per
 * block), Gray QAM symbols of the payload bits (detect.py:54-67; qam 16 or
 * 64), y = H s + sqrt(sigma2/2) g (detect.py:210-211) and, when csi_var >= 0,
 * H_est = H + sqrt(csi_var/2) c (channel.py:206-219; csi_var = (1/M)/eps).
 * Outputs (device, caller-owned): H, H_est (NULL iff csi_var < 0), y, bits
 * (T, bps*N), symbols (T, N) or NULL.  N <= 128. */
int fpm_simulate(uint64_t seed, int32_t context, int32_t point, int64_t trial0, int64_t T, int32_t M, int32_t N,
                 double zeta_r, double zeta_t, int32_t n_ue, int32_t block_diag_users, int32_t qam, double sigma2,
                 double csi_var, double* H, double* H_est, double* y, uint8_t* bits, double* symbols,
                 void* stream);

/* qam = 16 (reference) or 64 (extension).  tx_bits / rx_bits: (T, bits*N)
 * uint8 in the reference's layout, both nullable. */
int fpm_slice_count(const double* x, const uint8_t* tx_bits, int64_t T, int32_t N, int32_t qam,
                    uint8_t* rx_bits, int64_t* counters, void* stream);

/* Fused H, y -> x_hat, flags, sliced bits, counters.  Minv_in != NULL
 * injects precomputed block inverses (bit-exact mode); otherwise they are
 * built on-chip in fp64 from the Gram's diagonal blocks. */
int fpm_detect(const double* H, const double* y, const uint8_t* tx_bits, int64_t T, int32_t M, int32_t N,
               double sigma2, int32_t algorithm, int32_t L, int32_t iters, const fpm_precision* prec,
               int32_t rho_update, int32_t qam, const double* Minv_in, double* x, int32_t* breakdown_at,
               int32_t* diverged_at, uint8_t* rx_bits, int64_t* counters, void* stream);

/* As fpm_detect but every pointer is a HOST pointer (pinned memory gives
 * full PCIe rate).  chunk = realizations per pipeline stage (0 = auto).
 * Synchronous: returns when all outputs are in host memory. */
int fpm_detect_host(const double* H, const double* y, const uint8_t* tx_bits, int64_t T, int32_t M,
                    int32_t N, double sigma2, int32_t algorithm, int32_t L, int32_t iters,
                    const fpm_precision* prec, int32_t rho_update, int32_t qam, const double* Minv_in,
                    double* x, int32_t* breakdown_at, int32_t* diverged_at, uint8_t* rx_bits,
                    int64_t* counters, int64_t chunk);

/* Number of kernels this library launched in the calling process (all
 * entry points), for launch accounting in benchmarks. */
int64_t fpm_launch_count(void);

/* Name and specialisation of the last fused detector kernel this library
 * launched ("" before the first fpm_detect / fpm_detect_host call); for
 * benchmark / profile reports; kept per calling host thread. */
const char* fpm_last_kernel(void);

/* Diagnostic: measured rate of non-fused fp64 DMUL/DADD operations per
 * second on the current device (synchronous; the fp64 roofline denominator). */
int fpm_probe_fp64(int64_t iters, double* dp_ops_per_s);

/* Diagnostic builds only (compiled with -DFPM_DIAG, tools/): device buffer
 * that subsequent launches fill with clock64() phase stamps (NULL disables).
 * The product library keeps no such state and returns FPM_EUNSUPPORTED. */
int fpm_debug_set_trace(int64_t* dev_buf);

#ifdef __cplusplus
}
#endif
#endif /* FPMIMO_B200_H */
