"""Input generation on the GPU.

Restates the reference's simulated link (detect.py:189-214
`simulate_trials`; channel.py:101-161 `exp_correlation_matrix` /
`sample_channel`; channel.py:206-219 `perturb_csi`; detect.py:54-67,
87-93 modulation and noise) with the random draws made on the device by
`fpm_gen_trials` (per-trial keyed Philox streams); `simulate_batch` runs
the whole link model -- colouring, payload, y = H s + n -- in one kernel
(`fpm_simulate`).  Every trial's inputs depend
only on (seed, context, point, trial), so batches, chunks and ranks can be
generated independently and a sharded sweep sees the same inputs at any GPU
count.  Parity with the reference generator is distribution-level (its NumPy
Philox + libm stream is not reproduced bit for bit).
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .errors import ContractViolation
from .solvers import _stream, _torch

__all__ = ["exp_correlation_matrix", "matrix_sqrt_psd", "noise_variance", "modulate", "gen_trials",
           "simulate_batch", "simulate_trials"]

_SCALE16 = 1.0 / math.sqrt(10.0)
_LEVEL_OF_PAIR16 = np.array([-3.0, -1.0, 3.0, 1.0]) * _SCALE16          # detect.py:47
_SCALE64 = 1.0 / math.sqrt(42.0)
_LEVEL_OF_TRIPLE64 = np.array([-7.0, -5.0, -1.0, -3.0, 7.0, 5.0, 1.0, 3.0]) * _SCALE64  # Gray, extension


def exp_correlation_matrix(n: int, zeta: float) -> np.ndarray:
    """zeta^|i-j| (channel.py:101-113)."""
    if not 0.0 <= zeta < 1.0:
        raise ContractViolation(f"zeta must lie in [0, 1), got {zeta}")
    if n < 1:
        raise ContractViolation("n must be positive")
    idx = np.arange(n)
    return (zeta ** np.abs(idx[:, None] - idx[None, :])).astype(np.complex128)


def user_correlation_matrix(N: int, zeta_t: float, N_UE: int = 1, block_diag_users: bool = False) -> np.ndarray:
    """channel.py:116-125: full exponential chain or independent users."""
    if not block_diag_users:
        return exp_correlation_matrix(N, zeta_t)
    block = exp_correlation_matrix(N_UE, zeta_t)
    R = np.zeros((N, N), np.complex128)
    for s in range(0, N, N_UE):
        R[s:s + N_UE, s:s + N_UE] = block
    return R


def matrix_sqrt_psd(R) -> np.ndarray:
    """Hermitian PSD square root by eigendecomposition (linalg.py:178-194)."""
    R = np.asarray(R, np.complex128)
    w, V = np.linalg.eigh(0.5 * (R + R.conj().T))
    tol = 10.0 * R.shape[0] * 2.0 ** -53 * max(abs(w[0]), abs(w[-1]))
    if w[0] < -tol:
        raise ContractViolation("matrix is not PSD")
    S = (V * np.sqrt(np.clip(w, 0.0, None))) @ V.conj().T
    return 0.5 * (S + S.conj().T)


def noise_variance(M: int, N: int, snr_db: float, convention: str = "receive_total") -> float:
    """detect.py:87-93."""
    if convention == "receive_total":
        return (N / M) * 10.0 ** (-snr_db / 10.0)
    if convention == "transmit":
        return 10.0 ** (-snr_db / 10.0)
    raise ContractViolation(f"unknown SNR convention {convention!r}")


def modulate(bits, qam: int = 16):
    """Gray-labelled unit-energy QAM (detect.py:54-67; 64-QAM extension):
    bits (..., bps*N) uint8 -> symbols (..., N) complex128, on bits' device."""
    torch = _torch()
    bps = 4 if qam == 16 else 6
    if bits.shape[-1] % bps:
        raise ContractViolation(f"bit count must be a multiple of {bps}")
    g = bits.reshape(*bits.shape[:-1], bits.shape[-1] // bps, bps).long()
    if qam == 16:
        lv = torch.as_tensor(_LEVEL_OF_PAIR16, dtype=torch.float64, device=bits.device)
        re, im = lv[2 * g[..., 0] + g[..., 1]], lv[2 * g[..., 2] + g[..., 3]]
    else:
        lv = torch.as_tensor(_LEVEL_OF_TRIPLE64, dtype=torch.float64, device=bits.device)
        re = lv[4 * g[..., 0] + 2 * g[..., 1] + g[..., 2]]
        im = lv[4 * g[..., 3] + 2 * g[..., 4] + g[..., 5]]
    return torch.complex(re, im)


def gen_trials(seed: int, point: int, trial0: int, T: int, M: int, N: int, *, context: int = 2, qam: int = 16,
               csi: bool = False, device=None):
    """Raw per-trial draws from fpm_gen_trials: W ~ CN(0, 1/M) (T,M,N),
    bits (T, bps*N), unit complex noise (T,M), optional CSI normals."""
    torch = _torch()
    dev = device or torch.device("cuda")
    bps = 4 if qam == 16 else 6
    W = torch.empty((T, M, N), dtype=torch.complex128, device=dev)
    bits = torch.empty((T, bps * N), dtype=torch.uint8, device=dev)
    noise = torch.empty((T, M), dtype=torch.complex128, device=dev)
    C = torch.empty((T, M, N), dtype=torch.complex128, device=dev) if csi else None
    rc = _lib.load().fpm_gen_trials(int(seed) & 0xFFFFFFFFFFFFFFFF, int(context), int(point), int(trial0), int(T),
                                    int(M), int(N), bps * N, W.data_ptr(), bits.data_ptr(), noise.data_ptr(),
                                    None if C is None else C.data_ptr(), _stream())
    _lib.check(rc, "gen_trials")
    return W, bits, noise, C


def simulate_batch(M: int, N: int, zeta_r: float, zeta_t: float, snr_db: float, trial0: int, T: int, seed: int, *,
                   point: int = 0, context: int = 2, qam: int = 16, epsilon_db: float | None = None,
                   convention: str = "receive_total", N_UE: int = 1, block_diag_users: bool = False, device=None):
    """simulate_trials (detect.py:189-214) on the GPU for trials
    trial0 .. trial0+T-1, one fused kernel (fpm_simulate): H coloured by the
    AR(1) / Cholesky factors of the exponential correlations (the same
    Kronecker distribution as sqrt(R_r) W sqrt(R_t), channel.py:138-161),
    uniform bits -> Gray QAM symbols s, y = H s + CN(0, sigma^2), optional
    imperfect CSI H_est (channel.py:206-219).  Returns the reference's batch
    dict keys (CUDA tensors; A and b are left to the detector, which builds
    them bit-exactly from H_est and y)."""
    torch = _torch()
    if not (0.0 <= zeta_r < 1.0 and 0.0 <= zeta_t < 1.0):
        raise ContractViolation("zeta must lie in [0, 1)")
    if block_diag_users and N % N_UE:
        raise ContractViolation("N must be a multiple of N_UE")
    dev = device or torch.device("cuda")
    bps = 4 if qam == 16 else 6
    sigma2 = noise_variance(M, N, snr_db, convention)
    csi_var = -1.0
    if epsilon_db is not None:  # channel.py:206-219: CN(0, (1/M)/eps) estimate error
        if not math.isfinite(epsilon_db):
            raise ContractViolation("epsilon_db must be finite")
        csi_var = (1.0 / M) / 10.0 ** (epsilon_db / 10.0)
    H = torch.empty((T, M, N), dtype=torch.complex128, device=dev)
    H_est = torch.empty_like(H) if csi_var >= 0 else None
    y = torch.empty((T, M), dtype=torch.complex128, device=dev)
    bits = torch.empty((T, bps * N), dtype=torch.uint8, device=dev)
    s = torch.empty((T, N), dtype=torch.complex128, device=dev)
    rc = _lib.load().fpm_simulate(int(seed) & 0xFFFFFFFFFFFFFFFF, int(context), int(point), int(trial0), int(T),
                                  int(M), int(N), float(zeta_r), float(zeta_t), int(N_UE) if block_diag_users else 1,
                                  int(bool(block_diag_users)), int(qam), float(sigma2), float(csi_var),
                                  H.data_ptr(), None if H_est is None else H_est.data_ptr(), y.data_ptr(),
                                  bits.data_ptr(), s.data_ptr(), _stream())
    _lib.check(rc, "simulate")
    return {"H": H, "H_est": H if H_est is None else H_est, "bits": bits, "symbols": s, "y": y, "sigma_n2": sigma2}


def simulate_trials(cfg, snr_idx: int, trial_ids, device=None, qam: int = 16):
    """Drop-in for detect.py:189 (reference BERConfig in, batch dict out) with
    GPU draws; `trial_ids` must be a contiguous range."""
    ids = list(trial_ids) if not isinstance(trial_ids, range) else trial_ids
    if len(ids) and (ids[-1] - ids[0] + 1 != len(ids)):
        raise ContractViolation("trial_ids must be contiguous")
    ch = cfg.channel
    t0 = ids[0] if len(ids) else 0
    return simulate_batch(ch.M, ch.N, ch.zeta_r, ch.zeta_t, float(cfg.snr_grid[snr_idx]), t0, len(ids), cfg.seed,
                          point=snr_idx, context=getattr(cfg, "context", 2), qam=qam,
                          epsilon_db=getattr(cfg, "epsilon_db", None),
                          convention=getattr(cfg, "snr_convention", "receive_total"),
                          N_UE=getattr(ch, "N_UE", 1), block_diag_users=getattr(ch, "block_diag_users", False),
                          device=device)
