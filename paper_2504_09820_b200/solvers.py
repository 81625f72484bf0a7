"""GPU drop-in for the reference solver layer (solvers.py).

    PrecisionConfig      <- solvers.py:56-85
    BatchResult          <- solvers.py:188-204 (x and flags; histories None)
    build_blocks_batch   <- solvers.py:232-253  (fpm_bj_setup)
    run_batch            <- solvers.py:262-393  (fpm_cg)

Arrays may be NumPy (host; results come back as NumPy, like the
reference) or torch CUDA tensors (results stay on the device).  Every
computation runs in libfpmimo_b200.so; there is no CPU path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ContractViolation
from .formats import FP64, FloatFormat, get_format

__all__ = ["PrecisionConfig", "BatchResult", "BatchBlocks", "build_blocks_batch", "run_batch",
           "pack_blocks"]


@dataclass(frozen=True)
class PrecisionConfig:
    work: FloatFormat = FP64
    matvec: FloatFormat = FP64
    inner: FloatFormat = FP64

    def __post_init__(self):
        for k in ("work", "matvec", "inner"):
            object.__setattr__(self, k, get_format(getattr(self, k)))
        if (self.work.unit_roundoff > self.matvec.unit_roundoff
                or self.work.unit_roundoff > self.inner.unit_roundoff):
            raise ContractViolation("working precision must be at least as fine as the "
                                    "matrix-vector and inner-product precisions")

    @classmethod
    def uniform(cls, fmt) -> "PrecisionConfig":
        fmt = get_format(fmt)
        return cls(work=fmt, matvec=fmt, inner=fmt)

    @property
    def is_native(self) -> bool:
        return self.work.is_native and self.matvec.is_native and self.inner.is_native

    def labels(self):
        return (self.work.name, self.matvec.name, self.inner.name)


@dataclass
class BatchResult:
    x: object                 # (T, N) complex128
    breakdown_at: object      # (T,) int64, -1 if none
    diverged_at: object       # (T,) int64, -1 if none
    iterations_run: int = 0
    residual_norms: object = None
    iterate_norms: object = None
    alphas: object = None
    betas: object = None
    b_norm: object = None
    converged_at: object = None
    residual_gaps: object = None      # (iters+1, T) record_gaps
    iterates: object = None           # (iters+1, T, N) record_iterates
    residual_vectors: object = None   # (iters+1, T, N) record_residual_vectors


class BatchBlocks:
    """Block-diagonal inverses, packed per realization with stride N*L
    (block k = row-major Lk x Lk at entry k*L*L), as the C ABI expects.
    `.mats` gives the reference's list-of-(T, Lk, Lk) view."""

    def __init__(self, packed, N: int, L: int):
        # a ragged tail block makes the natural concatenation shorter than
        # the fixed N*L stride; pad it
        if packed.shape[1] < N * L:
            if _is_torch(packed):
                torch = _torch()
                packed = torch.nn.functional.pad(packed, (0, N * L - packed.shape[1]))
            else:
                packed = np.pad(np.asarray(packed), ((0, 0), (0, N * L - packed.shape[1])))
        self.packed = packed
        self.N = N
        self.L = L

    @property
    def sizes(self):
        return [min(self.L, self.N - s) for s in range(0, self.N, self.L)]

    @property
    def mats(self):
        out, T = [], self.packed.shape[0]
        for k, Lk in enumerate(self.sizes):
            off = k * self.L * self.L
            out.append(self.packed[:, off:off + Lk * Lk].reshape(T, Lk, Lk))
        return out


def pack_blocks(mats, N: int, L: int):
    """list of (T, Lk, Lk) arrays (reference _BatchBlocks.mats) -> packed (T, N*L)."""
    T = mats[0].shape[0]
    out = np.zeros((T, N * L), np.complex128)
    for k, m in enumerate(mats):
        Lk = m.shape[-1]
        out[:, k * L * L:k * L * L + Lk * Lk] = np.asarray(m, np.complex128).reshape(T, Lk * Lk)
    return out


# ---------------------------------------------------------------------------
# device helpers
# ---------------------------------------------------------------------------

def _torch():
    import torch
    return torch


def _to_dev(a, dtype):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        if not a.is_cuda:
            a = a.cuda()
        return a.to(dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def _is_torch(a):
    try:
        import torch
        return isinstance(a, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def _stream():
    return ctypes_stream(_torch().cuda.current_stream())


def ctypes_stream(s):
    return s.cuda_stream


def _out(t, host):
    return t.cpu().numpy() if host else t


def build_blocks_batch(A, L: int, *, allow_ragged: bool = False) -> BatchBlocks:
    """Batched block-Jacobi setup (solvers.py:232-253) on the GPU: fp64
    Cholesky PD check + Hermitian inverse per diagonal block."""
    torch = _torch()
    host = not _is_torch(A)
    Ad = _to_dev(A, torch.complex128)
    T, N = Ad.shape[0], Ad.shape[-1]
    if N % L and not allow_ragged:
        raise ContractViolation(f"L={L} must divide the system dimension {N}")
    packed = torch.zeros((T, N * L), dtype=torch.complex128, device=Ad.device)
    bad = torch.empty((T,), dtype=torch.int32, device=Ad.device)
    lib = _lib.load()
    rc = lib.fpm_bj_setup(Ad.data_ptr(), T, N, L, int(allow_ragged), packed.data_ptr(), bad.data_ptr(),
                          _stream())
    if rc == _lib.FPM_ENOTPD:
        first = int(bad[bad >= 0][0].item()) if bool((bad >= 0).any()) else -1
        raise ContractViolation(f"non-PD diagonal block at {first}")
    _lib.check(rc, "build_blocks_batch")
    return BatchBlocks(_out(packed, host), N, L)


def solve_direct_batch(A, b):
    """Batched Cholesky solve x = A^-1 b (linalg.py:223-231,
    _solve_direct_batch: the LMMSE comparator) on the GPU.  Raises
    ContractViolation where scipy's cho_factor would fail (non-PD A)."""
    torch = _torch()
    host = not _is_torch(b)
    Ad = _to_dev(A, torch.complex128)
    bd = _to_dev(b, torch.complex128)
    T, N = bd.shape
    x = torch.empty((T, N), dtype=torch.complex128, device=bd.device)
    bad = torch.zeros((1,), dtype=torch.int32, device=bd.device)
    _lib.check(_lib.load().fpm_lmmse(Ad.data_ptr(), bd.data_ptr(), T, N, x.data_ptr(), bad.data_ptr(), _stream()),
               "solve_direct_batch")
    if int(bad.item()):
        raise ContractViolation("matrix is not positive definite")
    return _out(x, host)


def _norm2_t(v):
    """norm2 over the trailing axis (linalg.py:122-134) on the device:
    scale = max|v| (NaN-propagating, 1 unless finite and > 0), inf if any |v|
    is inf."""
    torch = _torch()
    mags = torch.abs(v)
    scale = mags.amax(-1) if mags.shape[-1] else torch.zeros(mags.shape[:-1], dtype=mags.dtype, device=mags.device)
    scale = torch.where(torch.isfinite(scale) & (scale > 0), scale, torch.ones_like(scale))
    sc = mags / scale[..., None]
    out = scale * torch.sqrt((sc * sc).sum(-1))
    return torch.where(torch.isinf(mags).any(-1), torch.full_like(out, float("inf")), out)


def herm_norm2(A):
    """||A_t||_2 of Hermitian matrices on the device (np.linalg.norm(A, 2) in
    the reference's convergence study, experiments.py:246-256): the library's
    Lanczos / Sturm-count kernel (fpm_herm_norm2).  Returns a (T,) float64
    CUDA tensor."""
    torch = _torch()
    Ad = _to_dev(A, torch.complex128).contiguous()
    T, N = Ad.shape[0], Ad.shape[-1]
    out = torch.empty((T,), dtype=torch.float64, device=Ad.device)
    _lib.check(_lib.load().fpm_herm_norm2(Ad.data_ptr(), T, N, out.data_ptr(), _stream()), "herm_norm2")
    return out


def run_batch(A, b, max_iters: int, prec: PrecisionConfig | None = None, blocks=None, *,
              rho_update: str = "as_written", rtol: float = 1e-6, x_ref=None, a_norm=None,
              record_gaps: bool = False, record_iterates: bool = False,
              record_residual_vectors: bool = False) -> BatchResult:
    """Lockstep mixed-precision (BJ-)CG on the GPU (solvers.py:262-393).

    `blocks` may be a BatchBlocks, or anything with a `.mats` list of
    (T, Lk, Lk) arrays (the reference's _BatchBlocks).  Returns the
    reference's BatchResult: x, breakdown_at, diverged_at, alphas, betas and
    the record_iterates / record_residual_vectors outputs bit-identical;
    residual / iterate norms and gaps within a few ulps (norm2's hypot and
    summation order).  NumPy in -> NumPy out; CUDA tensors -> CUDA tensors.
    """
    torch = _torch()
    if prec is None:
        prec = PrecisionConfig()
    if rho_update not in _lib.FPM_RHO:
        raise ContractViolation(f"unknown rho_update variant {rho_update!r}")
    if max_iters < 1:
        raise ContractViolation("max_iters must be at least 1")
    if record_gaps and x_ref is None:
        raise ContractViolation("gap recording needs a reference solution")
    host = not _is_torch(b)
    Ad = _to_dev(A, torch.complex128)
    bd = _to_dev(b, torch.complex128)
    T, N = bd.shape
    minv = None
    L = 1
    if blocks is not None:
        # a preconditioner built for another system size or batch is a
        # contract violation (solvers.py:222-225 apply, tests/test_solvers.py:284-290)
        if isinstance(blocks, BatchBlocks):
            L, packed = blocks.L, blocks.packed
            if blocks.N != N or packed.shape[0] != T:
                raise ContractViolation(f"block-Jacobi blocks are for n={blocks.N}, T={packed.shape[0]}; "
                                        f"system has n={N}, T={T}")
        else:
            mats = blocks.mats
            L = mats[0].shape[-1]
            if sum(m.shape[-1] for m in mats) != N or any(m.shape[0] != T for m in mats):
                raise ContractViolation(f"block-Jacobi blocks do not partition n={N} over T={T} systems")
            packed = pack_blocks([np.asarray(m) for m in mats], N, L)
        minv = _to_dev(packed, torch.complex128)
    dev = bd.device
    it1 = max_iters + 1
    x = torch.empty((T, N), dtype=torch.complex128, device=dev)
    brk = torch.empty((T,), dtype=torch.int32, device=dev)
    div = torch.empty((T,), dtype=torch.int32, device=dev)
    res = torch.empty((it1, T), dtype=torch.float64, device=dev)
    xnh = torch.empty((it1, T), dtype=torch.float64, device=dev)
    alphas = torch.empty((max_iters, T), dtype=torch.complex128, device=dev)
    betas = torch.empty((max_iters, T), dtype=torch.complex128, device=dev)
    conv = torch.empty((T,), dtype=torch.int32, device=dev)
    need_vec = record_iterates or record_gaps
    xit = torch.empty((it1, T, N), dtype=torch.complex128, device=dev) if need_vec else None
    rit = torch.empty((it1, T, N), dtype=torch.complex128, device=dev) \
        if (record_residual_vectors or record_gaps) else None
    hist = _lib.CgHistory(res.data_ptr(), xnh.data_ptr(), alphas.data_ptr(), betas.data_ptr(), conv.data_ptr(),
                          float(rtol), None if xit is None else xit.data_ptr(),
                          None if rit is None else rit.data_ptr())
    lib = _lib.load()
    ps = _lib.precision_struct(prec)
    rc = lib.fpm_cg_ex(Ad.data_ptr(), bd.data_ptr(), None if minv is None else minv.data_ptr(), T, N, L,
                       int(max_iters), ps, _lib.FPM_RHO[rho_update], x.data_ptr(), brk.data_ptr(),
                       div.data_ptr(), hist, _stream())
    _lib.check(rc, "run_batch")
    gaps = None
    if record_gaps:  # solvers.py:289-294, 375-377: ||b - A x_i - r_i|| / (||A|| ||x_ref||)
        xr = _to_dev(x_ref, torch.complex128)
        if a_norm is None:
            an = herm_norm2(Ad)
        else:
            an = _to_dev(np.asarray(a_norm, np.float64) if not _is_torch(a_norm) else a_norm, torch.float64)
        scale = (an * _norm2_t(xr)).contiguous()
        gaps = torch.zeros((it1, T), dtype=torch.float64, device=dev)
        _lib.check(lib.fpm_residual_gaps(Ad.data_ptr(), bd.data_ptr(), xit.data_ptr(), rit.data_ptr(),
                                         scale.data_ptr(), T, N, int(max_iters), gaps.data_ptr(), _stream()),
                   "residual_gaps")
    return BatchResult(
        x=_out(x, host), breakdown_at=_out(brk.to(torch.int64), host), diverged_at=_out(div.to(torch.int64), host),
        iterations_run=int(max_iters), residual_norms=_out(res, host), iterate_norms=_out(xnh, host),
        alphas=_out(alphas, host), betas=_out(betas, host), b_norm=_out(res[0].clone(), host),
        converged_at=_out(conv.to(torch.int64), host), residual_gaps=None if gaps is None else _out(gaps, host),
        iterates=_out(xit, host) if record_iterates else None,
        residual_vectors=_out(rit, host) if record_residual_vectors else None)