"""Warp-per-realization CG (csrc/fpm_cgw.cu) through the C ABI `fpm_cg`:
bit-exact against the oracle's run_batch restatement (solvers.py:262-393)
for every native matvec/inner kind, N in {32, 64}, plain CG and block-Jacobi
L in {1, 2, 4, 8}, both rho updates, the freeze flags (stall / breakdown /
divergence), and bit-identical to the CTA-lockstep fpm_cg_kernel at batch
sizes the oracle would take minutes on."""

import ctypes

import numpy as np
import pytest

from conftest import bits_equal, knob_child, run_knob_child, save_child_out

pytestmark = pytest.mark.gpu

KINDS = {"fp64": (53, 11), "fp32": (24, 8), "fp16": (11, 5), "bfloat16": (8, 8)}


def _cg_capi(A, b, minv, L, iters, fmt, rho_update, env=None, monkeypatch=None):
    """fpm_cg (no histories) on device copies; returns x, brk, div, kernel."""
    import torch
    from paper_2504_09820_b200 import _lib
    from paper_2504_09820_b200.solvers import _stream
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    T, N = b.shape
    Ad = torch.from_numpy(np.ascontiguousarray(A, np.complex128)).to(dev)
    bd = torch.from_numpy(np.ascontiguousarray(b, np.complex128)).to(dev)
    md = None if minv is None else torch.from_numpy(np.ascontiguousarray(minv, np.complex128)).to(dev)
    x = torch.empty((T, N), dtype=torch.complex128, device=dev)
    brk = torch.empty(T, dtype=torch.int32, device=dev)
    div = torch.empty(T, dtype=torch.int32, device=dev)
    sig, ex = KINDS[fmt]
    ps = _lib.Precision(_lib.Format(53, 11, 1), _lib.Format(sig, ex, 1), _lib.Format(sig, ex, 1))
    rc = lib.fpm_cg(Ad.data_ptr(), bd.data_ptr(), None if md is None else md.data_ptr(), T, N, L if md is not None else 1,
                    iters, ctypes.byref(ps), 0 if rho_update == "as_written" else 1, x.data_ptr(), brk.data_ptr(),
                    div.data_ptr(), _stream())
    _lib.check(rc, "fpm_cg")
    torch.cuda.synchronize()
    kern = lib.fpm_last_kernel().decode()
    return x.cpu().numpy(), brk.cpu().numpy(), div.cpu().numpy(), kern


def _pack(mats, N, L):
    from paper_2504_09820_b200.solvers import pack_blocks
    return pack_blocks(mats, N, L)


def _system(O, M, N, T, seed, snr=10.0):
    H, y, _, s2 = O.simulate(M, N, 0.5, snr, range(T), seed)
    return O.gram_mf(H, y, s2)


@pytest.mark.parametrize("fmt", list(KINDS))
@pytest.mark.parametrize("N", [32, 64])
def test_cgw_matches_oracle(oracle, fmt, N):
    O = oracle
    T = 7
    A, b = _system(O, 2 * N, N, T, 31 + N)
    of = O.REGISTRY[fmt]
    for L in (0, 1, 2, 4, 8):
        mats = O.bj_inverses(A, L) if L else None
        for rv in ("as_written", "textbook"):
            if L == 0 and rv == "textbook":
                continue
            ref = O.cg_batch(A, b, 6, O.FP64, of, of, mats, rho_update=rv)
            x, brk, div, kern = _cg_capi(A, b, _pack(mats, N, L) if L else None, L, 6, fmt, rv)
            assert kern.startswith("fpm_cgw_kernel"), kern
            assert bits_equal(x, ref.x), (fmt, N, L, rv)
            np.testing.assert_array_equal(brk, ref.breakdown_at)
            np.testing.assert_array_equal(div, ref.diverged_at)


@pytest.mark.parametrize("fmt", ["fp64", "fp16", "bfloat16"])
def test_cgw_freeze_flags(oracle, fmt):
    """Stall (b = 0), breakdown (negative definite A), divergence (fp16
    overflow of the matvec / a NaN entry) and healthy lanes side by side."""
    O = oracle
    N, T = 32, 6
    A0, b = _system(O, 64, N, T, 5)
    A = A0.copy()
    b = b.copy()
    b[1] = 0.0                                   # stall at sweep 1
    A[2] = -A[2]                                 # Re(phi) < 0: breakdown at sweep 1
    A[3] *= 1e6                                  # fp16 / bf16 matvec overflow
    b[3] *= 1e6
    A[4, 3, 5] = np.nan                          # non-finite update
    for L in (0, 4):
        mats = O.bj_inverses(A0, L) if L else None  # preconditioner of the clean systems
        of = O.REGISTRY[fmt]
        ref = O.cg_batch(A, b, 6, O.FP64, of, of, mats)
        x, brk, div, kern = _cg_capi(A, b, _pack(mats, N, L) if L else None, L, 6, fmt, "as_written")
        assert kern.startswith("fpm_cgw_kernel"), kern
        assert bits_equal(x, ref.x), (fmt, L)
        np.testing.assert_array_equal(brk, ref.breakdown_at)
        np.testing.assert_array_equal(div, ref.diverged_at)


def _lockstep_case(fmt, L):
    N, T = 64, 4096
    rng = np.random.default_rng(7)
    Hh = (rng.standard_normal((T, 128, N)) + 1j * rng.standard_normal((T, 128, N))) / np.sqrt(256)
    s = (rng.integers(0, 2, (T, N)) * 2 - 1 + 1j * (rng.integers(0, 2, (T, N)) * 2 - 1)) / np.sqrt(2)
    y = np.einsum("tmn,tn->tm", Hh, s) + 0.05 * (rng.standard_normal((T, 128)) + 1j * rng.standard_normal((T, 128)))
    from paper_2504_09820_b200.detect import gram_mf
    from paper_2504_09820_b200.solvers import build_blocks_batch
    A, b = gram_mf(Hh, y, 0.005)
    minv = build_blocks_batch(A, L).packed if L else None
    return _cg_capi(A, b, minv, L, 8, fmt, "as_written")


LOCKSTEP_CASES = [("fp16", 4), ("bfloat16", 0), ("fp64", 4), ("fp32", 2)]


@pytest.mark.parametrize("fmt,L", LOCKSTEP_CASES)
def test_cgw_equals_lockstep_kernel_at_scale(fmt, L):
    """The warp kernel and the CTA-lockstep kernel (knob FPM_NO_CGW, in a fresh
    process) give the same bits on a 4096-realization c5-shaped batch."""
    x1, b1, d1, k1 = _lockstep_case(fmt, L)
    o = run_knob_child(f"tests/test_gpu_cgw.py::test_child_lockstep[{fmt}-{L}]", {"FPM_NO_CGW": "1"})
    assert k1.startswith("fpm_cgw_kernel") and not str(o["k"]).startswith("fpm_cgw_kernel"), (k1, o["k"])
    assert bits_equal(x1, o["x"])
    np.testing.assert_array_equal(b1, o["b"])
    np.testing.assert_array_equal(d1, o["d"])


@knob_child
@pytest.mark.parametrize("fmt,L", LOCKSTEP_CASES)
def test_child_lockstep(fmt, L):
    x, b, d, k = _lockstep_case(fmt, L)
    save_child_out(x=x, b=b, d=d, k=np.array(k))


@pytest.mark.parametrize("fmt", ["fp16", "bfloat16"])
def test_cgw_tmem_variant_matches_oracle(fmt):
    """The opt-in TMEM variant (knob FPM_CGW_TMEM=1: A in tensor memory, four
    warps per CTA) gives the oracle's bits, including a partial last CTA."""
    run_knob_child(f"tests/test_gpu_cgw.py::test_child_tmem[{fmt}]", {"FPM_CGW_TMEM": "1"})


@knob_child
@pytest.mark.parametrize("fmt", ["fp16", "bfloat16"])
def test_child_tmem(oracle, fmt):
    O = oracle
    T, N = 7, 64
    A, b = _system(O, 128, N, T, 77)
    of = O.REGISTRY[fmt]
    for L in (0, 4):
        mats = O.bj_inverses(A, L) if L else None
        for rv in (("as_written", "textbook") if L else ("as_written",)):
            ref = O.cg_batch(A, b, 6, O.FP64, of, of, mats, rho_update=rv)
            x, brk, div, kern = _cg_capi(A, b, _pack(mats, N, L) if L else None, L, 6, fmt, rv)
            assert bits_equal(x, ref.x), (fmt, L, rv)
            np.testing.assert_array_equal(brk, ref.breakdown_at)
            np.testing.assert_array_equal(div, ref.diverged_at)


@pytest.mark.parametrize("fmt,N,L", [("fp16", 64, 4), ("bfloat16", 32, 0), ("fp64", 64, 4), ("fp32", 32, 2)])
def test_cgw_run_batch_histories(oracle, fmt, N, L):
    """The Python run_batch mirror (solvers.py:262-393; it always requests the
    norm histories) on the warp kernel: every BatchResult field against the
    oracle's run_batch restatement, with stall / breakdown / divergence lanes
    so the frozen-sweep recording is exercised."""
    from paper_2504_09820_b200 import _lib
    from paper_2504_09820_b200.formats import get_format
    from paper_2504_09820_b200.solvers import BatchBlocks, PrecisionConfig, run_batch
    from test_gpu_parity import HIST_NORMS, _check_history
    O = oracle
    T = 6
    A0, b = _system(O, 2 * N, N, T, 11 + N)
    A, b = A0.copy(), b.copy()
    b[1] = 0.0          # stall at sweep 1
    A[2] = -A[2]        # breakdown at sweep 1
    A[4, 3, 5] = np.nan  # non-finite update
    mats = O.bj_inverses(A0, L) if L else None
    of = O.REGISTRY[fmt]
    f = get_format(fmt)
    want = O.cg_batch(A, b, 6, O.FP64, of, of, mats, rtol=1e-3, record=True)
    res = run_batch(A, b, 6, PrecisionConfig(matvec=f, inner=f), BatchBlocks(_pack(mats, N, L), N, L) if L else None,
                    rtol=1e-3, record_iterates=True, record_residual_vectors=True)
    assert _lib.load().fpm_last_kernel().decode().startswith("fpm_cgw_kernel")
    _check_history(res, {k: getattr(want, k) for k in
                         ("x", "breakdown_at", "diverged_at", "alphas", "betas", "converged_at", "iterates",
                          "residual_vectors") + HIST_NORMS}, f"{fmt}-{N}-{L}")
