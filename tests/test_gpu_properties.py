"""Behavioural properties the reference's own tests assert about the hot path
(tests/test_solvers.py, tests/test_detect.py in the reference), checked on
the CUDA path at BASELINE batch sizes: identities that hold bit for bit
(degenerate equivalences, lockstep == per-system, exact preconditioner) and
statistical ones (noiseless sanity, BER monotone in SNR, CG at full budget
vs LMMSE)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def _batch(T, M=128, N=64, zeta=0.5, snr=15.0, seed=1, block_diag=False):
    from paper_2504_09820_b200 import channel
    return channel.simulate_batch(M, N, zeta, zeta, snr, 0, T, seed, N_UE=4 if block_diag else 1,
                                  block_diag_users=block_diag)


def _system(T, **kw):
    from paper_2504_09820_b200.detect import gram_mf
    b = _batch(T, **kw)
    A, rhs = gram_mf(b["H_est"], b["y"], b["sigma_n2"])
    return A, rhs, b


def _identity_blocks(T, N, L):
    torch = _torch()
    from paper_2504_09820_b200.solvers import BatchBlocks
    eye = torch.eye(L, dtype=torch.complex128, device="cuda").reshape(-1)
    packed = eye.repeat(T, N // L)
    return BatchBlocks(packed.contiguous(), N, L)


def test_identity_system_converges_in_one_step_and_stalls_gracefully():
    """test_solvers.py:26-59 (the reference's identity system, replicated
    over 4096 lanes): x_1 = b exactly, converged at 1, residual 0, further
    sweeps stall without a breakdown flag."""
    torch = _torch()
    from paper_2504_09820_b200.solvers import run_batch
    T, n = 4096, 4
    A = torch.eye(n, dtype=torch.complex128, device="cuda").expand(T, n, n).contiguous()
    b1 = torch.complex(torch.arange(1.0, n + 1, dtype=torch.float64), torch.arange(0.0, n, dtype=torch.float64))
    b = b1.to("cuda").expand(T, n).contiguous()
    for iters in (1, 3):
        r = run_batch(A, b, iters)
        assert torch.equal(r.x, b)
        assert bool((r.converged_at == 1).all())
        assert bool((r.residual_norms[1] == 0).all())
        assert bool((r.breakdown_at == -1).all()) and bool((r.diverged_at == -1).all())


def test_fp_cg_with_native_formats_is_bit_identical_to_cg():
    """test_solvers.py:96-110, at the c5 shape through both boundaries."""
    torch = _torch()
    from paper_2504_09820_b200.detect import DetectorSpec, detect
    from paper_2504_09820_b200.solvers import PrecisionConfig, run_batch
    A, b, bt = _system(4096, zeta=0.8)
    ref = run_batch(A, b, 25, record_iterates=True, record_residual_vectors=True)
    got = run_batch(A, b, 25, PrecisionConfig.uniform("fp64"), record_iterates=True, record_residual_vectors=True)
    for f in ("x", "iterates", "residual_vectors", "alphas", "betas", "residual_norms", "converged_at"):
        assert torch.equal(getattr(got, f), getattr(ref, f)), f
    d1 = detect(DetectorSpec("cg", iters=12), bt["H_est"], bt["y"], bt["sigma_n2"], bt["bits"])
    d2 = detect(DetectorSpec("fp_cg", iters=12), bt["H_est"], bt["y"], bt["sigma_n2"], bt["bits"])
    assert torch.equal(d1.x, d2.x)


def test_bj_identity_blocks_textbook_is_bit_identical_to_cg():
    """test_solvers.py:112-125: identity block inverses + textbook rho
    reproduce plain CG bit for bit (iterates, residual vectors, alphas,
    betas, x)."""
    torch = _torch()
    from paper_2504_09820_b200.solvers import run_batch
    A, b, _ = _system(4096, zeta=0.8)
    T, N = b.shape
    ref = run_batch(A, b, 20, record_iterates=True, record_residual_vectors=True)
    got = run_batch(A, b, 20, blocks=_identity_blocks(T, N, 8), rho_update="textbook", record_iterates=True,
                    record_residual_vectors=True)
    for f in ("x", "iterates", "residual_vectors", "alphas", "betas"):
        assert torch.equal(getattr(got, f), getattr(ref, f)), f


def test_bj_identity_blocks_as_written_tracks_cg():
    """test_solvers.py:127-140: as_written pairs r with p, equal to plain CG
    only up to roundoff; early sweeps stay extremely close."""
    torch = _torch()
    from paper_2504_09820_b200.solvers import run_batch
    A, b, _ = _system(2048, zeta=0.8)
    T, N = b.shape
    ref = run_batch(A, b, 15, record_iterates=True)
    got = run_batch(A, b, 15, blocks=_identity_blocks(T, N, N if N <= 16 else 16), rho_update="as_written",
                    record_iterates=True)
    torch.testing.assert_close(got.alphas[:5], ref.alphas[:5], rtol=1e-12, atol=0)
    torch.testing.assert_close(got.iterates[:6], ref.iterates[:6], rtol=1e-10, atol=1e-13)


def test_exact_preconditioner_converges_immediately():
    """test_solvers.py:234-238: one block = A^-1 (c1 shape, N = 16) ->
    converged at sweep 1 for every realization."""
    torch = _torch()
    from paper_2504_09820_b200.solvers import build_blocks_batch, run_batch
    A, b, _ = _system(4096, M=128, N=16, zeta=0.8)
    r = run_batch(A, b, 2, blocks=build_blocks_batch(A, 16), rtol=1e-8)
    assert bool((r.converged_at == 1).all())


def test_block_diagonal_system_converges_immediately():
    """test_solvers.py:240-246: A replaced by its 4x4 block-diagonal part,
    L = 8 blocks (exact inverse of it) -> converged at sweep 1."""
    torch = _torch()
    from paper_2504_09820_b200.solvers import build_blocks_batch, run_batch
    A, b, _ = _system(2048, zeta=0.8)
    T, N = b.shape
    mask = torch.block_diag(*[torch.ones(4, 4) for _ in range(N // 4)]).to(device="cuda", dtype=torch.bool)
    Abd = torch.where(mask, A, torch.zeros_like(A))
    r = run_batch(Abd, b, 3, blocks=build_blocks_batch(Abd, 8), rtol=1e-8)
    assert bool((r.converged_at == 1).all())


def test_preconditioning_speeds_up_correlated_systems():
    """test_solvers.py:248-255 (the reference's system: M = 256, K = 8 x
    N_UE = 4, zeta = 0.8): BJ-CG (L = 8) reaches rtol 1e-6 within 40 sweeps
    and in fewer sweeps than plain CG on average."""
    torch = _torch()
    from paper_2504_09820_b200.solvers import build_blocks_batch, run_batch
    A, b, _ = _system(1024, M=256, N=32, zeta=0.8, snr=20.0)
    plain = run_batch(A, b, 40, rtol=1e-6)
    pre = run_batch(A, b, 40, blocks=build_blocks_batch(A, 8), rtol=1e-6)
    assert float((pre.converged_at > 0).double().mean()) >= 0.99
    cp = torch.where(plain.converged_at > 0, plain.converged_at, torch.full_like(plain.converged_at, 41))
    assert float(pre.converged_at.double().mean()) < float(cp.double().mean())


def test_rho_variants_track_each_other():
    """test_solvers.py:276-282."""
    torch = _torch()
    from paper_2504_09820_b200.solvers import build_blocks_batch, run_batch
    A, b, _ = _system(1024, M=256, zeta=0.8)
    blk = build_blocks_batch(A, 8)
    a = run_batch(A, b, 20, blocks=blk, rho_update="as_written")
    t = run_batch(A, b, 20, blocks=blk, rho_update="textbook")
    torch.testing.assert_close(a.alphas[:6], t.alphas[:6], rtol=1e-10, atol=0)
    torch.testing.assert_close(a.x, t.x, rtol=1e-6, atol=1e-9)


def test_lockstep_batch_equals_per_system_runs():
    """test_solvers.py:293-317: every lane of a batched run equals the same
    system run alone (fp16 matvec / inner, with and without BJ)."""
    torch = _torch()
    from paper_2504_09820_b200.solvers import PrecisionConfig, build_blocks_batch, run_batch
    A, b, _ = _system(512, zeta=0.8)
    prec = PrecisionConfig(work="fp64", matvec="fp16", inner="fp16")
    blk = build_blocks_batch(A, 8)
    full = run_batch(A, b, 12, prec)
    fullb = run_batch(A, b, 10, prec, blocks=blk)
    for t in (0, 1, 137, 511):
        one = run_batch(A[t:t + 1], b[t:t + 1], 12, prec)
        assert torch.equal(one.x[0], full.x[t]) and torch.equal(one.alphas[:, 0], full.alphas[:, t])
        oneb = run_batch(A[t:t + 1], b[t:t + 1], 10, prec, blocks=build_blocks_batch(A[t:t + 1], 8))
        assert torch.equal(oneb.x[0], fullb.x[t]) and torch.equal(oneb.alphas[:, 0], fullb.alphas[:, t])


def test_finite_termination_and_gap_start():
    """test_solvers.py:68-74, 88-93: plain CG run for N sweeps reaches the
    direct solution to 1e-8 (M = 256, zeta = 0.5); the recorded gap starts
    at exactly 0."""
    torch = _torch()
    from paper_2504_09820_b200.solvers import run_batch, solve_direct_batch
    A, b, _ = _system(256, M=256, N=64, zeta=0.5)
    x_ref = solve_direct_batch(A, b)
    r = run_batch(A, b, 64, x_ref=x_ref, record_gaps=True)
    rel = torch.linalg.vector_norm(r.x - x_ref, dim=-1) / torch.linalg.vector_norm(x_ref, dim=-1)
    assert float(rel.max()) <= 1e-8
    assert bool((r.residual_gaps[0] == 0).all())


def test_a_norm_error_decreases_monotonically():
    """test_solvers.py:76-86, every lane of a batch until it converges."""
    torch = _torch()
    from paper_2504_09820_b200.solvers import run_batch, solve_direct_batch
    A, b, _ = _system(256, zeta=0.5)
    x_ref = solve_direct_batch(A, b)
    r = run_batch(A, b, 20, x_ref=x_ref, rtol=1e-6, record_iterates=True)
    e = x_ref[None] - r.iterates                                   # (21, T, N)
    err = torch.einsum("itn,tnm,itm->it", e.conj(), A, e).real      # e^H A e
    for t in range(b.shape[0]):
        stop = int(r.converged_at[t]) if int(r.converged_at[t]) > 0 else 20
        assert bool((torch.diff(err[: stop + 1, t]) < 0).all()), t


def test_mismatched_preconditioner_and_bad_variant_rejected():
    """test_solvers.py:284-290, 319-322."""
    from paper_2504_09820_b200.errors import ContractViolation
    from paper_2504_09820_b200.solvers import run_batch
    A, b, _ = _system(8, N=16)
    with pytest.raises(ContractViolation):
        run_batch(A, b, 2, blocks=_identity_blocks(8, 8, 4))
    with pytest.raises(ContractViolation):
        run_batch(A, b, 2, rho_update="fused")


def test_noiseless_sanity_all_detectors_errorless():
    """test_detect.py:98-123: at the reference's sweep shape (M = 32,
    K = 4 x N_UE = 2, zeta = 0.5) every detector of that test is errorless
    at 300 dB, here over 16384 realizations; at the c5 shape the direct
    solve and CG run to N sweeps are errorless too."""
    from paper_2504_09820_b200.detect import DetectorSpec, detect
    bt = _batch(1 << 14, M=32, N=8, snr=300.0, seed=77)
    for det in (DetectorSpec("lmmse"), DetectorSpec("cg", iters=16),
                DetectorSpec("fp_bj_cg", iters=8, L=4, matvec="fp16", inner="fp16")):
        res = detect(det, bt["H_est"], bt["y"], bt["sigma_n2"], bt["bits"])
        assert int(res.counters["bit_errors"]) == 0, det.name
    bt = _batch(1 << 14, snr=300.0)
    for det in (DetectorSpec("lmmse"), DetectorSpec("cg", iters=64)):
        res = detect(det, bt["H_est"], bt["y"], bt["sigma_n2"], bt["bits"])
        assert int(res.counters["bit_errors"]) == 0, det.name


def test_ber_not_increasing_in_snr_and_cg_full_budget_matches_lmmse():
    """test_detect.py:142-156 at the c5 shape (8192 realizations per point):
    BER at 0 dB >= BER at 20 dB for every detector; CG with N sweeps within
    the LMMSE point's Wilson interval."""
    from paper_2504_09820_b200.detect import DetectorSpec, detect
    from paper_2504_09820_b200.parallel import wilson_interval
    dets = (DetectorSpec("lmmse"), DetectorSpec("cg", iters=8),
            DetectorSpec("fp_bj_cg", iters=8, L=4, matvec="fp16", inner="fp16"))
    T, nbits = 8192, 8192 * 4 * 64
    ber = {}
    for snr in (0.0, 10.0, 20.0):
        bt = _batch(T, snr=snr, seed=11)
        for det in dets:
            res = detect(det, bt["H_est"], bt["y"], bt["sigma_n2"], bt["bits"])
            ber[(det.name, snr)] = int(res.counters["bit_errors"]) / nbits
    for det in dets:
        assert ber[(det.name, 0.0)] >= ber[(det.name, 20.0)], det.name
    bt = _batch(T, snr=8.0, seed=12)
    lm = detect(dets[0], bt["H_est"], bt["y"], bt["sigma_n2"], bt["bits"])
    cg = detect(DetectorSpec("cg", iters=64), bt["H_est"], bt["y"], bt["sigma_n2"], bt["bits"])
    e_lm, e_cg = int(lm.counters["bit_errors"]), int(cg.counters["bit_errors"])
    lo, hi = wilson_interval(e_lm, nbits)
    assert abs(e_lm / nbits - e_cg / nbits) <= hi - lo
