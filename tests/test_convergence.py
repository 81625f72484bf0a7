"""Convergence-trace artefacts (sweep.run_convergence vs the files the
reference's experiments.py:281-325 wrote for the same study,
tests/golden/conv_run/).

CPU: the per-chunk work is the oracle, so the files must be byte-identical
(pins the wire format, the chunk-ordered reductions and the gloo sharding).
GPU: the per-chunk work is the CUDA path; the CG iterates / alphas / betas
are bit-exact, the norms within a few ulps (CUDA hypot vs libm), the gaps and
the LMMSE level within the Cholesky / Lanczos-norm tolerance."""

import csv
import io
import os
import socket
import tempfile

import numpy as np
import pytest

import fpm_oracle as O
from conftest import GOLDEN
from paper_2504_09820_b200 import sweep

FMT = {"fp64": O.FP64, "fp32": O.FP32, "fp16": O.FP16, "bfloat16": O.BF16}
CFG = {"kind": "convergence", "channel": {"M": 16, "K": 4, "zeta_r": 0.3, "zeta_t": 0.3},
       "detectors": [{"algorithm": "cg"},
                     {"algorithm": "fp_bj_cg", "L": 2, "matvec": "fp16", "inner": "fp16"},
                     {"algorithm": "fp_cg", "matvec": "bfloat16", "inner": "bfloat16", "rho_update": "textbook",
                      "label": "fpcg_bf16_tb"},
                     {"algorithm": "lmmse"}],
       "run": {"trials": 40, "iters": 6, "snr_db": 10.0, "chunk": 16}}
SEED = 7


def _ref_simulate(cfg, snr_idx, ids):
    """The reference generator (restated bit-identically in the oracle)."""
    ch = cfg.channel
    H, y, bits, s2 = O.simulate(ch.M, ch.N, ch.zeta_t, cfg.snr_grid[snr_idx], ids, cfg.seed, point=snr_idx,
                                context=cfg.context)
    return {"H": H, "H_est": H, "y": y, "bits": bits, "symbols": O.mod16(bits), "sigma_n2": s2}


def _oracle_chunk(detectors, batch, iters):
    """experiments.py:215-256 with the oracle as the arithmetic."""
    A, b = O.gram_mf(batch["H_est"], batch["y"], batch["sigma_n2"])
    s = batch["symbols"]
    x_hat = O.lmmse(A, b)
    w = np.linalg.eigvalsh(A)
    a_norm = np.maximum(np.abs(w[:, 0]), np.abs(w[:, -1]))
    out = {}
    for det in detectors:
        if det.algorithm == "lmmse":
            err = O._norm2(x_hat - s) ** 2
            zero = np.zeros((iters + 1, s.shape[0]))
            out[det.name] = {"res": zero, "gap": zero, "mse": np.tile(err, (iters + 1, 1)), "div": 0,
                             "alphas": None, "betas": None}
            continue
        mats = O.bj_inverses(A, det.L) if det.algorithm == "fp_bj_cg" else None
        fm = (O.FP64, O.FP64, O.FP64) if det.algorithm == "cg" else (FMT[det.work], FMT[det.matvec], FMT[det.inner])
        r = O.cg_batch(A, b, iters, *fm, mats=mats, rho_update=det.rho_update, rtol=det.rtol, x_ref=x_hat,
                       a_norm=a_norm, record=True)
        out[det.name] = {"res": r.residual_norms, "gap": r.residual_gaps,
                         "mse": O._norm2(r.iterates - s[None]) ** 2, "div": int(np.sum(r.diverged_at >= 0)),
                         "alphas": r.alphas[:, 0], "betas": r.betas[:, 0]}
    out["_lmmse_mse"] = float(np.sum(O._norm2(x_hat - s) ** 2))
    return out


def _golden():
    d = os.path.join(GOLDEN, "conv_run")
    return {f: open(os.path.join(d, f)).read() for f in sorted(os.listdir(d))}


def test_oracle_run_matches_reference_files(tmp_path):
    man = sweep.run_convergence(CFG, tmp_path, SEED, simulate=_ref_simulate, chunk_fn=_oracle_chunk)
    for f, text in _golden().items():
        assert open(tmp_path / f).read() == text, f
    assert sorted(man["outputs"]) == sorted(_golden())
    assert man["kind"] == "convergence" and man["seed"] == SEED


def test_run_experiment_dispatch(tmp_path):
    from paper_2504_09820_b200.errors import ContractViolation
    man = sweep.run_experiment(dict(CFG, seed=SEED), tmp_path, simulate=_ref_simulate, chunk_fn=_oracle_chunk)
    assert man["seed"] == SEED and "summary.csv" in man["outputs"]
    with pytest.raises(ContractViolation):
        sweep.run_experiment({"kind": "cost"}, tmp_path)
    with pytest.raises(ContractViolation):
        sweep.run_convergence(dict(CFG, run={"iters": 0}), tmp_path, SEED, simulate=_ref_simulate,
                              chunk_fn=_oracle_chunk)


def test_iterations_to_match():
    assert sweep.iterations_to_match([3.0, 2.0, 1.05, 1.0], 1.0) == 2
    assert sweep.iterations_to_match([3.0, 2.0], 1.0) is None
    assert sweep.iterations_to_match([0.5], 1.0, margin=0.4) is None


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        sweep.run_convergence(CFG, out_dir, SEED, simulate=_ref_simulate, chunk_fn=_oracle_chunk)
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_run_matches_reference_files(world):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _port(), d), nprocs=world, join=True, start_method="spawn")
        for f, text in _golden().items():
            assert open(os.path.join(d, f)).read() == text, f


def _rows(text):
    return list(csv.reader(io.StringIO(text)))


def _num(v):
    if v.startswith("np.float64("):
        v = v[len("np.float64("):-1]
    return float(v)


@pytest.mark.gpu
def test_gpu_run_reproduces_reference_files(tmp_path):
    """Same study with the per-chunk work on the B200."""
    sweep.run_convergence(CFG, tmp_path, SEED, simulate=_ref_simulate)
    for f, text in _golden().items():
        want, got = _rows(text), _rows(open(tmp_path / f).read())
        assert len(want) == len(got) and want[0] == got[0], f
        head = want[0]
        for rw, rg in zip(want[1:], got[1:]):
            for col, a, b in zip(head, rw, rg):
                if col in ("alpha", "beta", "iter", "detector", "precision_w", "precision_mv", "precision_ip", "L",
                           "zeta", "iters", "iters_to_lmmse", "divergence_rate"):
                    assert a == b, (f, col, a, b)        # bit-exact CG scalars, labels, counts
                elif col in ("res_norm", "sym_mse", "final_sym_mse"):
                    tol = 1e-9 if f.endswith("lmmse.csv") else 1e-12
                    assert _num(b) == pytest.approx(_num(a), rel=tol, abs=1e-300), (f, col, a, b)
                elif col in ("gap", "final_gap"):         # ||b - Ax - r||: einsum order, LMMSE x_ref, eigvalsh
                    assert _num(b) == pytest.approx(_num(a), rel=1e-6, abs=1e-14), (f, col, a, b)
                elif col == "lmmse_mse":
                    assert _num(b) == pytest.approx(_num(a), rel=1e-9), (f, col, a, b)
                else:
                    raise AssertionError(col)


@pytest.mark.gpu
@pytest.mark.parametrize("M,N", [(128, 16), (128, 32), (128, 64), (512, 128), (24, 5)])
def test_diagnostic_kernels_against_numpy(M, N):
    """fpm_herm_norm2 (Lanczos + Sturm multisection) vs np.linalg.norm(A, 2)
    (experiments.py:246-256) and fpm_residual_gaps vs the reference formula
    ||b - A x_i - r_i|| / scale (solvers.py:289-294, 375-377) on Gram matrices
    of every BASELINE size, an odd size, and indefinite / degenerate Hermitian
    matrices."""
    import ctypes  # noqa: F401
    import torch
    from paper_2504_09820_b200 import _lib
    from paper_2504_09820_b200.solvers import _stream, herm_norm2
    rng = np.random.default_rng(5 + N)
    T = 37
    H = (rng.standard_normal((T, M, N)) + 1j * rng.standard_normal((T, M, N))) / np.sqrt(2 * M)
    A = np.einsum("tmi,tmj->tij", H.conj(), H) + 0.05 * np.eye(N)
    A = 0.5 * (A + A.conj().transpose(0, 2, 1))
    # indefinite (largest |lambda| negative), identity (Lanczos ends after one step), repeated top eigenvalue
    Q = np.linalg.qr(rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N)))[0]
    lam = np.linspace(-3.0, 1.0, N)
    A[0] = (Q * lam) @ Q.conj().T
    A[0] = 0.5 * (A[0] + A[0].conj().T)
    A[1] = np.eye(N)
    lam2 = np.linspace(0.1, 1.0, N)
    lam2[-2:] = 2.5
    A[2] = (Q * lam2) @ Q.conj().T
    A[2] = 0.5 * (A[2] + A[2].conj().T)
    ref = np.array([np.linalg.norm(a, 2) for a in A])
    got = herm_norm2(A).cpu().numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-10)

    iters = 4
    b = rng.standard_normal((T, N)) + 1j * rng.standard_normal((T, N))
    xit = rng.standard_normal((iters + 1, T, N)) + 1j * rng.standard_normal((iters + 1, T, N))
    rit = b[None] - np.einsum("tnk,itk->itn", A, xit) + 1e-9 * (rng.standard_normal((iters + 1, T, N)) + 0j)
    scale = ref * np.linalg.norm(xit[-1], axis=1)
    want = np.linalg.norm(b[None] - np.einsum("tnk,itk->itn", A, xit) - rit, axis=2) / scale
    dev = torch.device("cuda", 0)
    d = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)  # noqa: E731
    Ad, bd, xd, rd, sd = d(A, torch.complex128), d(b, torch.complex128), d(xit, torch.complex128), \
        d(rit, torch.complex128), d(scale, torch.float64)
    gaps = torch.zeros((iters + 1, T), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().fpm_residual_gaps(Ad.data_ptr(), bd.data_ptr(), xd.data_ptr(), rd.data_ptr(), sd.data_ptr(),
                                             T, N, iters, gaps.data_ptr(), _stream()), "gaps")
    g = gaps.cpu().numpy()
    assert np.all(g[0] == 0.0)
    np.testing.assert_allclose(g[1:], want[1:], rtol=1e-6, atol=1e-18)
