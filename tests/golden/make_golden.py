"""Generate golden vectors for the detector hot path FROM THE REFERENCE.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array below is produced by the reference package `fpmimo` itself
(simulate_trials / build_blocks_batch / run_batch / demodulate_16qam / the
error sum of run_ber_sweep, detect.py:189-262, solvers.py:232-393), so the
fixtures pin both the oracle (tests/test_oracle_golden.py, CPU) and the CUDA
path (tests/test_gpu_parity.py, B200).  Shapes follow BASELINE.json's configs
at fixture-sized batch counts; channel and SNR conventions are the
reference's (W ~ CN(0, 1/M), sigma^2 = (N/M) 10^(-snr/10)).  Seed 20261020.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from fpmimo.channel import ChannelConfig  # noqa: E402
from fpmimo.detect import (BERConfig, DetectorSpec, demodulate_16qam,  # noqa: E402
                           simulate_trials)
from fpmimo.formats import get_format, make_format  # noqa: E402
from fpmimo.linalg import axpy_fp, dot_fp, matvec_fp  # noqa: E402
from fpmimo.solvers import (PrecisionConfig, _BatchBlocks,  # noqa: E402
                            build_blocks_batch, run_batch)

SEED = 20261020
OUT = os.path.dirname(os.path.abspath(__file__))

# name: (M, K, zeta, snr_db, T, detector kwargs)
CASES = {
    "c1_cg_fp64": (128, 16, 0.0, 10.0, 48, dict(algorithm="cg", iters=8)),
    "c2_fpcg_fp16_snr0": (128, 32, 0.5, 0.0, 12, dict(algorithm="fp_cg", iters=10, matvec="fp16", inner="fp16")),
    "c2_fpcg_fp16_snr20": (128, 32, 0.5, 20.0, 12, dict(algorithm="fp_cg", iters=10, matvec="fp16", inner="fp16")),
    "c2_fpcg_bf16_snr10": (128, 32, 0.5, 10.0, 12, dict(algorithm="fp_cg", iters=10, matvec="bfloat16", inner="bfloat16")),
    "c3_bj4_fp16": (256, 64, 0.7, 20.0, 4, dict(algorithm="fp_bj_cg", iters=6, L=4, matvec="fp16", inner="fp16")),
    "c4_bj8_fp16": (512, 128, 0.8, 25.0, 2, dict(algorithm="fp_bj_cg", iters=8, L=8, matvec="fp16", inner="fp16")),
    "c5_bj4_fp16": (128, 64, 0.5, 15.0, 8, dict(algorithm="fp_bj_cg", iters=8, L=4, matvec="fp16", inner="fp16")),
    "c5_bj4_fp64": (128, 64, 0.5, 15.0, 8, dict(algorithm="fp_bj_cg", iters=8, L=4)),
    "c5_bj4_textbook_fp32": (128, 64, 0.5, 15.0, 4, dict(algorithm="fp_bj_cg", iters=8, L=4, matvec="fp32", inner="fp32", rho_update="textbook")),
    "mix_w32_mv16_ip16": (64, 16, 0.5, 10.0, 8, dict(algorithm="fp_cg", iters=12, work="fp32", matvec="fp16", inner="fp16")),
    "mix_w64_mv16_ip32_bj2": (64, 16, 0.8, 12.0, 8, dict(algorithm="fp_bj_cg", iters=10, L=2, matvec="fp16", inner="fp32")),
    "mix_w16_all_bj4": (64, 16, 0.3, 8.0, 8, dict(algorithm="fp_bj_cg", iters=6, L=4, work="fp16", matvec="fp16", inner="fp16")),
}


def _detector_case(name, M, K, zeta, snr, T, kw):
    ch = ChannelConfig(M=M, K=K, N_UE=1, zeta_r=zeta, zeta_t=zeta)
    det = DetectorSpec(**kw)
    cfg = BERConfig(channel=ch, detectors=(det,), snr_grid=(snr,), trials=T, seed=SEED)
    batch = simulate_trials(cfg, 0, range(T))
    A, b = batch["A"], batch["b"]
    blocks = build_blocks_batch(A, det.L) if det.algorithm == "fp_bj_cg" else None
    res = run_batch(A, b, det.iters, det.precision(), blocks=blocks,
                    rho_update=det.rho_update, rtol=det.rtol)
    got = demodulate_16qam(res.x)
    errs = (got != batch["bits"]).sum(-1).astype(np.int64)
    prec = det.precision()
    out = dict(
        H=batch["H_est"], y=batch["y"], sigma2=np.float64(batch["sigma_n2"]),
        tx_bits=batch["bits"], A=A, b=b, x=res.x,
        breakdown_at=res.breakdown_at, diverged_at=res.diverged_at,
        converged_at=res.converged_at, residual_norms=res.residual_norms,
        rx_bits=got, bit_errors=errs, iters=np.int64(det.iters),
        L=np.int64(det.L or 0), rho_update=np.array(det.rho_update),
        algorithm=np.array(det.algorithm),
        fmts=np.array([[f.sig_bits, f.exp_bits, int(f.subnormals_enabled)]
                       for f in (prec.work, prec.matvec, prec.inner)], np.int64),
    )
    if blocks is not None:
        out["Minv"] = np.concatenate([m.reshape(T, -1) for m in blocks.mats], axis=1)
    return out


def _solver_edge_cases():
    """Flag semantics of run_batch (solvers.py:342-357) on crafted systems."""
    rng = np.random.default_rng(5)
    N = 8
    B = rng.standard_normal((4, 16, N)) + 1j * rng.standard_normal((4, 16, N))
    A = np.einsum("tmi,tmj->tij", B.conj(), B) / 16 + 0.1 * np.eye(N)
    A = 0.5 * (A + np.swapaxes(A.conj(), -1, -2))
    b = rng.standard_normal((4, N)) + 1j * rng.standard_normal((4, N))
    A[1] = -A[1]                 # negative definite -> breakdown at 1
    b[2] = 0                     # rho == 0 -> stall, x stays 0
    b[3] = b[3] * 1e8            # fp16 overflow -> diverged
    out = {}
    for tag, prec in (("fp16", PrecisionConfig(matvec=get_format("fp16"), inner=get_format("fp16"))),
                      ("p5e4", PrecisionConfig(matvec=make_format(5, 4), inner=make_format(6, 5))),
                      ("fp64", PrecisionConfig())):
        res = run_batch(A, b, 6, prec)
        out[f"{tag}_x"] = res.x
        out[f"{tag}_breakdown_at"] = res.breakdown_at
        out[f"{tag}_diverged_at"] = res.diverged_at
        out[f"{tag}_fmts"] = np.array([[f.sig_bits, f.exp_bits, int(f.subnormals_enabled)]
                                       for f in (prec.work, prec.matvec, prec.inner)], np.int64)
    # ragged block-Jacobi (L=3 on N=8), all fp64, both rho variants
    Ap = A[[0]].repeat(2, 0)
    bp = b[[0]].repeat(2, 0)
    blocks = build_blocks_batch(Ap, 3, allow_ragged=True)
    for rv in ("as_written", "textbook"):
        res = run_batch(Ap, bp, 5, PrecisionConfig(matvec=get_format("fp16"), inner=get_format("fp16")),
                        blocks=blocks, rho_update=rv)
        out[f"ragged_{rv}_x"] = res.x
    out["ragged_Minv"] = np.concatenate([m.reshape(2, -1) for m in blocks.mats], axis=1)
    out["A"], out["b"] = A, b
    out["ragged_A"], out["ragged_b"] = Ap, bp
    return out


def _kernel_kats():
    """matvec_fp / dot_fp / axpy_fp (linalg.py:45-119) per registry format."""
    rng = np.random.default_rng(7)
    A = (rng.standard_normal((6, 24, 24)) + 1j * rng.standard_normal((6, 24, 24))) * 3.0
    v = rng.standard_normal((6, 24)) + 1j * rng.standard_normal((6, 24))
    a = rng.standard_normal(6) + 1j * rng.standard_normal(6)
    out = dict(A=A, v=v, a=a)
    for name in ("fp64", "fp32", "fp16", "bfloat16"):
        f = get_format(name)
        out[f"matvec_{name}"] = matvec_fp(A, v, f)
        out[f"dot_{name}"] = dot_fp(A[:, 0, :], v, f)
        out[f"axpy_{name}"] = axpy_fp(a, A[:, 1, :], v, f)
    return out


def _cg_history():
    """run_batch's full BatchResult (solvers.py:188-204, 306-393): residual /
    iterate norm histories, alphas, betas, b_norm, converged_at and the
    record_iterates / record_residual_vectors / record_gaps outputs, on the
    crafted flag systems (breakdown, stall, divergence lanes) and on a c5
    block-Jacobi batch."""
    e = _solver_edge_cases()
    A, b = e["A"], e["b"]
    out = {"edge_A": A, "edge_b": b}
    x_ref = np.linalg.solve(A, b[..., None])[..., 0]
    for tag, prec in (("fp16", PrecisionConfig(matvec=get_format("fp16"), inner=get_format("fp16"))),
                      ("fp64", PrecisionConfig())):
        res = run_batch(A, b, 6, prec, x_ref=x_ref, record_gaps=True, record_iterates=True,
                        record_residual_vectors=True, rtol=1e-3)
        for k in ("x", "residual_norms", "iterate_norms", "alphas", "betas", "b_norm", "converged_at",
                  "breakdown_at", "diverged_at", "residual_gaps", "iterates", "residual_vectors"):
            out[f"edge_{tag}_{k}"] = getattr(res, k)
    out["edge_x_ref"] = x_ref
    d = _detector_case("c5_hist", 128, 64, 0.5, 15.0, 4,
                       dict(algorithm="fp_bj_cg", iters=8, L=4, matvec="fp16", inner="fp16"))
    A5, b5 = d["A"], d["b"]
    blocks = build_blocks_batch(A5, 4)
    res = run_batch(A5, b5, 8, PrecisionConfig(matvec=get_format("fp16"), inner=get_format("fp16")), blocks=blocks,
                    record_iterates=True, record_residual_vectors=True, rtol=1e-2)
    out["c5_A"], out["c5_b"] = A5, b5
    out["c5_Minv"] = np.concatenate([m.reshape(4, -1) for m in blocks.mats], axis=1)
    for k in ("x", "residual_norms", "iterate_norms", "alphas", "betas", "b_norm", "converged_at",
              "iterates", "residual_vectors"):
        out[f"c5_{k}"] = getattr(res, k)
    return out


def _lmmse():
    """The direct comparator (detect.py:230-231 -> linalg.py:223-231) on a
    c5-shaped and a c2-shaped batch."""
    from fpmimo.linalg import _solve_direct_batch
    out = {}
    for tag, (M, K, zeta, snr, T) in (("c5", (128, 64, 0.5, 15.0, 8)), ("c2", (128, 32, 0.5, 4.0, 8))):
        ch = ChannelConfig(M=M, K=K, N_UE=1, zeta_r=zeta, zeta_t=zeta)
        det = DetectorSpec("lmmse")
        cfg = BERConfig(channel=ch, detectors=(det,), snr_grid=(snr,), trials=T, seed=SEED)
        batch = simulate_trials(cfg, 0, range(T))
        x = _solve_direct_batch(batch["A"], batch["b"])
        got = demodulate_16qam(x)
        out.update({f"{tag}_H": batch["H_est"], f"{tag}_y": batch["y"], f"{tag}_sigma2": np.float64(batch["sigma_n2"]),
                    f"{tag}_A": batch["A"], f"{tag}_b": batch["b"], f"{tag}_x": x, f"{tag}_tx_bits": batch["bits"],
                    f"{tag}_rx_bits": got, f"{tag}_bit_errors": (got != batch["bits"]).sum(-1).astype(np.int64)})
    return out


BER_RUN_CFG = {"kind": "ber", "channel": {"M": 16, "K": 4, "zeta_r": 0.3, "zeta_t": 0.3},
               "detectors": [{"algorithm": "cg", "iters": 4},
                             {"algorithm": "fp_bj_cg", "L": 2, "matvec": "fp16", "inner": "fp16", "iters": 4},
                             {"algorithm": "fp_cg", "matvec": "bfloat16", "inner": "bfloat16", "iters": 5,
                              "label": "fpcg_bf16"},
                             {"algorithm": "lmmse"}],
               "run": {"snr_db": [0.0, 6.0], "trials": 40, "chunk": 16}}


def _ber_run():
    """The reference's BER artefacts (experiments.py:353-384) for a small
    sweep: ber.csv + ber_plotdata_<detector>.csv, written by its own code."""
    import tempfile
    from pathlib import Path
    from fpmimo.experiments import _run_ber
    out = {}
    with tempfile.TemporaryDirectory() as d:
        files = _run_ber(BER_RUN_CFG, Path(d), 7, 1)
        for f in files:
            out[f] = (Path(d) / f).read_text()
    return out


CONV_RUN_CFG = {"kind": "convergence", "channel": {"M": 16, "K": 4, "zeta_r": 0.3, "zeta_t": 0.3},
                "detectors": [{"algorithm": "cg"},
                              {"algorithm": "fp_bj_cg", "L": 2, "matvec": "fp16", "inner": "fp16"},
                              {"algorithm": "fp_cg", "matvec": "bfloat16", "inner": "bfloat16",
                               "rho_update": "textbook", "label": "fpcg_bf16_tb"},
                              {"algorithm": "lmmse"}],
                "run": {"trials": 40, "iters": 6, "snr_db": 10.0, "chunk": 16}}


def _conv_run():
    """The reference's convergence artefacts (experiments.py:281-325):
    convergence_/trace_<detector>.csv + summary.csv, written by its own code."""
    import tempfile
    from pathlib import Path
    from fpmimo.experiments import _run_convergence
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for f in _run_convergence(CONV_RUN_CFG, Path(d), 7, 1):
            out[f] = (Path(d) / f).read_text()
    return out


def _write_run(name, files):
    os.makedirs(os.path.join(OUT, name), exist_ok=True)
    for f, text in files.items():
        with open(os.path.join(OUT, name, f), "w") as fh:
            fh.write(text)


def main():
    if "--runs-only" in sys.argv:
        _write_run("ber_run", _ber_run())
        _write_run("conv_run", _conv_run())
        return
    for name, (M, K, zeta, snr, T, kw) in CASES.items():
        d = _detector_case(name, M, K, zeta, snr, T, kw)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
        print(name, "T", T, "errors", int(d["bit_errors"].sum()),
              "diverged", int((d["diverged_at"] >= 0).sum()))
    np.savez_compressed(os.path.join(OUT, "solver_edges.npz"), **_solver_edge_cases())
    np.savez_compressed(os.path.join(OUT, "kernel_kats.npz"), **_kernel_kats())
    np.savez_compressed(os.path.join(OUT, "hist_cg.npz"), **_cg_history())
    np.savez_compressed(os.path.join(OUT, "lmmse.npz"), **_lmmse())
    _write_run("ber_run", _ber_run())
    _write_run("conv_run", _conv_run())
    # slicer known answers (detect.py:70-84, tests/test_detect.py:55-69)
    vals = np.array([complex(np.nan, 1.0), complex(np.inf, np.inf), complex(-np.inf, -np.inf),
                     -2 / np.sqrt(10), 0.0, 2 / np.sqrt(10), complex(0.3, -0.9), complex(-0.0, 0.0)])
    np.savez_compressed(os.path.join(OUT, "slicer.npz"), x=vals, bits=demodulate_16qam(vals))


if __name__ == "__main__":
    main()
