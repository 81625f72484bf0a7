"""BER sweep artefacts in the reference's wire format.

    run_convergence(cfg, out, seed) <- experiments.py:281-325 (_run_convergence,
                                    with _mean_curves :236-278 and
                                    _run_detector_chunk :215-233): trial-mean
                                    residual / gap / symbol-MSE curves, the
                                    first trial's trace, summary.csv (SURVEY.md
                                    8(f) #3)
    run_experiment(cfg, out)     <- experiments.py:523-556 for the two kinds on
                                    the hot path ("ber", "convergence")
    run_ber(cfg, out, seed)      <- experiments.py:353-384 (_run_ber): the
                                    [channel] / [[detectors]] / [run] tables,
                                    swept on the GPU (sharded over ranks under
                                    torchrun), written as ber.csv +
                                    ber_plotdata_<detector>.csv + manifest.json
    write_ber_outputs(curves, out)  the CSV files (experiments.py:366-383)
    write_manifest(...)             manifest.json (experiments.py:544-555)

Values are formatted as the reference formats them (`repr` for floats,
experiments.py:74-77), so the files are byte-compatible with its outputs for
the same counts.
"""

from __future__ import annotations

import csv
import hashlib
import json
import time
from pathlib import Path

from .errors import ContractViolation

__all__ = ["write_ber_outputs", "write_manifest", "run_ber", "run_convergence", "run_experiment", "detectors_from",
           "ber_config_from", "iterations_to_match"]

BER_HEADER = ["detector", "precision_w", "precision_mv", "precision_ip", "L", "zeta", "snr_db", "iters", "trials",
              "bit_errors", "ber", "ci_low", "ci_high", "divergence_rate"]


def _fmt(value) -> str:
    """experiments.py:74-77."""
    if isinstance(value, float):
        return repr(value)
    return str(value)


def _write_csv(path: Path, header, rows) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        for row in rows:
            w.writerow([_fmt(v) for v in row])


def write_ber_outputs(curves, out) -> list[str]:
    """ber.csv and one ber_plotdata_<name>.csv per detector
    (experiments.py:366-383).  `curves`: BERCurve-like objects
    (.detector with name/work/matvec/inner/L/iters, .zeta, .points)."""
    out = Path(out)
    out.mkdir(parents=True, exist_ok=True)
    rows, files = [], []
    for curve in curves:
        det = curve.detector
        for p in curve.points:
            rows.append([det.name, det.work, det.matvec, det.inner, det.L or "", curve.zeta, p.snr_db, det.iters,
                         p.trials, p.bit_errors, p.ber, p.ci_low, p.ci_high, p.divergence_rate])
        pname = f"ber_plotdata_{det.name}.csv"
        _write_csv(out / pname, ["snr_db", "ber"], [[p.snr_db, p.ber] for p in curve.points])
        files.append(pname)
    _write_csv(out / "ber.csv", BER_HEADER, rows)
    files.append("ber.csv")
    return files


def write_manifest(kind: str, seed: int, cfg: dict, files, wall_time_s: float, out) -> dict:
    """manifest.json (experiments.py:544-555)."""
    from . import __version__
    blob = json.dumps(cfg, sort_keys=True, default=str).encode()
    manifest = {"kind": kind, "seed": seed, "config": cfg, "config_sha256": hashlib.sha256(blob).hexdigest(),
                "version": __version__, "wall_time_s": round(wall_time_s, 3), "outputs": list(files)}
    with open(Path(out) / "manifest.json", "w") as fh:
        json.dump(manifest, fh, indent=2, default=str)
    return manifest


class _Channel:
    def __init__(self, M, K, N_UE=1, zeta_r=0.0, zeta_t=0.0, block_diag_users=False):
        if M < 1 or K < 1 or N_UE < 1:
            raise ContractViolation("M, K, N_UE must be positive")
        self.M, self.K, self.N_UE = M, K, N_UE
        self.N = K * N_UE
        if self.N > M:
            raise ContractViolation(f"need N <= M, got N={self.N}, M={M}")
        for z in (zeta_r, zeta_t):
            if not 0.0 <= z < 1.0:
                raise ContractViolation("zeta must lie in [0, 1)")
        self.zeta_r, self.zeta_t, self.block_diag_users = zeta_r, zeta_t, block_diag_users


class _BERConfig:
    def __init__(self, channel, detectors, snr_grid, trials, seed, epsilon_db=None, snr_convention="receive_total",
                 chunk=1000, context=2):
        self.channel, self.detectors, self.snr_grid = channel, detectors, snr_grid
        self.trials, self.seed, self.epsilon_db = trials, seed, epsilon_db
        self.snr_convention, self.chunk, self.context = snr_convention, chunk, context


def detectors_from(cfg: dict):
    """[[detectors]] entries (experiments.py:111-133)."""
    from .detect import DetectorSpec
    entries = cfg.get("detectors")
    if not isinstance(entries, list) or not entries:
        raise ContractViolation("detectors: need at least one [[detectors]] entry")
    run_iters = cfg.get("run", {}).get("iters", 10)
    return [DetectorSpec(algorithm=str(e.get("algorithm", "")), iters=int(e.get("iters", run_iters)), L=e.get("L"),
                         work=str(e.get("work", "fp64")), matvec=str(e.get("matvec", "fp64")),
                         inner=str(e.get("inner", "fp64")), rtol=float(e.get("rtol", 1e-6)),
                         rho_update=str(e.get("rho_update", "as_written")), label=e.get("label"))
            for e in entries]


def ber_config_from(cfg: dict, seed: int):
    """The BERConfig _run_ber builds (experiments.py:353-365)."""
    ch = cfg.get("channel")
    if not isinstance(ch, dict):
        raise ContractViolation("channel: missing table")
    channel = _Channel(M=int(ch.get("M", 0)), K=int(ch.get("K", 0)), N_UE=int(ch.get("N_UE", 1)),
                       zeta_r=float(ch.get("zeta_r", 0.0)), zeta_t=float(ch.get("zeta_t", 0.0)),
                       block_diag_users=bool(ch.get("block_diag_users", False)))
    run = cfg.get("run", {})
    grid = run.get("snr_db", [])
    grid = [grid] if isinstance(grid, (int, float)) else grid
    return _BERConfig(channel=channel, detectors=tuple(detectors_from(cfg)),
                      snr_grid=tuple(float(s) for s in grid), trials=int(run.get("trials", 1000)),
                      seed=seed, epsilon_db=run.get("epsilon_db"),
                      snr_convention=run.get("snr_convention", "receive_total"), chunk=int(run.get("chunk", 1000)))


def run_ber(cfg: dict, out, seed: int, *, simulate=None, counts_fn=None) -> dict:
    """_run_ber on the GPU: inputs from channel.simulate_trials (unless
    `simulate` is given, e.g. the reference's own simulate_trials), detection
    by the fused kernel, counts all-reduced over ranks; rank 0 writes the
    artefacts.  Returns the manifest (rank 0) or {}."""
    from . import channel, parallel
    started = time.time()
    bc = ber_config_from(cfg, seed)
    if bc.trials < 1:
        raise ContractViolation("trials must be positive")
    curves = parallel.sharded_ber_sweep(bc, simulate or channel.simulate_trials, counts_fn=counts_fn)
    rank, _, _ = parallel.dist_info()
    if rank != 0:
        return {}
    files = write_ber_outputs(curves, out)
    return write_manifest(cfg.get("kind", "ber"), seed, cfg, files, time.time() - started, out)


def iterations_to_match(mean_curve, reference_level: float, margin: float = 1.1):
    """First sweep whose mean error reaches margin x the LMMSE level
    (detect.py:276-285), or None."""
    import numpy as np
    hits = np.nonzero(np.asarray(mean_curve) <= margin * reference_level)[0]
    return int(hits[0]) if hits.size else None


def _gpu_chunk(detectors, batch: dict, iters: int) -> dict:
    """_mean_curves._one (experiments.py:246-256) + _run_detector_chunk
    (:215-233) on the device: bit-exact Gram, LMMSE reference solution
    (fpm_lmmse), ||A||_2 by fpm_herm_norm2, the CG with recorded iterates and
    gaps.  Returns per-trial arrays on the host for the reference's
    chunk-ordered reductions."""
    import numpy as np
    from .detect import gram_mf
    from .solvers import _norm2_t, _to_dev, _torch, build_blocks_batch, herm_norm2, run_batch, solve_direct_batch
    torch = _torch()
    A, b = gram_mf(_to_dev(batch["H_est"], torch.complex128), _to_dev(batch["y"], torch.complex128),
                   batch["sigma_n2"])
    s = torch.as_tensor(batch["symbols"], device=A.device)
    x_hat = solve_direct_batch(A, b)
    a_norm = herm_norm2(A)
    lm_err = (_norm2_t(x_hat - s) ** 2).cpu().numpy()
    T = b.shape[0]
    out = {}
    for det in detectors:
        if det.algorithm == "lmmse":
            zero = np.zeros((iters + 1, T))
            out[det.name] = {"res": zero, "gap": zero, "mse": np.tile(lm_err, (iters + 1, 1)), "div": 0,
                             "alphas": None, "betas": None}
            continue
        blocks = build_blocks_batch(A, det.L) if det.algorithm == "fp_bj_cg" else None
        r = run_batch(A, b, iters, det.precision(), blocks=blocks, rho_update=det.rho_update, rtol=det.rtol,
                      x_ref=x_hat, a_norm=a_norm, record_gaps=True, record_iterates=True)
        mse = _norm2_t(r.iterates - s[None]) ** 2
        out[det.name] = {"res": r.residual_norms.cpu().numpy(), "gap": r.residual_gaps.cpu().numpy(),
                         "mse": mse.cpu().numpy(), "div": int((r.diverged_at >= 0).sum().item()),
                         "alphas": r.alphas[:, 0].cpu().numpy(), "betas": r.betas[:, 0].cpu().numpy()}
    out["_lmmse_mse"] = float(np.sum(lm_err))
    return out


def _mean_curves(bc, detectors, iters: int, simulate, chunk_fn):
    """_mean_curves (experiments.py:236-278): chunks dealt round-robin over
    ranks, per-chunk partials gathered and reduced on every rank in chunk
    order, exactly as the reference reduces its thread-pool partials, so the
    curves do not depend on the rank count."""
    import numpy as np
    from . import parallel
    rank, world, _ = parallel.dist_info()
    trials, chunk = bc.trials, bc.chunk
    chunks = [range(lo, min(lo + chunk, trials)) for lo in range(0, trials, chunk)]
    mine = {i: chunk_fn(detectors, simulate(bc, 0, ids), iters) for i, ids in enumerate(chunks) if i % world == rank}
    if world > 1:
        import torch.distributed as dist
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        mine = {k: v for g in gathered for k, v in g.items()}
    partials = [mine[i] for i in range(len(chunks))]
    curves = {}
    lmmse_level = sum(p["_lmmse_mse"] for p in partials) / trials
    for det in detectors:
        res = sum(np.sum(p[det.name]["res"], axis=1) for p in partials) / trials
        gap = sum(np.sum(p[det.name]["gap"], axis=1) for p in partials) / trials
        mse = sum(np.sum(p[det.name]["mse"], axis=1) for p in partials) / trials
        div = sum(p[det.name]["div"] for p in partials) / trials
        first = partials[0][det.name]
        curves[det.name] = {"res_norm": np.asarray(res), "gap": np.asarray(gap), "sym_mse": np.asarray(mse),
                            "divergence_rate": div,
                            "first_trace": {"res": np.asarray(first["res"])[:, 0],
                                            "gap": np.asarray(first["gap"])[:, 0],
                                            "alphas": first["alphas"], "betas": first["betas"]}}
    return curves, lmmse_level


def run_convergence(cfg: dict, out, seed: int, *, simulate=None, chunk_fn=None) -> dict:
    """_run_convergence (experiments.py:281-325) on the GPU: inputs from
    channel.simulate_trials at context 4 (unless `simulate` is given), the
    per-chunk work by `chunk_fn` (default _gpu_chunk), chunks sharded over
    ranks under torchrun.  Rank 0 writes convergence_<det>.csv,
    trace_<det>.csv, summary.csv and manifest.json; returns the manifest
    (rank 0) or {}."""
    from . import channel, parallel
    started = time.time()
    bc = ber_config_from(cfg, seed)   # channel + detectors (experiments.py:282-283)
    run = cfg.get("run", {})
    iters = int(run.get("iters", 40))
    trials = int(run.get("trials", 200))
    snr_db = float(run.get("snr_db", 20.0))
    margin = float(run.get("margin", 1.1))
    if iters < 1:
        raise ContractViolation("run.iters must be a positive iteration budget")
    if trials < 1:
        raise ContractViolation("run.trials must be a positive integer")
    bc.snr_grid, bc.trials, bc.chunk, bc.context = (snr_db,), trials, int(run.get("chunk", 500)), 4
    curves, lmmse_level = _mean_curves(bc, bc.detectors, iters, simulate or channel.simulate_trials,
                                       chunk_fn or _gpu_chunk)
    rank, _, _ = parallel.dist_info()
    if rank != 0:
        return {}
    out = Path(out)
    out.mkdir(parents=True, exist_ok=True)
    files, summary_rows = [], []
    for det in bc.detectors:
        mc = curves[det.name]
        name = f"convergence_{det.name}.csv"
        _write_csv(out / name, ["iter", "res_norm", "gap", "sym_mse"],
                   [[i, mc["res_norm"][i], mc["gap"][i], mc["sym_mse"][i]] for i in range(len(mc["res_norm"]))])
        files.append(name)
        tr = mc["first_trace"]
        rows = []
        for i in range(len(tr["res"])):
            alpha = tr["alphas"][i - 1] if tr["alphas"] is not None and i >= 1 else ""
            beta = tr["betas"][i - 1] if tr["betas"] is not None and i >= 1 else ""
            rows.append([i, tr["res"][i], tr["gap"][i], alpha, beta])
        tname = f"trace_{det.name}.csv"
        _write_csv(out / tname, ["iter", "res_norm", "gap", "alpha", "beta"], rows)
        files.append(tname)
        reached = iterations_to_match(mc["sym_mse"], lmmse_level, margin)
        summary_rows.append([det.name, det.work, det.matvec, det.inner, det.L or "", bc.channel.zeta_t, iters,
                             reached if reached is not None else "", mc["gap"][-1], mc["sym_mse"][-1],
                             mc["divergence_rate"], lmmse_level])
    _write_csv(out / "summary.csv",
               ["detector", "precision_w", "precision_mv", "precision_ip", "L", "zeta", "iters", "iters_to_lmmse",
                "final_gap", "final_sym_mse", "divergence_rate", "lmmse_mse"], summary_rows)
    files.append("summary.csv")
    return write_manifest(cfg.get("kind", "convergence"), seed, cfg, files, time.time() - started, out)


_RUNNERS = {"ber": run_ber, "convergence": run_convergence}


def run_experiment(cfg: dict, out, *, seed: int | None = None, **kw) -> dict:
    """run_experiment (experiments.py:523-556) for the hot-path kinds; the
    analysis-only kinds (heuristic, cost, break_even, gram_stats) are outside
    this package's scope and raise ContractViolation."""
    kind = cfg.get("kind")
    if kind not in _RUNNERS:
        raise ContractViolation(f"kind {kind!r} is not on the accelerated path (supported: {sorted(_RUNNERS)})")
    seed = int(cfg.get("seed", 0)) if seed is None else int(seed)
    return _RUNNERS[kind](cfg, out, seed, **kw)
