"""BER sweep artefacts in the reference's wire format.

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

__all__ = ["write_ber_outputs", "write_manifest", "run_ber", "detectors_from", "ber_config_from"]

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
    return _BERConfig(channel=channel, detectors=tuple(detectors_from(cfg)),
                      snr_grid=tuple(float(s) for s in run.get("snr_db", [])), trials=int(run.get("trials", 1000)),
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
