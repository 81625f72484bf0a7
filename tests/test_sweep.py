"""BER artefacts in the reference's wire format (sweep.py vs the files the
reference's experiments.py:353-384 wrote for the same sweep,
tests/golden/ber_run/)."""

import os

import numpy as np
import pytest

import fpm_oracle as O
from conftest import GOLDEN
from paper_2504_09820_b200 import parallel as P
from paper_2504_09820_b200 import sweep

FMT = {"fp64": O.FP64, "fp32": O.FP32, "fp16": O.FP16, "bfloat16": O.BF16}
CFG = {"kind": "ber", "channel": {"M": 16, "K": 4, "zeta_r": 0.3, "zeta_t": 0.3},
       "detectors": [{"algorithm": "cg", "iters": 4},
                     {"algorithm": "fp_bj_cg", "L": 2, "matvec": "fp16", "inner": "fp16", "iters": 4},
                     {"algorithm": "fp_cg", "matvec": "bfloat16", "inner": "bfloat16", "iters": 5,
                      "label": "fpcg_bf16"},
                     {"algorithm": "lmmse"}],
       "run": {"snr_db": [0.0, 6.0], "trials": 40, "chunk": 16}}
SEED = 7


def _ref_simulate(cfg, snr_idx, ids):
    """The reference generator (restated bit-identically in the oracle)."""
    ch = cfg.channel
    H, y, bits, s2 = O.simulate(ch.M, ch.N, ch.zeta_t, cfg.snr_grid[snr_idx], ids, cfg.seed, point=snr_idx)
    return {"H": H, "H_est": H, "y": y, "bits": bits, "sigma_n2": s2}


def _oracle_counts(det, batch, cnt):
    import torch
    if det.algorithm == "lmmse":
        A, b = O.gram_mf(batch["H_est"], batch["y"], batch["sigma_n2"])
        x = O.lmmse(A, b)
        brk = div = np.full(len(x), -1)
    else:
        _, _, _, out = O.detect(batch["H_est"], batch["y"], batch["sigma_n2"], det.algorithm, det.iters, det.L,
                                FMT[det.work], FMT[det.matvec], FMT[det.inner])
        x, brk, div = out.x, out.breakdown_at, out.diverged_at
    cnt += torch.from_numpy(P.counters_from_arrays(O.demod16(x), batch["bits"], div, brk))


def _golden_files():
    d = os.path.join(GOLDEN, "ber_run")
    return {f: open(os.path.join(d, f)).read() for f in sorted(os.listdir(d))}


def _check(out):
    want = _golden_files()
    for f, text in want.items():
        assert open(os.path.join(out, f)).read() == text, f


def test_run_ber_artefacts_match_reference_files(tmp_path):
    import torch
    man = sweep.run_ber(CFG, tmp_path, SEED, simulate=_ref_simulate,
                        counts_fn=lambda d, b, c: _oracle_counts(d, b, c))
    _check(tmp_path)
    assert sorted(man["outputs"]) == sorted(_golden_files())
    assert man["kind"] == "ber" and man["seed"] == SEED and len(man["config_sha256"]) == 64
    assert os.path.exists(tmp_path / "manifest.json")
    del torch


def test_config_errors_are_contract_violations():
    from paper_2504_09820_b200.errors import ContractViolation
    with pytest.raises(ContractViolation):
        sweep.ber_config_from({"detectors": [{"algorithm": "cg"}]}, 1)
    with pytest.raises(ContractViolation):
        sweep.ber_config_from({"channel": {"M": 4, "K": 8}, "detectors": [{"algorithm": "cg"}]}, 1)
    with pytest.raises(ContractViolation):
        sweep.ber_config_from({"channel": {"M": 8, "K": 4}, "detectors": []}, 1)


@pytest.mark.gpu
def test_run_ber_on_gpu_reproduces_reference_files(tmp_path):
    """Same sweep, detection on the B200 (fused kernel / LMMSE comparator),
    inputs from the reference generator: the reference's files exactly."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sweep.run_ber(CFG, tmp_path, SEED, simulate=_ref_simulate)
    _check(tmp_path)
