"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden vectors and the oracle.  Run on a B200: pytest -m gpu.

Bars (BASELINE.json north_star):
  * Gram / matched filter, x_hat with injected block inverses, flags, sliced
    bits, error counts: BIT-EXACT.
  * x_hat with on-chip (GPU fp64 Cholesky) block inverses: normwise relative
    difference per realization <= 1e-12 for fp64 paths and <= 2**-(p-2) for
    p-bit paths (p = stored fraction bits: fp16 10, bf16 7, fp32 23); sliced
    bits identical.
"""

import os

import numpy as np
import pytest

from conftest import bits_equal, golden_cases, knob_child, load_golden, run_knob_child, save_child_out

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_09820_b200 import build
    build.build()


def _spec_from_golden(g):
    from paper_2504_09820_b200.detect import DetectorSpec
    names = {(53, 11): "fp64", (24, 8): "fp32", (11, 5): "fp16", (8, 8): "bfloat16"}
    w, mv, ip = (names[(int(r[0]), int(r[1]))] for r in g["fmts"])
    L = int(g["L"]) or None
    return DetectorSpec(str(g["algorithm"]), iters=int(g["iters"]), L=L, work=w, matvec=mv, inner=ip,
                        rho_update=str(g["rho_update"]))


# norm2 (linalg.py:122-134) runs through hypot and a pairwise sum in NumPy,
# through CUDA hypot and a sequential sum here: a few ulps apart
NORM_RTOL = 1e-14


def _prec_tol(g):
    sig = int(g["fmts"][1][0])          # matvec significand bits incl. hidden
    return 1e-12 if sig == 53 else 2.0 ** -(sig - 1 - 2)


@pytest.mark.parametrize("name", golden_cases())
def test_gram_bit_exact(name):
    from paper_2504_09820_b200.detect import gram_mf
    g = load_golden(name)
    A, b = gram_mf(g["H"], g["y"], float(g["sigma2"]))
    assert bits_equal(A, g["A"])
    assert bits_equal(b, g["b"])


@pytest.mark.parametrize("name", golden_cases())
def test_fused_detect_bit_exact_injected_blocks(name):
    from paper_2504_09820_b200.detect import detect
    g = load_golden(name)
    det = _spec_from_golden(g)
    res = detect(det, g["H"], g["y"], float(g["sigma2"]), g["tx_bits"], minv=g.get("Minv"), want_bits=True)
    assert bits_equal(res.x, g["x"])
    np.testing.assert_array_equal(res.breakdown_at, g["breakdown_at"])
    np.testing.assert_array_equal(res.diverged_at, g["diverged_at"])
    np.testing.assert_array_equal(res.bits, g["rx_bits"])
    assert res.counters["bit_errors"] == int(g["bit_errors"].sum())
    assert res.counters["trials"] == g["H"].shape[0]
    assert res.counters["diverged"] == int((g["diverged_at"] >= 0).sum())


@pytest.mark.parametrize("name", golden_cases())
def test_fused_detect_onchip_blocks(name):
    from paper_2504_09820_b200.detect import detect
    g = load_golden(name)
    det = _spec_from_golden(g)
    res = detect(det, g["H"], g["y"], float(g["sigma2"]), g["tx_bits"], want_bits=True)
    if "Minv" not in g:
        assert bits_equal(res.x, g["x"])
    rel = np.linalg.norm(res.x - g["x"], axis=1) / np.linalg.norm(g["x"], axis=1)
    assert rel.max() <= _prec_tol(g), rel.max()
    np.testing.assert_array_equal(res.bits, g["rx_bits"])
    assert res.counters["bit_errors"] == int(g["bit_errors"].sum())


@pytest.mark.parametrize("name", golden_cases())
def test_run_batch_bit_exact(name):
    from paper_2504_09820_b200.solvers import BatchBlocks, run_batch
    g = load_golden(name)
    det = _spec_from_golden(g)
    N = g["b"].shape[1]
    blocks = BatchBlocks(g["Minv"], N, int(g["L"])) if "Minv" in g else None
    res = run_batch(g["A"], g["b"], det.iters, det.precision(), blocks, rho_update=det.rho_update)
    assert bits_equal(res.x, g["x"])
    np.testing.assert_array_equal(res.breakdown_at, g["breakdown_at"])
    np.testing.assert_array_equal(res.diverged_at, g["diverged_at"])
    # norm histories: NumPy's hypot / pairwise sum vs a sequential sum
    np.testing.assert_allclose(res.residual_norms, g["residual_norms"], rtol=NORM_RTOL, atol=0)
    np.testing.assert_array_equal(res.converged_at, g["converged_at"])


@pytest.mark.parametrize("name", [n for n in golden_cases() if "bj" in n])
def test_block_inverses_close_to_lapack(name):
    from paper_2504_09820_b200.solvers import build_blocks_batch
    g = load_golden(name)
    bb = build_blocks_batch(g["A"], int(g["L"]))
    np.testing.assert_allclose(bb.packed, g["Minv"], rtol=1e-11, atol=1e-13)


def test_generic_emulation_path_matches_native():
    """The integer RNE emulation kernels (any (sig, exp); knob
    FPM_FORCE_GENERIC in a fresh process) reproduce the reference's bits,
    i.e. what the native fp16/bf16/fp32 kernels give (test_golden_*)."""
    run_knob_child("tests/test_gpu_parity.py::test_child_generic_emulation", {"FPM_FORCE_GENERIC": "1"})


@knob_child
def test_child_generic_emulation():
    from paper_2504_09820_b200.detect import detect
    for name in ("c2_fpcg_fp16_snr0", "c2_fpcg_bf16_snr10", "c5_bj4_textbook_fp32", "mix_w16_all_bj4",
                 "mix_w32_mv16_ip16"):
        g = load_golden(name)
        det = _spec_from_golden(g)
        res = detect(det, g["H"], g["y"], float(g["sigma2"]), g["tx_bits"], minv=g.get("Minv"))
        assert bits_equal(res.x, g["x"]), name


def test_solver_edge_flags():
    from paper_2504_09820_b200.formats import FP16, make_format
    from paper_2504_09820_b200.solvers import BatchBlocks, PrecisionConfig, run_batch
    g = load_golden("solver_edges")
    precs = {"fp16": PrecisionConfig(matvec=FP16, inner=FP16),
             "p5e4": PrecisionConfig(matvec=make_format(5, 4), inner=make_format(6, 5)),
             "fp64": PrecisionConfig()}
    for tag, prec in precs.items():
        res = run_batch(g["A"], g["b"], 6, prec)
        assert bits_equal(res.x, g[f"{tag}_x"]), tag
        np.testing.assert_array_equal(res.breakdown_at, g[f"{tag}_breakdown_at"])
        np.testing.assert_array_equal(res.diverged_at, g[f"{tag}_diverged_at"])
    for rv in ("as_written", "textbook"):
        res = run_batch(g["ragged_A"], g["ragged_b"], 5, precs["fp16"], BatchBlocks(g["ragged_Minv"], 8, 3),
                        rho_update=rv)
        assert bits_equal(res.x, g[f"ragged_{rv}_x"]), rv


def test_slicer_known_answers():
    from paper_2504_09820_b200.detect import demodulate_16qam
    g = load_golden("slicer")
    np.testing.assert_array_equal(demodulate_16qam(g["x"]), g["bits"])


def test_nonpd_block_raises():
    from paper_2504_09820_b200.errors import ContractViolation
    from paper_2504_09820_b200.solvers import build_blocks_batch
    A = np.tile(np.eye(8, dtype=np.complex128), (3, 1, 1))
    A[1, 4, 4] = -1.0
    with pytest.raises(ContractViolation):
        build_blocks_batch(A, 4)


def _oracle_inputs(M, N, zeta, snr, T, seed=20261020, qam=16):
    import fpm_oracle as O
    return O.simulate(M, N, zeta, snr, range(T), seed, qam=qam)


@pytest.mark.parametrize("cfg", [
    # (M, N, zeta, snr, T, algorithm, L, iters, mv)
    (128, 16, 0.0, 10.0, 300, "cg", None, 8, "fp64"),
    (128, 32, 0.5, 6.0, 160, "fp_cg", None, 10, "fp16"),
    (128, 64, 0.5, 15.0, 48, "fp_bj_cg", 4, 8, "fp16"),
    (128, 64, 0.5, 15.0, 48, "fp_bj_cg", 4, 8, "fp64"),
    (96, 24, 0.6, 12.0, 40, "fp_bj_cg", 6, 7, "fp32"),   # N not a multiple of 8
    (64, 12, 0.3, 9.0, 70, "fp_cg", None, 5, "bfloat16"),
])
def test_random_batches_against_oracle(cfg):
    import fpm_oracle as O
    from paper_2504_09820_b200.detect import DetectorSpec, detect
    M, N, zeta, snr, T, alg, L, iters, mv = cfg
    H, y, bits, s2 = _oracle_inputs(M, N, zeta, snr, T)
    det = DetectorSpec(alg, iters=iters, L=L, matvec=mv, inner=mv)
    fm = O.REGISTRY[mv]
    A, b = O.gram_mf(H, y, s2)
    mats = O.bj_inverses(A, L) if alg == "fp_bj_cg" else None
    work = O.FP64
    ref = O.cg_batch(A, b, iters, work, fm if alg != "cg" else O.FP64, fm if alg != "cg" else O.FP64, mats)
    res = detect(det, H, y, s2, bits, minv=mats, want_bits=True)
    assert bits_equal(res.x, ref.x)
    np.testing.assert_array_equal(res.diverged_at, ref.diverged_at)
    ob = O.demod16(ref.x)
    np.testing.assert_array_equal(res.bits, ob)
    assert res.counters["bit_errors"] == int(O.bit_errors(ob, bits).sum())


def test_chunking_and_host_pipeline_invariance():
    """Counts do not depend on batching (tests/test_detect.py:133-140 analogue)
    and the host-buffer pipeline equals the device call."""
    from paper_2504_09820_b200.detect import DetectorSpec, detect, detect_host
    H, y, bits, s2 = _oracle_inputs(128, 64, 0.5, 15.0, 200)
    det = DetectorSpec("fp_bj_cg", iters=8, L=4, matvec="fp16", inner="fp16")
    full = detect(det, H, y, s2, bits, want_bits=True)
    parts = [detect(det, H[a:a + 37], y[a:a + 37], s2, bits[a:a + 37]) for a in range(0, 200, 37)]
    assert sum(p.counters["bit_errors"] for p in parts) == full.counters["bit_errors"]
    assert bits_equal(np.concatenate([p.x for p in parts]), full.x)
    hp = detect_host(det, H, y, s2, bits, want_bits=True, chunk=64)
    assert bits_equal(hp.x, full.x)
    np.testing.assert_array_equal(hp.bits, full.bits)
    assert hp.counters == full.counters


def test_qam64_extension_round_trip():
    """64-QAM slicer (extension; no reference oracle): noiseless decisions
    are exact and bits round-trip."""
    import fpm_oracle as O
    from paper_2504_09820_b200.detect import slice_count
    rng = np.random.default_rng(9)
    bits = rng.integers(0, 2, (32, 6 * 16), dtype=np.uint8)
    s = O.mod64(bits)
    got, cnt = slice_count(s, bits, qam=64)
    np.testing.assert_array_equal(got, bits)
    assert cnt["bit_errors"] == 0
    noisy = s + 0.03 * (rng.standard_normal(s.shape) + 1j * rng.standard_normal(s.shape))
    got, cnt = slice_count(noisy, bits, qam=64)
    np.testing.assert_array_equal(got, O.demod64(noisy))


def _gpu_batch(T, M, N, seed):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    H = (torch.randn((T, M, N), dtype=torch.complex128, device="cuda", generator=gen)) / np.sqrt(M)
    bits = torch.randint(0, 2, (T, 4 * N), dtype=torch.uint8, device="cuda", generator=gen)
    lv = torch.tensor([-3.0, -1.0, 3.0, 1.0], dtype=torch.float64, device="cuda") / np.sqrt(10.0)
    q = bits.view(T, N, 4).long()
    s = torch.complex(lv[2 * q[..., 0] + q[..., 1]], lv[2 * q[..., 2] + q[..., 3]])
    y = torch.einsum("tmn,tn->tm", H, s)
    return H, y, bits


def test_large_batch_properties():
    """Full-size batches: chunk-size invariance at the c5 shape (2**14
    realizations) and a noiseless zero-error sanity check
    (tests/test_detect.py:114-123 analogue) for CG run to N iterations."""
    from paper_2504_09820_b200.detect import DetectorSpec, detect
    T = 1 << 14
    H, y, bits = _gpu_batch(T, 128, 64, 1)
    det = DetectorSpec("fp_bj_cg", iters=8, L=4, matvec="fp16", inner="fp16")
    res = detect(det, H, y, 0.015811, bits)
    assert res.counters["trials"] == T
    half = detect(det, H[: T // 2], y[: T // 2], 0.015811, bits[: T // 2])
    assert torch.equal(half.x, res.x[: T // 2])
    H, y, bits = _gpu_batch(T, 128, 16, 2)
    res = detect(DetectorSpec("cg", iters=16), H, y, 1e-30, bits)
    assert res.counters["bit_errors"] == 0


def test_persistent_kernel_multi_group_and_partial_group():
    """The warp-specialised persistent kernel loops over several realization
    groups per CTA (148 CTAs) and ends with a partial group: bit-exact vs the
    oracle with injected block inverses, and the fallback kernel agrees."""
    import fpm_oracle as O
    from paper_2504_09820_b200.detect import DetectorSpec, detect
    T = 148 * 2 * 3 + 1
    H, y, bits, s2 = _oracle_inputs(128, 64, 0.5, 15.0, T)
    det = DetectorSpec("fp_bj_cg", iters=8, L=4, matvec="fp16", inner="fp16")
    A, b = O.gram_mf_einsum(H, y, s2)
    mats = O.bj_inverses(A, 4)
    ref = O.cg_batch(A, b, 8, O.FP64, O.FP16, O.FP16, mats)
    res = detect(det, H, y, s2, bits, minv=mats, want_bits=True)
    assert bits_equal(res.x, ref.x)
    ob = O.demod16(ref.x)
    np.testing.assert_array_equal(res.bits, ob)
    assert res.counters["bit_errors"] == int(O.bit_errors(ob, bits).sum())
    assert res.counters["trials"] == T
    assert "fpm_detect_ws_kernel" in _lib_last_kernel()
    o = run_knob_child("tests/test_gpu_parity.py::test_child_multi_group_fallback", {"FPM_NO_WS": "1"})
    assert "fpm_detect_ws_kernel" not in str(o["k"])
    assert bits_equal(o["x"], ref.x)


def _lib_last_kernel():
    from paper_2504_09820_b200 import _lib
    return _lib.load().fpm_last_kernel().decode()


@knob_child
def test_child_multi_group_fallback():
    import fpm_oracle as O
    from paper_2504_09820_b200.detect import DetectorSpec, detect
    T = 148 * 2 * 3 + 1
    H, y, bits, s2 = _oracle_inputs(128, 64, 0.5, 15.0, T)
    det = DetectorSpec("fp_bj_cg", iters=8, L=4, matvec="fp16", inner="fp16")
    A, b = O.gram_mf_einsum(H, y, s2)
    res2 = detect(det, H, y, s2, bits, minv=O.bj_inverses(A, 4))
    save_child_out(x=res2.x, k=np.array(_lib_last_kernel()))


def test_solver_warp_variant_bit_exact():
    """Opt-in variant (FPM_WS_SW=1, measured slower): the CG side
    of the fused kernel as four solver warps, one realization each
    (csrc/fpm_detect_sw.cuh: the run_batch warp kernel's arithmetic on the
    hand-off slot).  Bit-exact vs the oracle with injected inverses at c5 fp16
    (several groups per CTA, a partial last group, breakdown / divergence flags
    and counts included; on-chip inverses within tolerance with identical
    decisions) and at c2 (N = 32, plain fp_cg, fp16 and bf16)."""
    o = run_knob_child("tests/test_gpu_parity.py::test_child_solver_warps", {"FPM_WS_SW": "1"})
    for tag in ("c5_fp16", "c5_bf16", "c2", "c2_bf16"):
        assert "[sw]" in str(o["k_" + tag]), o["k_" + tag]
        assert bits_equal(o["x_" + tag], o["ref_" + tag]), tag
        assert np.array_equal(o["brk_" + tag], o["rbrk_" + tag]), tag
        assert np.array_equal(o["div_" + tag], o["rdiv_" + tag]), tag
        assert np.array_equal(o["bits_" + tag], o["rbits_" + tag]), tag
        assert int(o["be_" + tag]) == int(o["rbe_" + tag]), tag
        if "obits_" + tag in o:
            assert np.array_equal(o["obits_" + tag], o["rbits_" + tag]), tag
            assert float(o["oerr_" + tag]) < 2.0 ** -9, (tag, float(o["oerr_" + tag]))


@knob_child
def test_child_solver_warps():
    import fpm_oracle as O
    from paper_2504_09820_b200.detect import DetectorSpec, detect
    out = {}

    def run(tag, M, N, zeta, snr, T, det, fmt, L):
        H, y, bits, s2 = _oracle_inputs(M, N, zeta, snr, T)
        A, b = O.gram_mf_einsum(H, y, s2)
        mats = O.bj_inverses(A, L) if L else None
        res = detect(det, H, y, s2, bits, minv=mats, want_bits=True)
        ref = O.cg_batch(A, b, det.iters, O.FP64, fmt, fmt, mats)
        rbits = O.demod16(ref.x)
        out["x_" + tag], out["ref_" + tag] = res.x, ref.x
        out["k_" + tag] = np.array(_lib_last_kernel())
        out["brk_" + tag], out["rbrk_" + tag] = res.breakdown_at, ref.breakdown_at
        out["div_" + tag], out["rdiv_" + tag] = res.diverged_at, ref.diverged_at
        out["bits_" + tag], out["rbits_" + tag] = res.bits, rbits
        out["be_" + tag] = np.array(res.counters["bit_errors"])
        out["rbe_" + tag] = np.array(int(O.bit_errors(rbits, bits).sum()))
        if L:  # on-chip block inverses (one lane per block): same decisions, x within tolerance
            r2 = detect(det, H, y, s2, bits, want_bits=True)
            out["obits_" + tag] = r2.bits
            out["oerr_" + tag] = np.array((np.linalg.norm(r2.x - ref.x, axis=1) / np.linalg.norm(ref.x, axis=1)).max())

    T = 148 * 2 * 3 + 1
    run("c5_fp16", 128, 64, 0.5, 15.0, T, DetectorSpec("fp_bj_cg", iters=8, L=4, matvec="fp16", inner="fp16"), O.FP16, 4)
    run("c5_bf16", 128, 64, 0.5, 15.0, 148 * 2 + 1, DetectorSpec("fp_bj_cg", iters=8, L=4, matvec="bfloat16", inner="bfloat16"),
        O.BF16, 4)
    run("c2", 128, 32, 0.5, 10.0, 148 * 8 * 2 + 3, DetectorSpec("fp_cg", iters=10, matvec="fp16", inner="fp16"),
        O.FP16, 0)
    run("c2_bf16", 128, 32, 0.5, 10.0, 148 * 8 + 5, DetectorSpec("fp_cg", iters=10, matvec="bfloat16", inner="bfloat16"),
        O.BF16, 0)
    save_child_out(**out)


def test_tmem_matrix_variant_bit_exact():
    """Opt-in variant (FPM_TMEM_A=1, measured slower): the fp64
    matrix of the hand-off in tensor memory, staged through shared-memory
    rounds and read back by the CG warps' lanes (tcgen05.st / tcgen05.ld).
    Bit-exact vs the oracle with injected inverses at c5 fp64 over several
    groups per CTA and a partial last group, and at N = 16 plain CG (R = 32)."""
    o = run_knob_child("tests/test_gpu_parity.py::test_child_tmem_matrix", {"FPM_TMEM_A": "1"})
    for tag in ("c5", "c1"):
        assert "tmemA" in str(o["k_" + tag]), o["k_" + tag]
        assert bits_equal(o["x_" + tag], o["ref_" + tag]), tag


@knob_child
def test_child_tmem_matrix():
    import fpm_oracle as O
    from paper_2504_09820_b200.detect import DetectorSpec, detect
    out = {}
    T = 148 * 2 * 2 + 1
    H, y, bits, s2 = _oracle_inputs(128, 64, 0.5, 15.0, T)
    A, b = O.gram_mf_einsum(H, y, s2)
    mats = O.bj_inverses(A, 4)
    det = DetectorSpec("fp_bj_cg", iters=8, L=4)
    out["x_c5"] = detect(det, H, y, s2, bits, minv=mats).x
    out["k_c5"] = np.array(_lib_last_kernel())
    out["ref_c5"] = O.cg_batch(A, b, 8, O.FP64, O.FP64, O.FP64, mats).x
    T = 32 * 148 + 5
    H, y, bits, s2 = _oracle_inputs(128, 16, 0.0, 10.0, T)
    A, b = O.gram_mf_einsum(H, y, s2)
    out["x_c1"] = detect(DetectorSpec("cg", iters=8), H, y, s2, bits).x
    out["k_c1"] = np.array(_lib_last_kernel())
    out["ref_c1"] = O.cg_batch(A, b, 8, O.FP64, O.FP64, O.FP64, None).x
    save_child_out(**out)


HIST_EXACT = ("x", "breakdown_at", "diverged_at", "alphas", "betas", "converged_at", "iterates", "residual_vectors")
HIST_NORMS = ("residual_norms", "iterate_norms", "b_norm")


def _check_history(res, want, tag):
    for k in HIST_EXACT:
        got, w = getattr(res, k), want[k]
        assert got is not None, (tag, k)
        assert bits_equal(np.asarray(got, w.dtype), w), (tag, k)
    for k in HIST_NORMS:
        np.testing.assert_allclose(getattr(res, k), want[k], rtol=NORM_RTOL, atol=0, err_msg=f"{tag} {k}")


def test_run_batch_histories_match_reference():
    """Full BatchResult (solvers.py:188-204, 306-393) against the reference's
    own run_batch on the flag systems (breakdown / stall / divergence lanes,
    with record_iterates / record_residual_vectors / record_gaps) and on a
    c5 block-Jacobi batch."""
    from paper_2504_09820_b200.formats import get_format
    from paper_2504_09820_b200.solvers import BatchBlocks, PrecisionConfig, run_batch
    g = load_golden("hist_cg")
    for tag, prec in (("fp16", PrecisionConfig(matvec=get_format("fp16"), inner=get_format("fp16"))),
                      ("fp64", PrecisionConfig())):
        res = run_batch(g["edge_A"], g["edge_b"], 6, prec, x_ref=g["edge_x_ref"], record_gaps=True,
                        record_iterates=True, record_residual_vectors=True, rtol=1e-3)
        want = {k: g[f"edge_{tag}_{k}"] for k in HIST_EXACT + HIST_NORMS + ("residual_gaps",)}
        _check_history(res, want, tag)
        # gaps: a difference of nearly equal fp64 quantities through cuBLAS vs einsum
        np.testing.assert_allclose(res.residual_gaps, want["residual_gaps"], rtol=1e-6, atol=1e-13)
    prec = PrecisionConfig(matvec=get_format("fp16"), inner=get_format("fp16"))
    res = run_batch(g["c5_A"], g["c5_b"], 8, prec, BatchBlocks(g["c5_Minv"], 64, 4), record_iterates=True,
                    record_residual_vectors=True, rtol=1e-2)
    _check_history(res, {k: g[f"c5_{k}"] for k in HIST_EXACT if k not in ("breakdown_at", "diverged_at")}
                   | {k: g[f"c5_{k}"] for k in HIST_NORMS} | {"breakdown_at": np.full(4, -1), "diverged_at":
                                                             np.full(4, -1)}, "c5")


def test_run_batch_histories_all_lanes_frozen_early(oracle):
    """Every lane frozen after sweep 1 (breakdown + stall): the kernel exits
    early and must still record the remaining sweeps as the reference does
    (frozen norms and vectors, zero alphas / betas)."""
    from paper_2504_09820_b200.solvers import PrecisionConfig, run_batch
    O = oracle
    g = load_golden("hist_cg")
    A, b = g["edge_A"][1:3], g["edge_b"][1:3]
    res = run_batch(A, b, 6, PrecisionConfig(), record_iterates=True, record_residual_vectors=True)
    want = O.cg_batch(A, b, 6, record=True)
    _check_history(res, {k: getattr(want, k) for k in HIST_EXACT + HIST_NORMS}, "frozen")


def test_detect_batch_reentrant_from_threads(oracle):
    """The boundary may be called concurrently (experiments.py:257-261 runs
    detectors in a ThreadPoolExecutor): per-call streams and buffers, no
    shared mutable state -> identical results to sequential calls."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2504_09820_b200.detect import DetectorSpec, _detect_batch
    dets = [DetectorSpec("fp_bj_cg", iters=6, L=4, matvec="fp16", inner="fp16"),
            DetectorSpec("fp_cg", iters=5, matvec="bfloat16", inner="bfloat16"), DetectorSpec("cg", iters=4)]
    jobs = []
    for s in range(6):
        H, y, bits, s2 = oracle.simulate(64, 32, 0.5, 10.0, range(s * 24, s * 24 + 24), 11)
        jobs.append((dets[s % 3], {"H": H, "H_est": H, "y": y, "bits": bits, "sigma_n2": s2}))
    seq = [_detect_batch(d, b) for d, b in jobs]
    with ThreadPoolExecutor(4) as ex:
        par = list(ex.map(lambda j: _detect_batch(*j), jobs))
    for (x1, d1), (x2, d2) in zip(seq, par):
        assert bits_equal(x1, x2)
        np.testing.assert_array_equal(d1, d2)


def test_install_patches_reference_style_module():
    """install() swaps `_detect_batch` into a module the way run_ber_sweep
    looks it up (detect.py:259) and uninstall() restores it."""
    import types
    from paper_2504_09820_b200 import detect as D
    mod = types.ModuleType("fake_fpmimo_detect")
    sentinel = object()
    mod._detect_batch = sentinel
    prev = D.install(mod)
    assert prev is sentinel and mod._detect_batch is D._detect_batch
    D.uninstall(mod)
    assert mod._detect_batch is sentinel


def _normwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-300)


def test_lmmse_direct_solve_and_fused_detector():
    """LMMSE comparator (detect.py:230-231, linalg.py:223-231): x within
    1e-12 normwise of LAPACK's Cholesky solve (bits of zpotrf are not
    reproducible); sliced bits and error counts identical."""
    from paper_2504_09820_b200.detect import DetectorSpec, _detect_batch, detect, detect_host
    from paper_2504_09820_b200.solvers import solve_direct_batch
    g = load_golden("lmmse")
    det = DetectorSpec("lmmse")
    for tag in ("c5", "c2"):
        x = solve_direct_batch(g[f"{tag}_A"], g[f"{tag}_b"])
        assert _normwise(x, g[f"{tag}_x"]).max() <= 1e-12
        res = detect(det, g[f"{tag}_H"], g[f"{tag}_y"], float(g[f"{tag}_sigma2"]), g[f"{tag}_tx_bits"], want_bits=True)
        assert _normwise(res.x, g[f"{tag}_x"]).max() <= 1e-12
        np.testing.assert_array_equal(res.bits, g[f"{tag}_rx_bits"])
        assert res.counters["bit_errors"] == int(g[f"{tag}_bit_errors"].sum())
        assert res.counters["trials"] == g[f"{tag}_H"].shape[0]
        assert (res.diverged_at == -1).all() and (res.breakdown_at == -1).all()
        hres = detect_host(det, g[f"{tag}_H"], g[f"{tag}_y"], float(g[f"{tag}_sigma2"]), g[f"{tag}_tx_bits"])
        assert bits_equal(hres.x, res.x) and hres.counters["bit_errors"] == res.counters["bit_errors"]
        xb, bad = _detect_batch(det, {"H_est": g[f"{tag}_H"], "y": g[f"{tag}_y"], "sigma_n2": g[f"{tag}_sigma2"]})
        assert bits_equal(xb, res.x) and not bad.any()


def test_lmmse_non_pd_raises():
    from paper_2504_09820_b200.errors import ContractViolation
    from paper_2504_09820_b200.solvers import solve_direct_batch
    A = np.eye(4, dtype=np.complex128)[None].repeat(2, 0)
    A[1, 2, 2] = -1.0
    with pytest.raises(ContractViolation):
        solve_direct_batch(A, np.ones((2, 4), np.complex128))


SMALL_N = [(16, 8), (24, 8), (32, 16), (64, 32)]


def _small_n_case(O, M, N, tag):
    from paper_2504_09820_b200.detect import DetectorSpec, detect, gram_mf
    T = 40
    H, y, bits, s2 = O.simulate(M, N, 0.5, 4.0, range(T), 11)
    A, b = O.gram_mf(H, y, s2)
    Ag, bg = gram_mf(H, y, s2)
    assert bits_equal(Ag, A) and bits_equal(bg, b)
    for alg, mv in (("cg", O.FP64), ("fp_cg", O.FP16)):
        det = DetectorSpec(alg, iters=4, **({} if alg == "cg" else dict(matvec="fp16", inner="fp16")))
        r = detect(det, H, y, s2, bits)
        _, _, _, out = O.detect(H, y, s2, alg, 4, None, O.FP64, mv, mv)
        assert bits_equal(r.x, out.x), (alg, tag)


@pytest.mark.parametrize("M,N", SMALL_N)
def test_small_n_all_paths_against_oracle(oracle, M, N):
    """Small N (more matched-filter chains than Gram jobs) through the
    persistent kernel, the fallback fused kernel (knob FPM_NO_WS, fresh
    process) and the standalone Gram, plain CG fp64 and FP-CG fp16, against
    the oracle bit for bit."""
    _small_n_case(oracle, M, N, "ws")
    run_knob_child(f"tests/test_gpu_parity.py::test_child_small_n_fallback[{M}-{N}]", {"FPM_NO_WS": "1"})


@knob_child
@pytest.mark.parametrize("M,N", SMALL_N)
def test_child_small_n_fallback(oracle, M, N):
    _small_n_case(oracle, M, N, "fallback")


SHAPES = [  # (M, N, L) -- N multiples of 4 and not, L dividing N; every kernel geometry
    (8, 4, 2), (20, 8, 4), (33, 12, 3), (40, 16, 4), (41, 20, 5), (64, 24, 6), (70, 28, 4), (96, 32, 8),
    (100, 40, 8), (128, 48, 4), (130, 56, 7), (160, 64, 8), (200, 80, 8), (256, 96, 8), (300, 128, 8),
]


@pytest.mark.parametrize("M,N,L", SHAPES)
def test_shape_sweep_fused_detector_bit_exact(oracle, M, N, L):
    """Every (M, N, L) geometry class through the fused detector, plain fp16
    FP-CG and fp16 FP-BJ-CG with injected inverses, against the oracle bit
    for bit; partial realization groups included (T odd)."""
    from paper_2504_09820_b200.detect import DetectorSpec, detect
    O = oracle
    T = 37
    H, y, bits, s2 = O.simulate(M, N, 0.4, 8.0, range(T), 5)
    A, b = O.gram_mf(H, y, s2)
    mats = O.bj_inverses(A, L)
    for alg, mt in (("fp_cg", None), ("fp_bj_cg", mats)):
        det = DetectorSpec(alg, iters=5, L=L if alg == "fp_bj_cg" else None, matvec="fp16", inner="fp16")
        ref = O.cg_batch(A, b, 5, O.FP64, O.FP16, O.FP16, mt)
        res = detect(det, H, y, s2, bits, minv=mt, want_bits=True)
        assert bits_equal(res.x, ref.x), (alg, M, N, L)
        np.testing.assert_array_equal(res.breakdown_at, ref.breakdown_at)
        np.testing.assert_array_equal(res.bits, O.demod16(ref.x))


@pytest.mark.parametrize("M,N,L", SHAPES[::2])
@pytest.mark.parametrize("fmt", ["fp64", "fp32", "bfloat16", "p6e4"])
def test_shape_sweep_formats_gram_and_run_batch(oracle, M, N, L, fmt):
    """Gram (fpm_gram) and run_batch (fpm_cg) across the geometry classes for
    every matvec/inner kind (native fp64 / fp32 / bf16 and a generic
    emulated (6, 4) format), textbook and as-written BJ, bit for bit."""
    from paper_2504_09820_b200.formats import get_format, make_format
    from paper_2504_09820_b200.detect import gram_mf
    from paper_2504_09820_b200.solvers import PrecisionConfig, run_batch
    O = oracle
    T = 21
    H, y, bits, s2 = O.simulate(M, N, 0.4, 8.0, range(T), 9)
    A, b = O.gram_mf(H, y, s2)
    Ag, bg = gram_mf(H, y, s2)
    assert bits_equal(Ag, A) and bits_equal(bg, b)
    f = make_format(6, 4) if fmt == "p6e4" else get_format(fmt)
    of = O.Fmt("p6e4", 6, 4) if fmt == "p6e4" else O.REGISTRY[fmt]
    mats = O.bj_inverses(A, L)
    for rv in ("as_written", "textbook"):
        ref = O.cg_batch(A, b, 4, O.FP64, of, of, mats, rho_update=rv)
        res = run_batch(A, b, 4, PrecisionConfig(matvec=f, inner=f), _pack(mats, N, L), rho_update=rv)
        assert bits_equal(res.x, ref.x), (fmt, rv)
        np.testing.assert_array_equal(res.diverged_at, ref.diverged_at)


def _pack(mats, N, L):
    from paper_2504_09820_b200.solvers import BatchBlocks, pack_blocks
    return BatchBlocks(pack_blocks(mats, N, L), N, L)


def test_composed_path_fp64_matvec_at_n128(oracle):
    """fp64 matvec at N = 128 (c4 shape): A at u_MV does not fit shared
    memory, so the detector composes fpm_gram -> fpm_bj_setup -> fpm_cg with
    A read from global memory; bit-exact with injected inverses, identical
    bits with on-chip ones (tolerance on x)."""
    from paper_2504_09820_b200.detect import DetectorSpec, detect, detect_host
    O = oracle
    M, N, L, T = 256, 128, 8, 6
    H, y, bits, s2 = O.simulate(M, N, 0.5, 20.0, range(T), 3)
    A, b = O.gram_mf(H, y, s2)
    mats = O.bj_inverses(A, L)
    det = DetectorSpec("fp_bj_cg", iters=4, L=L)
    ref = O.cg_batch(A, b, 4, O.FP64, O.FP64, O.FP64, mats)
    r = detect(det, H, y, s2, bits, minv=mats, want_bits=True)
    assert bits_equal(r.x, ref.x)
    np.testing.assert_array_equal(r.bits, O.demod16(ref.x))
    assert r.counters["trials"] == T
    r2 = detect(det, H, y, s2, bits, want_bits=True)
    rel = np.linalg.norm(r2.x - ref.x, axis=1) / np.linalg.norm(ref.x, axis=1)
    assert rel.max() <= 1e-12
    np.testing.assert_array_equal(r2.bits, r.bits)
    r3 = detect_host(det, H, y, s2, bits, minv=mats)
    assert bits_equal(r3.x, ref.x)


@pytest.mark.parametrize("case", ["nan_h", "inf_y", "huge", "sigma0", "m_lt_n", "big_m"])
def test_edge_inputs_against_oracle(oracle, case):
    """Non-finite and extreme inputs, sigma^2 = 0, M < N, large M: the fused
    detector reproduces the reference semantics (NaN propagation, divergence
    and breakdown flags, frozen iterates) bit for bit."""
    from paper_2504_09820_b200.detect import DetectorSpec, detect
    O = oracle
    M, N, T = {"m_lt_n": (6, 8), "big_m": (1000, 16)}.get(case, (24, 8)) + (9,)
    H, y, bits, s2 = O.simulate(M, N, 0.3, 10.0, range(T), 13)
    H = H.copy()
    y = y.copy()
    if case == "nan_h":
        H[2, 3, 1] = complex(np.nan, 0.0)
    elif case == "inf_y":
        y[4, 0] = complex(np.inf, -1.0)
    elif case == "huge":
        H[1] *= 1e5       # fp16 matvec overflow -> divergence
        y[6] *= 1e-30     # tiny right-hand side
    elif case == "sigma0":
        s2 = 0.0
    for alg, mv in (("fp_cg", O.FP16), ("cg", O.FP64)):
        det = DetectorSpec(alg, iters=5, **({} if alg == "cg" else dict(matvec="fp16", inner="fp16")))
        A, b = O.gram_mf(H, y, s2)
        ref = O.cg_batch(A, b, 5, O.FP64, mv, mv)
        r = detect(det, H, y, s2, bits, want_bits=True)
        assert bits_equal(r.x, ref.x), (case, alg)
        np.testing.assert_array_equal(r.breakdown_at, ref.breakdown_at)
        np.testing.assert_array_equal(r.diverged_at, ref.diverged_at)
        np.testing.assert_array_equal(r.bits, O.demod16(ref.x))


@pytest.mark.parametrize("M,N,L,T", [(128, 64, 4, 5), (512, 128, 4, 5), (40, 16, 4, 5), (33, 12, 4, 5),
                                     (512, 128, 8, 300), (200, 128, 8, 151)])
def test_fp32_gram_extension(oracle, M, N, L, T):
    """FP32-Gram extension (BASELINE c4; parity unpinned -- no reference knob):
    the binary32 Gram / matched filter bit-exact against its restatement, and
    the detector on top of it bit-exact with injected inverses.  N = 128 with
    L = 8 runs the fused persistent kernel with binary32 Gram warps (stages
    converted in place by the producer warp; several groups per CTA at T =
    300, antenna rows not a multiple of the stage rows at M = 200); the rest
    the composed path (binary32 Gram kernel, then the standalone stages)."""
    from paper_2504_09820_b200 import _lib
    from paper_2504_09820_b200.detect import DetectorSpec, detect, gram_mf
    O = oracle
    H, y, bits, s2 = O.simulate(M, N, 0.6, 12.0, range(T), 17)
    A, b = O.gram_mf_fp32(H, y, s2)
    Ag, bg = gram_mf(H, y, s2, gram="fp32")
    assert bits_equal(Ag, A) and bits_equal(bg, b)
    mats = O.bj_inverses(A, L)
    det = DetectorSpec("fp_bj_cg", iters=4, L=L, matvec="fp16", inner="fp16", gram="fp32")
    ref = O.cg_batch(A, b, 4, O.FP64, O.FP16, O.FP16, mats)
    r = detect(det, H, y, s2, bits, minv=mats, want_bits=True)
    kname = _lib.load().fpm_last_kernel().decode()
    assert ("gram32" in kname and "ws" in kname) == (N == 128 and L == 8), kname
    assert bits_equal(r.x, ref.x)
    np.testing.assert_array_equal(r.bits, O.demod16(ref.x))
    # on-chip block inverses: the same decisions, x within the fp16 tolerance
    r2 = detect(det, H, y, s2, bits, want_bits=True)
    np.testing.assert_array_equal(r2.bits, O.demod16(ref.x))
    err = np.linalg.norm(r2.x - ref.x, axis=1) / np.linalg.norm(ref.x, axis=1)
    assert err.max() <= 2.0 ** -(10 - 2), err.max()


@pytest.mark.parametrize("scale", [1e-20, 3e-23, 3e19])
def test_fp32_gram_subnormal_and_overflow(oracle, scale):
    """Packed binary32 Gram (FMUL2 / FFMA2) keeps IEEE subnormals and
    overflow: products in the binary32 subnormal range (scale 1e-20, 3e-23)
    and sums past FLT_MAX (3e19: inf entries) match the NumPy float32 restatement bit for
    bit."""
    from paper_2504_09820_b200.detect import gram_mf
    O = oracle
    H, y, _, s2 = O.simulate(64, 32, 0.5, 10.0, range(3), 23)
    H, y = H * scale, y * scale
    with np.errstate(over="ignore", invalid="ignore"):
        A, b = O.gram_mf_fp32(H, y, s2)
    Ag, bg = gram_mf(H, y, s2, gram="fp32")
    assert bits_equal(Ag, A) and bits_equal(bg, b)


@pytest.mark.gpu
def test_empty_batches_match_reference_shapes():
    """T = 0 through every boundary call returns the reference's empty
    shapes (run_batch / build_blocks_batch / _solve_direct_batch accept an
    empty batch, solvers.py:262-393, linalg.py:223-231) and launches nothing
    that faults."""
    from paper_2504_09820_b200.detect import DetectorSpec, detect, gram_mf
    from paper_2504_09820_b200.solvers import PrecisionConfig, build_blocks_batch, run_batch, solve_direct_batch
    A = np.zeros((0, 8, 8), np.complex128)
    b = np.zeros((0, 8), np.complex128)
    r = run_batch(A, b, 3)
    assert r.x.shape == (0, 8) and r.diverged_at.shape == (0,) and r.breakdown_at.shape == (0,)
    assert r.residual_norms.shape == (4, 0) and r.iterate_norms.shape == (4, 0) and r.alphas.shape == (3, 0)
    assert r.converged_at.shape == (0,)
    bl = build_blocks_batch(A, 4)
    assert [m.shape for m in bl.mats] == [(0, 4, 4), (0, 4, 4)]
    r = run_batch(A, b, 3, PrecisionConfig.uniform("fp16"), blocks=bl, x_ref=b, record_gaps=True, record_iterates=True)
    assert r.x.shape == (0, 8) and r.residual_gaps.shape == (4, 0) and r.iterates.shape == (4, 0, 8)
    assert solve_direct_batch(A, b).shape == (0, 8)
    H = np.zeros((0, 16, 8), np.complex128)
    y = np.zeros((0, 16), np.complex128)
    Ag, bg = gram_mf(H, y, 0.1)
    assert Ag.shape == (0, 8, 8) and bg.shape == (0, 8)
    for alg in ("fp_bj_cg", "lmmse"):
        det = DetectorSpec(alg, iters=4, L=4, matvec="fp16", inner="fp16") if alg != "lmmse" else DetectorSpec(alg)
        res = detect(det, H, y, 0.1, np.zeros((0, 32), np.uint8), want_bits=True)
        assert res.x.shape == (0, 8) and res.bits.shape == (0, 32)
        assert int(res.counters["trials"]) == 0 and int(res.counters["bit_errors"]) == 0
    from paper_2504_09820_b200 import channel
    b0 = channel.simulate_batch(16, 8, 0.5, 0.5, 10.0, 0, 0, 7)
    assert b0["H"].shape == (0, 16, 8) and b0["bits"].shape == (0, 32) and b0["y"].shape == (0, 16)
