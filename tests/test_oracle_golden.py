"""Pin the CPU oracle against golden vectors produced by the reference.

CPU only.  If the oracle reproduces the reference's own outputs bit for bit
here, it can stand in for the reference on the GPU box (where
/root/reference does not exist).
"""

import numpy as np
import pytest

from conftest import bits_equal, golden_cases, load_golden


def _fmt(O, row):
    sig, exp, sub = (int(v) for v in row)
    for f in O.REGISTRY.values():
        if (f.sig, f.exp, f.subnormals) == (sig, exp, bool(sub)):
            return f
    return O.Fmt(f"p{sig}e{exp}", sig, exp, bool(sub))


def _mats_from_flat(flat, N, L):
    T = flat.shape[0]
    mats, off = [], 0
    for s in range(0, N, L):
        Lk = min(L, N - s)
        mats.append(flat[:, off:off + Lk * Lk].reshape(T, Lk, Lk))
        off += Lk * Lk
    return mats


@pytest.mark.parametrize("name", golden_cases())
def test_gram_matched_filter_bit_exact(oracle, name):
    g = load_golden(name)
    A, b = oracle.gram_mf(g["H"], g["y"], float(g["sigma2"]))
    assert bits_equal(A, g["A"])
    assert bits_equal(b, g["b"])


@pytest.mark.parametrize("name", golden_cases())
def test_cg_bit_exact_with_reference_blocks(oracle, name):
    g = load_golden(name)
    w, mv, ip = (_fmt(oracle, r) for r in g["fmts"])
    N = g["b"].shape[1]
    mats = _mats_from_flat(g["Minv"], N, int(g["L"])) if "Minv" in g else None
    out = oracle.cg_batch(g["A"], g["b"], int(g["iters"]), w, mv, ip, mats, str(g["rho_update"]))
    assert bits_equal(out.x, g["x"])
    np.testing.assert_array_equal(out.breakdown_at, g["breakdown_at"])
    np.testing.assert_array_equal(out.diverged_at, g["diverged_at"])
    np.testing.assert_array_equal(out.converged_at, g["converged_at"])
    assert bits_equal(out.residual_norms, g["residual_norms"])


@pytest.mark.parametrize("name", golden_cases())
def test_bj_inverses_and_slicer(oracle, name):
    g = load_golden(name)
    if "Minv" in g:
        mats = oracle.bj_inverses(g["A"], int(g["L"]))
        flat = np.concatenate([m.reshape(m.shape[0], -1) for m in mats], axis=1)
        # same LAPACK on the same host -> same bits; tolerance if BLAS differs
        np.testing.assert_allclose(flat, g["Minv"], rtol=1e-12, atol=1e-15)
    bits = oracle.demod16(g["x"])
    np.testing.assert_array_equal(bits, g["rx_bits"])
    np.testing.assert_array_equal(oracle.bit_errors(bits, g["tx_bits"]), g["bit_errors"])


def test_solver_edge_flags(oracle):
    g = load_golden("solver_edges")
    for tag in ("fp16", "p5e4", "fp64"):
        w, mv, ip = (_fmt(oracle, r) for r in g[f"{tag}_fmts"])
        out = oracle.cg_batch(g["A"], g["b"], 6, w, mv, ip)
        assert bits_equal(out.x, g[f"{tag}_x"]), tag
        np.testing.assert_array_equal(out.breakdown_at, g[f"{tag}_breakdown_at"])
        np.testing.assert_array_equal(out.diverged_at, g[f"{tag}_diverged_at"])
    mats = _mats_from_flat(g["ragged_Minv"], 8, 3)
    for rv in ("as_written", "textbook"):
        out = oracle.cg_batch(g["ragged_A"], g["ragged_b"], 5, oracle.FP64, oracle.FP16,
                              oracle.FP16, mats, rv)
        assert bits_equal(out.x, g[f"ragged_{rv}_x"]), rv


def test_kernel_kats(oracle):
    g = load_golden("kernel_kats")
    names = {"fp64": oracle.FP64, "fp32": oracle.FP32, "fp16": oracle.FP16, "bfloat16": oracle.BF16}
    for n, f in names.items():
        assert bits_equal(oracle.matvec(g["A"], g["v"], f), g[f"matvec_{n}"]), n
        assert bits_equal(oracle.dot(g["A"][:, 0, :], g["v"], f), g[f"dot_{n}"]), n
        assert bits_equal(oracle.axpy(g["a"], g["A"][:, 1, :], g["v"], f), g[f"axpy_{n}"]), n


def test_slicer_known_answers(oracle):
    g = load_golden("slicer")
    np.testing.assert_array_equal(oracle.demod16(g["x"]), g["bits"])


def test_division_is_numpy_smith(oracle):
    rng = np.random.default_rng(3)
    n = rng.standard_normal((4, 50000)) * np.exp(rng.uniform(-40, 40, (4, 50000)))
    num = n[0] + 1j * n[1]
    den = n[2] + 1j * n[3]
    den[:5] = [0, -0.0, complex(0, -0.0), complex(np.inf, 0), complex(np.nan, 1)]
    with np.errstate(all="ignore"):
        assert bits_equal(oracle.cdiv(num, den), num / den)


def test_qam64_round_trip_extension(oracle):
    # 64-QAM is not in the reference (parity unpinned); check self-consistency.
    rng = np.random.default_rng(4)
    bits = rng.integers(0, 2, (16, 6 * 8), dtype=np.uint8)
    s = oracle.mod64(bits)
    np.testing.assert_array_equal(oracle.demod64(s), bits)
    assert np.mean(np.abs(s) ** 2) == pytest.approx(1.0, rel=0.1)


def test_fast_paths_equal_restatement(oracle):
    rng = np.random.default_rng(11)
    x = rng.standard_normal(100000) * np.exp(rng.uniform(-40, 40, 100000))
    x = np.concatenate([x, [0.0, -0.0, np.inf, -np.inf, np.nan, 65504, 65520, 2**-24, 2**-25, 3 * 2**-26]])
    for f in (oracle.FP16, oracle.FP32):
        assert bits_equal(oracle.fmt_round(x, f), oracle.fmt_round_bits(x, f)), f.name
    H = (rng.standard_normal((3, 40, 12)) + 1j * rng.standard_normal((3, 40, 12))) / 9
    y = rng.standard_normal((3, 40)) + 1j * rng.standard_normal((3, 40))
    a1, b1 = oracle.gram_mf(H, y, 0.03)
    a2, b2 = oracle.gram_mf_einsum(H, y, 0.03)
    assert bits_equal(a1, a2) and bits_equal(b1, b2)


HIST_KEYS = ("x", "residual_norms", "iterate_norms", "alphas", "betas", "b_norm", "converged_at",
             "iterates", "residual_vectors")


def test_cg_histories_bit_exact(oracle):
    """The oracle's BatchResult histories (solvers.py:306-393) equal the
    reference's on the flag systems (breakdown / stall / divergence lanes)
    and on a c5 block-Jacobi batch, including the record_* outputs."""
    O = oracle
    g = load_golden("hist_cg")
    for tag, (mv, ip) in (("fp16", (O.FP16, O.FP16)), ("fp64", (O.FP64, O.FP64))):
        out = O.cg_batch(g["edge_A"], g["edge_b"], 6, O.FP64, mv, ip, None, rtol=1e-3, x_ref=g["edge_x_ref"],
                         record=True)
        for k in HIST_KEYS + ("breakdown_at", "diverged_at", "residual_gaps"):
            got, want = getattr(out, k), g[f"edge_{tag}_{k}"]
            assert bits_equal(np.asarray(got, want.dtype), want), (tag, k)
    mats = O.unpack_blocks(g["c5_Minv"], 64, 4) if hasattr(O, "unpack_blocks") else \
        [g["c5_Minv"][:, k * 16:(k + 1) * 16].reshape(-1, 4, 4) for k in range(16)]
    out = O.cg_batch(g["c5_A"], g["c5_b"], 8, O.FP64, O.FP16, O.FP16, mats, rtol=1e-2, record=True)
    for k in HIST_KEYS:
        got, want = getattr(out, k), g[f"c5_{k}"]
        assert bits_equal(np.asarray(got, want.dtype), want), k


def test_lmmse_restatement_matches_reference(oracle):
    """linalg.py:223-231 restated (scipy cho_factor / cho_solve) equals the
    reference's _solve_direct_batch bit for bit on the fixture systems."""
    g = load_golden("lmmse")
    for tag in ("c5", "c2"):
        assert bits_equal(oracle.lmmse(g[f"{tag}_A"], g[f"{tag}_b"]), g[f"{tag}_x"])
        np.testing.assert_array_equal(oracle.demod16(g[f"{tag}_x"]), g[f"{tag}_rx_bits"])


def test_fp32_gram_extension_is_a_binary32_gram(oracle):
    """EXTENSION (parity unpinned): the binary32 Gram restatement agrees with
    the reference Gram to binary32 accuracy and its values lie on the binary32
    grid."""
    g = load_golden("c5_bj4_fp16")
    A32, b32 = oracle.gram_mf_fp32(g["H"], g["y"], float(g["sigma2"]))
    A, b = g["A"], g["b"]
    assert np.abs(A32 - A).max() <= 2e-6 * np.abs(A).max()
    assert np.abs(b32 - b).max() <= 2e-6 * np.abs(b).max()
    for v in (A32.real, A32.imag, b32.real, b32.imag):
        assert np.array_equal(v, v.astype(np.float32).astype(np.float64))
