"""Input generation (paper_2504_09820_b200/channel.py + csrc/fpm_gen.cu):
the keyed Philox generator pinned by known answers and by the oracle's
restatement, modulation / correlation helpers against the oracle, and on
the GPU the distribution-level parity with the reference's link model
(detect.py:189-214, channel.py:101-161, 206-219)."""

import math

import numpy as np
import pytest

import fpm_oracle as O
from conftest import bits_equal

torch = pytest.importorskip("torch")
from paper_2504_09820_b200 import channel as C  # noqa: E402


def test_philox4x32_10_known_answers():
    # Random123 kat_vectors for philox4x32_10 (the published algorithm)
    kat = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, want in kat:
        got = O.philox4x32_10(np.array([ctr], np.uint64), key)[0]
        assert tuple(int(v) for v in got) == want


@pytest.mark.parametrize("qam", [16, 64])
def test_modulate_matches_oracle(qam):
    rng = np.random.default_rng(3)
    bps = 4 if qam == 16 else 6
    bits = rng.integers(0, 2, size=(5, bps * 12), dtype=np.uint8)
    got = C.modulate(torch.from_numpy(bits), qam).numpy()
    want = O.mod16(bits) if qam == 16 else O.mod64(bits)
    assert bits_equal(got, want)
    # slicing the noiseless symbols returns the bits
    back = O.demod16(got) if qam == 16 else O.demod64(got)
    np.testing.assert_array_equal(back, bits)


def test_correlation_helpers():
    R = C.exp_correlation_matrix(16, 0.7)
    np.testing.assert_allclose(R, O.exp_corr(16, 0.7))
    S = C.matrix_sqrt_psd(R)
    np.testing.assert_allclose(S @ S, R, atol=1e-13)
    np.testing.assert_allclose(S, O._psd_sqrt(O.exp_corr(16, 0.7)), atol=1e-13)
    Ru = C.user_correlation_matrix(8, 0.5, N_UE=2, block_diag_users=True)
    assert Ru[0, 1] == 0.5 and Ru[1, 2] == 0 and Ru[2, 3] == 0.5
    assert C.noise_variance(128, 64, 15.0) == O.noise_variance(128, 64, 15.0)
    with pytest.raises(Exception):
        C.exp_correlation_matrix(4, 1.0)
    with pytest.raises(Exception):
        C.noise_variance(4, 4, 0.0, "nope")


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.gpu
def test_gen_bits_exact_and_chunk_invariant():
    _cuda()
    W, bits, g, _ = C.gen_trials(20261020, 3, 100, 24, 16, 8)
    np.testing.assert_array_equal(bits.cpu().numpy(), O.gen_bits(20261020, 2, 3, 100, 24, 32))
    W1, b1, g1, _ = C.gen_trials(20261020, 3, 100, 10, 16, 8)
    W2, b2, g2, _ = C.gen_trials(20261020, 3, 110, 14, 16, 8)
    assert torch.equal(torch.cat([W1, W2]), W) and torch.equal(torch.cat([b1, b2]), bits)
    assert torch.equal(torch.cat([g1, g2]), g)
    W3, _, _, _ = C.gen_trials(20261020, 4, 100, 24, 16, 8)  # another SNR point: other streams
    assert not torch.equal(W3, W)


@pytest.mark.gpu
def test_generated_distributions():
    _cuda()
    M, N, T = 32, 8, 4096
    W, bits, g, Cn = C.gen_trials(7, 0, 0, T, M, N, csi=True)
    w = W.flatten()
    assert abs(w.real.mean().item()) < 5e-3 and abs(w.imag.mean().item()) < 5e-3
    assert abs((w.abs() ** 2).mean().item() * M - 1.0) < 0.01          # CN(0, 1/M)
    assert abs(w.real.var().item() * 2 * M - 1.0) < 0.01
    assert abs(bits.float().mean().item() - 0.5) < 0.01
    for z in (g.flatten(), Cn.flatten()):            # re, im ~ N(0, 1) (rng.py:33-39 pairs)
        assert abs((z.abs() ** 2).mean().item() - 2.0) < 0.02
        k = (z.real ** 4).mean().item() / (z.real ** 2).mean().item() ** 2
        assert abs(k - 3.0) < 0.1                                        # Gaussian kurtosis


@pytest.mark.gpu
def test_simulate_batch_channel_and_noise_statistics():
    """E[H^H H] = R_t (tr R_r = M, W ~ CN(0,1/M)); y - H s has variance
    sigma^2 per antenna (detect.py:87-93, 210-211)."""
    _cuda()
    M, N, T, snr = 32, 8, 8192, 6.0
    b = C.simulate_batch(M, N, 0.6, 0.5, snr, 0, T, 11, epsilon_db=10.0)
    G = torch.einsum("tmi,tmj->ij", b["H"].conj(), b["H"]) / T
    Rt = torch.as_tensor(C.exp_correlation_matrix(N, 0.5), device=G.device)
    assert (G - Rt).abs().max().item() < 0.05
    n = b["y"] - torch.einsum("tmn,tn->tm", b["H"], b["symbols"])
    s2 = C.noise_variance(M, N, snr)
    assert abs((n.abs() ** 2).mean().item() / s2 - 1.0) < 0.02
    e = b["H_est"] - b["H"]
    assert abs((e.abs() ** 2).mean().item() * M * 10.0 - 1.0) < 0.02    # CN(0, (1/M)/eps), eps = 10 dB


@pytest.mark.gpu
def test_simulated_ber_matches_oracle_generator_statistically():
    """BER of the fused detector on GPU-generated inputs agrees with the BER
    on the reference generator's inputs (oracle restatement) within the
    Monte-Carlo spread."""
    _cuda()
    from paper_2504_09820_b200.detect import DetectorSpec, detect
    M, N, zeta, snr, T = 64, 16, 0.5, 4.0, 4096
    det = DetectorSpec("fp_bj_cg", iters=6, L=4, matvec="fp16", inner="fp16")
    b = C.simulate_batch(M, N, zeta, zeta, snr, 0, T, 20261020)
    r = detect(det, b["H_est"], b["y"], b["sigma_n2"], b["bits"])
    ber_gpu = r.counters["bit_errors"] / (T * 4 * N)
    H, y, bits, s2 = O.simulate(M, N, zeta, snr, range(1024), 20261020)
    r2 = detect(det, H, y, s2, bits)
    ber_ref = r2.counters["bit_errors"] / (1024 * 4 * N)
    sd = math.sqrt(ber_ref * (1 - ber_ref) / (1024 * 4 * N)) + math.sqrt(ber_gpu * (1 - ber_gpu) / (T * 4 * N))
    assert abs(ber_gpu - ber_ref) < 5 * sd + 1e-3, (ber_gpu, ber_ref)


def _ar_factor(n, zeta, n_ue=None):
    """Lower factor of the AR(1) recursion x_0 = w_0, x_k = zeta x_{k-1} +
    sqrt(1 - zeta^2) w_k (restarting every n_ue entries when given)."""
    F = np.zeros((n, n))
    for k in range(n):
        start = k == 0 or (n_ue and k % n_ue == 0)
        if start:
            F[k, k] = 1.0
        else:
            F[k] = zeta * F[k - 1]
            F[k, k] = math.sqrt(1 - zeta * zeta)
    return F


@pytest.mark.parametrize("zeta,n_ue", [(0.0, None), (0.5, None), (0.8, None), (0.7, 4)])
def test_ar1_recursion_is_the_cholesky_factor_of_exponential_correlation(zeta, n_ue):
    """fpm_simulate colours with the AR(1) recursion: it IS the lower
    Cholesky factor of [R]_ij = zeta^|i-j| (block-diagonal per user block),
    so F W F^T has the reference's Kronecker distribution."""
    n = 16
    R = C.user_correlation_matrix(n, zeta, n_ue or 1, block_diag_users=bool(n_ue)).real
    F = _ar_factor(n, zeta, n_ue)
    np.testing.assert_allclose(F @ F.T, R, atol=1e-14)
    np.testing.assert_allclose(F, np.linalg.cholesky(R), atol=1e-14)


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,zr,zt,qam,bd", [(16, 8, 0.0, 0.0, 16, 0), (32, 64, 0.6, 0.5, 16, 0),
                                              (24, 128, 0.8, 0.8, 64, 0), (16, 48, 0.3, 0.7, 16, 4),
                                              (8, 20, 0.5, 0.5, 64, 0)])
def test_fused_simulate_against_draws(M, N, zr, zt, qam, bd):
    """fpm_simulate == the AR(1) colouring of fpm_gen_trials' draws, QAM of
    its bits, y = H s + sqrt(sigma^2/2) g (bit-exact draws / bits, 1e-13 on
    the coloured values: the kernel uses FMAs and a different sum order)."""
    _cuda()
    T, snr, seed = 37, 7.0, 99
    bps = 4 if qam == 16 else 6
    b = C.simulate_batch(M, N, zr, zt, snr, 5, T, seed, point=2, qam=qam, N_UE=bd or 1, block_diag_users=bool(bd),
                         epsilon_db=12.0)
    W, bits, g, Cn = C.gen_trials(seed, 2, 5, T, M, N, qam=qam, csi=True)
    assert torch.equal(b["bits"], bits)
    W, g, Cn = W.cpu().numpy(), g.cpu().numpy(), Cn.cpu().numpy()
    Fr, Ft = _ar_factor(M, zr), _ar_factor(N, zt, bd or None)
    H = np.einsum("ij,tjn,kn->tik", Fr, W, Ft)
    Hg = b["H"].cpu().numpy()
    if zr == 0 and zt == 0:
        assert bits_equal(Hg, W)
    np.testing.assert_allclose(Hg, H, rtol=0, atol=1e-13)
    s = b["symbols"].cpu().numpy()
    want_s = O.mod16(bits.cpu().numpy()) if qam == 16 else O.mod64(bits.cpu().numpy())
    assert bits_equal(s, want_s)
    s2 = C.noise_variance(M, N, snr)
    y = np.einsum("tmn,tn->tm", Hg, s) + math.sqrt(s2 / 2) * g
    np.testing.assert_allclose(b["y"].cpu().numpy(), y, rtol=0, atol=1e-13)
    var = (1.0 / M) / 10.0 ** 1.2
    np.testing.assert_allclose(b["H_est"].cpu().numpy(), Hg + math.sqrt(var / 2) * Cn, rtol=0, atol=1e-14)
