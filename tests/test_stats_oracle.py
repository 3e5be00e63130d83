"""Pins of the statistics oracle (NEXT-3): correlation / noise-variance estimators and the closed-form
robustness sweep of PAPER.md Fig. fig7 c/d -- CPU only."""
import dataclasses

import numpy as np
import pytest

import oracle
import workload
from workload import CONFIGS


def test_correlation_estimate_brute_force():
    rng = np.random.default_rng(0)
    H = rng.standard_normal((3, 9)) + 1j * rng.standard_normal((3, 9))
    R = oracle.correlation_estimate(H, 4)
    for d in range(4):
        acc = 0
        for c in range(3):
            for n in range(9 - d):
                acc += H[c, n + d] * np.conj(H[c, n])
        assert abs(R[d] - acc / (3 * (9 - d))) < 1e-12


def test_noise_estimator_normalisation_parseval():
    """With the window = all N bins the delay-domain power equals the tone-domain power (Parseval):
    pins the unitary sqrt(N) scaling of the IDFT."""
    rng = np.random.default_rng(1)
    H = rng.standard_normal((5, 64)) + 1j * rng.standard_normal((5, 64))
    assert abs(oracle.noise_variance_estimate(H, 64) - np.mean(np.abs(H) ** 2)) < 1e-12
    assert list(oracle.noise_bins(64, 8)) == list(range(28, 36))


def test_noise_estimate_on_white_noise_is_unbiased():
    rng = np.random.default_rng(2)
    s2 = 0.37
    W = np.sqrt(s2 / 2) * (rng.standard_normal((4000, 256)) + 1j * rng.standard_normal((4000, 256)))
    est = oracle.noise_variance_estimate(W, 32)
    se = s2 / np.sqrt(4000 * 32)                      # |CN|^2 is exponential: sd = mean
    assert abs(est - s2) < 5 * se


@pytest.mark.parametrize("cfg_id", [3, 5])
def test_stats_recovered_from_synthetic_pilots(cfg_id):
    """r_hat, sigma2_hat from one instance of the config's pilots vs the generator's true statistics."""
    cfg = dataclasses.replace(CONFIGS[cfg_id], slots=1, M=64 if cfg_id == 3 else 16)
    r, s2 = workload.channel_stats(cfg, 0)
    x = workload.gen_pilots(cfg, 0)
    y = workload.gen_instances(cfg, 0, x=x)
    r_hat, s2_hat = oracle.estimate_stats(y, x, D=cfg.b, B=cfg.N // 8)
    assert abs(s2_hat / s2[0] - 1) < 0.05, (s2_hat, s2[0])
    # r_hat[d]: sample correlation over C*(N-d) correlated terms; the channel part fluctuates with the
    # C independent channel draws (relative spread ~ 1/sqrt(C))
    C = cfg.M * cfg.K
    assert np.max(np.abs(r_hat - r[0, :cfg.b])) < 6 / np.sqrt(C), np.max(np.abs(r_hat - r[0, :cfg.b]))


def test_mismatched_mse_closed_form_and_optimality():
    """Matched design = the LMMSE closed form (oracle.block_mse); any other design is worse (optimality)."""
    cfg = CONFIGS[3]
    r, s2 = workload.channel_stats(cfg, 0)
    b = 24
    m = oracle.mismatched_block_mse(r[0], s2[0], r[0], s2[0], b)
    assert abs(m - oracle.block_mse(r[0], s2[0], b)) < 1e-14
    d = np.arange(cfg.N)
    for L in (2.0, 30.0, 300.0):
        for s2d in (1e-4, s2[0], 1.0):
            assert oracle.mismatched_block_mse(r[0], s2[0], oracle.rd_uniform(L, cfg.Nfft, d), s2d, b) >= m - 1e-15


def test_mismatched_mse_monte_carlo():
    """Closed form vs the oracle estimator run with a mismatched design on synthetic data (5 SE)."""
    cfg = dataclasses.replace(CONFIGS[1], M=200, slots=1)
    r, s2 = workload.channel_stats(cfg, 0)
    rd = oracle.rd_uniform(2.0, cfg.Nfft, np.arange(cfg.N))
    x = workload.gen_pilots(cfg, 0)
    y, H = workload.gen_instances(cfg, 0, x=x, return_channel=True)
    h = oracle.block_lmmse(y, x, rd[None], np.array([0.3]), None, cfg.b, cfg.stride)
    e = (np.abs(h - H) ** 2).reshape(-1, cfg.N).mean(axis=1)     # per column (independent draws)
    cf = oracle.mismatched_block_mse(r[0], s2[0], rd, 0.3, cfg.b)
    assert abs(e.mean() - cf) < 5 * e.std() / np.sqrt(e.size)


def test_robustness_sweep_fig7cd():
    """PAPER.md:556-558 (Fig. fig7 c/d): with the channel drawn from the uniform-delay model itself the
    sweep over the assumed L is minimised exactly at the true L and over SNR_fixed at the true SNR
    (LMMSE optimality); qualitatively (7 discrete taps, true SNR 25 dB), MSE rises steeply when L or
    SNR_fixed are set too low and only mildly when set too high."""
    N, Nfft, b = 1200, 2048, 100
    d = np.arange(N)
    s2 = 10 ** (-2.5)
    r_uni = oracle.rd_uniform(7.0, Nfft, d)
    msL = [oracle.mismatched_block_mse(r_uni, s2, oracle.rd_uniform(L, Nfft, d), s2, b) for L in range(1, 16)]
    assert int(np.argmin(msL)) + 1 == 7
    msS = [oracle.mismatched_block_mse(r_uni, s2, r_uni, 10 ** (-snr / 10), b) for snr in range(0, 41, 5)]
    assert int(np.argmin(msS)) * 5 == 25
    r7 = np.exp(-2j * np.pi * np.outer(d, np.arange(7)) / Nfft).mean(axis=1)     # 7 equal discrete taps
    msL = [oracle.mismatched_block_mse(r7, s2, oracle.rd_uniform(L, Nfft, d), 1e-4, b) for L in range(1, 16)]
    assert msL[0] > 5 * min(msL) and msL[-1] < 2 * min(msL)
    msS = [oracle.mismatched_block_mse(r7, s2, oracle.rd_uniform(7.0, Nfft, d), 10 ** (-snr / 10), b)
           for snr in (0, 25, 40)]
    assert msS[0] > 5 * msS[1] and msS[2] < 1.5 * msS[1]
