"""Seeded inputs for the comb-pilot estimators (NEXT-1); no estimator arithmetic.

    y[t,m,k] = H_{t,m,u}(k) x[t,k] + w,  u = k mod S (UE u owns tones u, u+S, ...; Eq. 6)
    H_{t,m,u}(k) = sum_l h_l exp(-j 2 pi k tau_l / Nfft),  h_l ~ CN(0, p_l) i.i.d. over (t, m, u, l)
    x = (+-1 +- j)/sqrt(2),  w ~ CN(0, sigma_t^2),  sigma_t^2 = 10^(-SNR/10) * sum p_l

Statistics handed to the estimator: the paper's fixed design r_d (Eq. eqrd with L_assumed, normalised
by Nfft -- reading A5) and sigma^2 = 10^(-SNR_fixed/10) (Table III).
Seeds: PCG64 from SeedSequence([seed, 100, stream, t, m]) (stream 1 pilots, 2 taps, 3 noise).
"""
from __future__ import annotations

import numpy as np

from .configs import CombConfig, get_comb_config


def _rng(seed, stream, t, m=0):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 100, stream, t, m])))


def comb_stats(cfg):
    """(r [N] complex128, sigma2 float): fixed-design statistics of the estimator."""
    cfg = get_comb_config(cfg)
    d = np.arange(cfg.N, dtype=np.float64)
    r = np.ones(cfg.N, np.complex128)
    z = 2j * np.pi * cfg.L_assumed * d[1:] / cfg.Nfft
    r[1:] = (1.0 - np.exp(-z)) / z
    return r, 10.0 ** (-cfg.snr_fixed_db / 10.0)


def comb_true_stats(cfg):
    """True first column of R_hh of the synthetic channel (for MSE checks)."""
    cfg = get_comb_config(cfg)
    p = 10.0 ** (np.asarray(cfg.tap_db) / 10.0)
    d = np.arange(cfg.N, dtype=np.float64)
    tau = np.asarray(cfg.tap_delays, np.float64)
    r = (p[None, :] * np.exp(-2j * np.pi * np.outer(d, tau) / cfg.Nfft)).sum(axis=1)
    return r, 10.0 ** (-cfg.snr_db / 10.0) * p.sum()


def comb_pilots(cfg, seed=0):
    cfg = get_comb_config(cfg)
    out = np.empty((cfg.T, cfg.N), np.complex64)
    a = np.float32(1.0 / np.sqrt(2.0))
    for t in range(cfg.T):
        bits = _rng(seed, 1, t).integers(0, 2, size=(2, cfg.N))
        out[t].real = a * (1 - 2 * bits[0])
        out[t].imag = a * (1 - 2 * bits[1])
    return out


def comb_instances(cfg, seed=0, x=None, m_lo=0, m_hi=None, return_channel=False):
    """y complex64 [T][m_hi-m_lo][N]; with return_channel also H complex128 [T][M'][S][N]."""
    cfg = get_comb_config(cfg)
    m_hi = cfg.M if m_hi is None else m_hi
    if x is None:
        x = comb_pilots(cfg, seed)
    p = 10.0 ** (np.asarray(cfg.tap_db) / 10.0)
    tau = np.asarray(cfg.tap_delays, np.float64)
    k = np.arange(cfg.N, dtype=np.float64)
    E = np.exp(-2j * np.pi * np.outer(tau, k) / cfg.Nfft)               # [L][N]
    sigma2 = 10.0 ** (-cfg.snr_db / 10.0) * p.sum()
    owner = np.arange(cfg.N) % cfg.S
    nm = m_hi - m_lo
    y = np.empty((cfg.T, nm, cfg.N), np.complex64)
    H_all = np.empty((cfg.T, nm, cfg.S, cfg.N), np.complex128) if return_channel else None
    for t in range(cfg.T):
        for j, m in enumerate(range(m_lo, m_hi)):
            g = _rng(seed, 2, t, m)
            h = (g.standard_normal((cfg.S, len(p))) + 1j * g.standard_normal((cfg.S, len(p)))) * np.sqrt(p / 2)
            H = h @ E                                                       # [S][N]
            Hk = H[owner, np.arange(cfg.N)]
            w = _rng(seed, 3, t, m).standard_normal((2, cfg.N))
            y[t, j] = (Hk * x[t] + np.sqrt(sigma2 / 2) * (w[0] + 1j * w[1])).astype(np.complex64)
            if return_channel:
                H_all[t, j] = H
    return (y, H_all) if return_channel else y
