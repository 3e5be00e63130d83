"""Seeded input draws for the pilot channel estimator (no estimator arithmetic here).

Signal model (Eq. 1-5, restated per tone in SURVEY.md §8(d)):

    y[t,m,k,n] = H[t,m,k,n] * x[t,k,n] + w[t,m,k,n]
    H[t,m,k,n] = sum_l h_l exp(-j 2 pi n tau_l / Nfft),  h_l ~ CN(0, p_l)  i.i.d. over (slot, m, k, l)
    x[t,k,n]   = (+-1 +- j)/sqrt(2)  (unit-modulus QPSK pilot)
    w          ~ CN(0, sigma2_t),     sigma2_t = 10^(-SNR_t/10)   (sum p_l = 1, sigma_s^2 = 1)

The statistics handed to the estimator are the *true* ones (reading A4, matched
per-slot statistics):  r[d] = E{H(n+d) H*(n)} = sum_l p_l exp(-j 2 pi d tau_l / Nfft),
d = 0..N-1 (the first column of the Hermitian Toeplitz R_hh).

PDP (reading A6): L taps, p_l proportional to 10^(-0.3 l) (3 dB/tap), normalised to
sum 1; delays tau_l = l * Delta samples at the Nfft rate, Delta = 1 (configs 1-2) or
Delta = tau_rms * f_s / rho_L (rms-specified configs), rho_L = rms spread of the
profile in tap units.

Seeding (reading A12): numpy PCG64 from SeedSequence([seed, cfg_id, stream, i, j]):
stream 0 = per-slot statistics (slot), 1 = pilots (t), 2 = taps (slot, m),
3 = noise (t, m).  Every (t, m) slice is generator-independent, so antenna shards
and sampled parity checks draw exactly the same numbers as a full draw.
"""
from __future__ import annotations

import numpy as np

from .configs import Config, get_config

STREAM_STATS, STREAM_PILOTS, STREAM_TAPS, STREAM_NOISE = 0, 1, 2, 3


def _rng(seed: int, cfg_id: int, stream: int, i: int, j: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, cfg_id, stream, i, j])))


def _tap_powers(L: int) -> np.ndarray:
    p = 10.0 ** (-0.3 * np.arange(L))
    return p / p.sum()


def rms_spread_taps(L: int) -> float:
    """rho_L: rms delay spread of the 3 dB/tap profile, in tap-spacing units (reading A6)."""
    p = _tap_powers(L)
    l = np.arange(L, dtype=np.float64)
    mean = (p * l).sum()
    return float(np.sqrt((p * l * l).sum() - mean * mean))


def slot_draws(cfg, seed: int, slot: int):
    """(tau_rms seconds or None, snr_db) of one slot (stream 0)."""
    cfg = get_config(cfg)
    rng = _rng(seed, cfg.cfg_id, STREAM_STATS, slot)
    tau_rms = cfg.tau_rms_s
    if cfg.tau_rms_range_s is not None:
        tau_rms = float(rng.uniform(*cfg.tau_rms_range_s))
    if cfg.snr_choice_db is not None:
        snr = float(rng.choice(np.asarray(cfg.snr_choice_db)))
    elif cfg.snr_range_db is not None:
        snr = float(rng.uniform(*cfg.snr_range_db))
    else:
        snr = float(cfg.snr_db)
    return tau_rms, snr


def pdp(cfg, tau_rms_s=None):
    """(p_l, tau_l in samples at the Nfft rate) of the exponential PDP (reading A6)."""
    cfg = get_config(cfg)
    L = cfg.n_taps
    p = _tap_powers(L)
    if cfg.tap_spacing is not None:
        delta = cfg.tap_spacing
    else:
        delta = tau_rms_s * cfg.fs_hz / rms_spread_taps(L)
    return p, delta * np.arange(L, dtype=np.float64)


def _slot_stats(cfg: Config, seed: int, slot: int):
    tau_rms, snr = slot_draws(cfg, seed, slot)
    p, tau = pdp(cfg, tau_rms)
    return p, tau, 10.0 ** (-snr / 10.0)


def channel_stats(cfg, seed: int = 0):
    """Per-set statistics handed to ce_init.

    Returns (r [n_sets][N] complex128, sigma2 [n_sets] float64).  With
    per_slot_stats the set of slot s is s; otherwise one set (slot 0 draws).
    """
    cfg = get_config(cfg)
    d = np.arange(cfg.N, dtype=np.float64)
    r = np.empty((cfg.n_sets, cfg.N), np.complex128)
    s2 = np.empty(cfg.n_sets, np.float64)
    for s in range(cfg.n_sets):
        p, tau, sigma2 = _slot_stats(cfg, seed, s)
        r[s] = (p[None, :] * np.exp(-2j * np.pi * np.outer(d, tau) / cfg.Nfft)).sum(axis=1)
        s2[s] = sigma2
    return r, s2


def set_of_instance(cfg) -> np.ndarray:
    """int32 [T]: statistic set of each estimation instance (reading A3/A4)."""
    cfg = get_config(cfg)
    t = np.arange(cfg.T)
    if cfg.per_slot_stats:
        return (t // cfg.pilots_per_slot).astype(np.int32)
    return np.zeros(cfg.T, np.int32)


def gen_pilots(cfg, seed: int = 0, t_lo: int = 0, t_hi=None) -> np.ndarray:
    """complex64 [t_hi-t_lo][K][N] unit-modulus QPSK pilots (stream 1, per instance)."""
    cfg = get_config(cfg)
    t_hi = cfg.T if t_hi is None else t_hi
    out = np.empty((t_hi - t_lo, cfg.K, cfg.N), np.complex64)
    a = np.float32(1.0 / np.sqrt(2.0))
    for i, t in enumerate(range(t_lo, t_hi)):
        bits = _rng(seed, cfg.cfg_id, STREAM_PILOTS, t).integers(0, 2, size=(2, cfg.K, cfg.N))
        out[i].real = a * (1 - 2 * bits[0])
        out[i].imag = a * (1 - 2 * bits[1])
    return out


def gen_instances(cfg, seed: int = 0, t_lo: int = 0, t_hi=None, m_lo: int = 0, m_hi=None,
                  x=None, return_channel: bool = False, noiseless: bool = False):
    """Received pilot symbols y, complex64 [t][m][K][N] for t in [t_lo,t_hi), m in [m_lo,m_hi).

    ``x`` (pilots for the same t range) may be passed to avoid redrawing.  With
    ``return_channel`` also returns the true H (complex128, same shape).
    """
    cfg = get_config(cfg)
    t_hi = cfg.T if t_hi is None else t_hi
    m_hi = cfg.M if m_hi is None else m_hi
    if x is None:
        x = gen_pilots(cfg, seed, t_lo, t_hi)
    nt, nm = t_hi - t_lo, m_hi - m_lo
    y = np.empty((nt, nm, cfg.K, cfg.N), np.complex64)
    H_all = np.empty((nt, nm, cfg.K, cfg.N), np.complex128) if return_channel else None
    n = np.arange(cfg.N, dtype=np.float64)
    slot_cache = {}
    for i, t in enumerate(range(t_lo, t_hi)):
        slot = t // cfg.pilots_per_slot
        if slot not in slot_cache:
            st = slot if cfg.per_slot_stats else 0
            p, tau, sigma2 = _slot_stats(cfg, seed, st)
            E = np.exp(-2j * np.pi * np.outer(tau, n) / cfg.Nfft)      # [L][N]
            slot_cache[slot] = (p, E, sigma2)
        p, E, sigma2 = slot_cache[slot]
        xt = x[i].astype(np.complex128)
        for j, m in enumerate(range(m_lo, m_hi)):
            g = _rng(seed, cfg.cfg_id, STREAM_TAPS, slot, m)
            h = (g.standard_normal((cfg.K, cfg.n_taps)) + 1j * g.standard_normal((cfg.K, cfg.n_taps)))
            h *= np.sqrt(p / 2.0)[None, :]
            H = h @ E                                                    # [K][N]
            yt = H * xt
            if not noiseless:
                gw = _rng(seed, cfg.cfg_id, STREAM_NOISE, t, m)
                w = gw.standard_normal((2, cfg.K, cfg.N))
                yt = yt + np.sqrt(sigma2 / 2.0) * (w[0] + 1j * w[1])
            y[i, j] = yt.astype(np.complex64)
            if return_channel:
                H_all[i, j] = H
    if return_channel:
        return y, H_all
    return y
